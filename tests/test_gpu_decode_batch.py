"""K4 ckv_cluster_decode_batch (clustering.hpp:310-332) — the fused
one-launch k-means of every unit's decode batch (k_kmeans_small) — against
the CPU oracle: labels (with the fresh cluster ids), appended centroids and
iteration counts bit-exact; repairs forced with duplicated keys; the
reference's ValidationError predicates."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import ClusterConfig as OCfg
from oracle.oracle import to_bf16_representable
from tests._inputs import bf16_bits, head, port

pytestmark = pytest.mark.gpu


def _run(gpu_ctx, batches, base_clusters, c_plus, seeds, pos0, max_iters=50):
    import torch
    from paper_2412_03213_b200 import _native as N
    U, rows, _ = batches.shape
    p_cap, c_cap = pos0 + rows + 8, base_clusters + c_plus + 4
    dev = gpu_ctx.device
    keys = torch.zeros((U, p_cap, 128), dtype=torch.int16, device=dev)
    keys[:, pos0:pos0 + rows] = torch.from_numpy(bf16_bits(batches).view(np.int16)).to(dev)
    cents = torch.zeros((U, c_cap, 128), dtype=torch.float32, device=dev)
    labels = torch.full((U, p_cap), -7, dtype=torch.int32, device=dev)
    ncl = torch.full((U,), base_clusters, dtype=torch.int32, device=dev)
    desc = N.DecodeClusterDesc(U, pos0, rows, p_cap, c_cap, c_plus, max_iters)
    sd = (C.c_uint64 * U)(*seeds)
    it = (C.c_uint32 * U)()
    N.check(N.lib().ckv_cluster_decode_batch(gpu_ctx.h, C.byref(desc), keys.data_ptr(),
                                             C.cast(sd, C.c_void_p), cents.data_ptr(),
                                             labels.data_ptr(), ncl.data_ptr(), C.cast(it, C.c_void_p)))
    return (cents.cpu().numpy(), labels.cpu().numpy(), ncl.cpu().numpy(), list(it))


@pytest.mark.parametrize("rows,c_plus", [(320, 4), (100, 8), (512, 32), (3, 4), (1, 4)])
def test_decode_batch_matches_oracle(gpu_ctx, rows, c_plus):
    U, pos0, base = 3, 1000, 13
    batches = np.stack([head(5, 1, u, 64, T=max(rows, 2))["dK"][:rows] for u in range(U)])
    seeds = [port().mix_seed(0, 1, u) for u in range(U)]
    cents, labels, ncl, iters = _run(gpu_ctx, batches, base, c_plus, seeds, pos0)
    C_ = min(c_plus, rows)
    for u in range(U):
        oc0 = np.zeros((base, 128), np.float32)
        ol0 = np.full(pos0, -1, np.int32)
        oc, ol, oit = port().cluster_decode_batch(oc0, ol0, batches[u],
                                                  OCfg(seed=seeds[u], c_plus=c_plus))
        assert ncl[u] == base + C_
        assert iters[u] == oit
        assert np.array_equal(labels[u, pos0:pos0 + rows], ol[pos0:])
        assert np.array_equal(cents[u, base:base + C_].view(np.uint32),
                              oc[base:base + C_].view(np.uint32))
        assert (labels[u, :pos0] == -7).all()  # untouched


def test_decode_batch_repair(gpu_ctx):
    rng = np.random.default_rng(4)
    b = rng.standard_normal((1, 40, 128)).astype(np.float32)
    b[0, :30] = b[0, 0]  # most keys identical: init centroids tie -> empty clusters
    b = to_bf16_representable(b)
    for seed in range(6):
        cents, labels, ncl, iters = _run(gpu_ctx, b, 0, 6, [seed], 0)
        oc, ol, oit = port().cluster_decode_batch(np.zeros((0, 128), np.float32),
                                                  np.zeros(0, np.int32), b[0],
                                                  OCfg(seed=seed, c_plus=6))
        assert iters[0] == oit
        assert np.array_equal(labels[0, :40], ol)
        assert np.array_equal(cents[0, :6].view(np.uint32), oc.view(np.uint32))


def test_decode_batch_validation(gpu_ctx):
    from paper_2412_03213_b200._native import ValidationError
    z = np.zeros((2, 10, 128), np.float32)
    with pytest.raises(ValidationError, match="degenerate"):
        _run(gpu_ctx, z, 0, 4, [1, 2], 0)
    bad = to_bf16_representable(np.random.default_rng(1).standard_normal((2, 10, 128)).astype(np.float32))
    bad[1, 3, 5] = np.inf
    with pytest.raises(ValidationError, match="finite"):
        _run(gpu_ctx, bad, 0, 4, [1, 2], 0)
