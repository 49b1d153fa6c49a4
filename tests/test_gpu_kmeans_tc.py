"""K1 tcgen05 assignment: the tensor-core filter + exact f64 fix-up must give
the same labels / centroids / iteration counts as the exact CUDA-core path
and the CPU oracle — across unit switches inside the persistent kernel,
C spanning one and two 256-column TMEM chunks, and converged units dropping
out of later passes."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import to_bf16_representable
from tests._inputs import head, port

pytestmark = pytest.mark.gpu


def _batched_kmeans(keys_units, Cn, seeds, max_iters, flags):
    import torch
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200.api import Context
    ctx = Context.default()
    U, n, d = keys_units.shape
    bits = (np.ascontiguousarray(keys_units, np.float32).view(np.uint32) >> 16).astype(np.uint16)
    kb = torch.from_numpy(bits.view(np.int16)).to(ctx.device)
    rows = np.stack([port().kmeans_init_rows(n, Cn, s) for s in seeds]).astype(np.uint32)
    dr = torch.from_numpy(rows.view(np.int32)).to(ctx.device)
    cents = torch.zeros((U, Cn, d), dtype=torch.float32, device=ctx.device)
    labels = torch.zeros((U, n), dtype=torch.int32, device=ctx.device)
    desc = N.KMeansDesc(U, n, Cn, max_iters, n * d, Cn, n, flags)
    info = (N.KMeansInfo * U)()
    N.check(N.lib().ckv_kmeans(ctx.h, C.byref(desc), kb.data_ptr(), dr.data_ptr(),
                               cents.data_ptr(), labels.data_ptr(), info, None, None))
    return (cents.cpu().numpy(), labels.cpu().numpy(),
            [(i.iterations_used, bool(i.converged)) for i in info])


@pytest.mark.parametrize("Cn,n,U", [(51, 4080, 5), (409, 4096, 3), (500, 2048, 2), (33, 700, 4)])
def test_tc_path_equals_exact_path(gpu_ctx, Cn, n, U):
    from paper_2412_03213_b200 import _native as N
    keys = np.stack([head(17, 0, u, n + 16)["K"][16:] for u in range(U)])
    seeds = [port().mix_seed(0, 0, u) for u in range(U)]
    c1, l1, i1 = _batched_kmeans(keys, Cn, seeds, 50, 0)
    c2, l2, i2 = _batched_kmeans(keys, Cn, seeds, 50, N.CKV_KM_EXACT_ONLY)
    assert i1 == i2
    assert np.array_equal(l1, l2)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))


def test_tc_path_vs_oracle_c409(gpu_ctx):
    """C = 409 (the 32k C0), two TMEM chunks, against the CPU oracle."""
    keys = head(23, 1, 2, 4096 + 16)["K"][16:]
    seed = port().mix_seed(0, 1, 2)
    c, l, info = _batched_kmeans(keys[None], 409, [seed], 50, 0)
    o = port().kmeans(keys, 409, seed, 50)
    assert info[0] == (o.iterations_used, o.converged)
    assert np.array_equal(l[0], o.labels)
    assert np.array_equal(c[0].view(np.uint32), o.centroids.view(np.uint32))


def test_tc_path_near_ties(gpu_ctx):
    """Keys built so many scores tie or nearly tie in bf16: exercises the
    fix-up list (2-4 candidates and the full re-score)."""
    rng = np.random.default_rng(3)
    base = rng.standard_normal((64, 128)).astype(np.float32)
    keys = base[rng.integers(0, 64, 3000)] + 1e-3 * rng.standard_normal((3000, 128)).astype(np.float32)
    keys = to_bf16_representable(keys)
    from paper_2412_03213_b200 import _native as N
    seeds = [11]
    c1, l1, i1 = _batched_kmeans(keys[None], 96, seeds, 30, 0)
    c2, l2, i2 = _batched_kmeans(keys[None], 96, seeds, 30, N.CKV_KM_EXACT_ONLY)
    assert i1 == i2 and np.array_equal(l1, l2)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))


@pytest.mark.parametrize("Cn,n,U", [(513, 4096, 2), (1638, 8192, 2), (1100, 3000, 3)])
def test_tc_multi_range_equals_exact_path(gpu_ctx, Cn, n, U):
    """C > 512 (config E: C0 = 1638): column ranges with their own resident
    B, per-range summaries merged by k_assign_merge, then the fix-up."""
    from paper_2412_03213_b200 import _native as N
    keys = np.stack([head(19, 0, u, n + 16)["K"][16:] for u in range(U)])
    seeds = [port().mix_seed(0, 3, u) for u in range(U)]
    c1, l1, i1 = _batched_kmeans(keys, Cn, seeds, 6, 0)
    c2, l2, i2 = _batched_kmeans(keys, Cn, seeds, 6, N.CKV_KM_EXACT_ONLY)
    assert i1 == i2
    assert np.array_equal(l1, l2)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))


def test_tc_multi_range_near_ties(gpu_ctx):
    rng = np.random.default_rng(5)
    base = rng.standard_normal((700, 128)).astype(np.float32)
    keys = base[rng.integers(0, 700, 6000)] + 1e-3 * rng.standard_normal((6000, 128)).astype(np.float32)
    keys = to_bf16_representable(keys)
    from paper_2412_03213_b200 import _native as N
    c1, l1, i1 = _batched_kmeans(keys[None], 900, [5], 8, 0)
    c2, l2, i2 = _batched_kmeans(keys[None], 900, [5], 8, N.CKV_KM_EXACT_ONLY)
    assert i1 == i2 and np.array_equal(l1, l2)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))


def test_tc_multi_range_vs_oracle(gpu_ctx):
    keys = head(29, 0, 1, 6000 + 16)["K"][16:]
    c, l, info = _batched_kmeans(keys[None], 700, [77], 4, 0)
    o = port().kmeans(keys, 700, 77, 4)
    assert info[0] == (o.iterations_used, o.converged)
    assert np.array_equal(l[0], o.labels)
    assert np.array_equal(c[0].view(np.uint32), o.centroids.view(np.uint32))
