"""The native sequence-sharded k-means (ckv_kmeans_sharded, ckv_comm.cu): the
reference loop in C++ with NCCL / LOCAL collectives, no torch.distributed.

world 1 over NCCL (one GPU per rank: gpurun gives one); worlds 2-3 over the
LOCAL backend, the ranks as threads sharing cuda:0, each with its own context
(the C-ABI releases the GIL).  Results equal the single-process CPU oracle
bit for bit (labels, centroids, iterations, convergence, repair passes)."""
import threading

import numpy as np
import pytest

from tests._inputs import bf16_bits, head, port

pytestmark = pytest.mark.gpu


def _run(keys, C_, seeds, max_iters, init_rows, world, backend):
    import torch

    from paper_2412_03213_b200.api import Context
    from paper_2412_03213_b200.sharded import NativeComm, kmeans_cosine_native, shard_range
    U, n_total, _ = keys.shape
    group = NativeComm.local_group(world) if backend == "local" else None
    out, errs = [None] * world, []

    def rank_fn(r):
        try:
            torch.cuda.set_device(0)
            ctx = Context(0)
            lo, hi = shard_range(n_total, world, r)
            kb = torch.from_numpy(bf16_bits(keys[:, lo:hi]).view(np.int16)).cuda(0)
            comm = NativeComm(ctx, world, r, group=group)
            res = kmeans_cosine_native(kb, C_, n_total, lo, comm, seeds=seeds,
                                       init_rows=init_rows, max_iters=max_iters)
            ctx.sync()
            out[r] = dict(labels=res.labels.cpu().numpy(), centroids=res.centroids.cpu().numpy(),
                          iters=res.iterations_used, converged=res.converged,
                          reps=res.repair_iterations)
            comm.close()
        except Exception as e:  # surfaced in the main thread
            errs.append(e)

    th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errs, errs
    return out


def _check(res, keys, C_, seeds, max_iters=50, init_rows=None):
    for u in range(keys.shape[0]):
        o = port().kmeans(keys[u], C_, seeds[u] if seeds is not None else 0, max_iters,
                          init_rows=None if init_rows is None else init_rows[u])
        labels = np.concatenate([r["labels"][u] for r in res])
        assert np.array_equal(labels, o.labels), f"unit {u}: labels differ"
        for r in res:
            assert np.array_equal(r["centroids"][u].view(np.uint32), o.centroids.view(np.uint32))
            assert int(r["iters"][u]) == o.iterations_used
            assert bool(r["converged"][u]) == o.converged
            assert r["reps"][u] == len(o.repair_iterations)


def test_native_sharded_nccl_world1(gpu_ctx):
    # L = 8192: C0 = 102 clusters -> the tensor-core assignment
    keys = np.stack([head(11, 2, h, 8192)["K"][16:] for h in range(2)])
    seeds = [port().mix_seed(0, 2, h) for h in range(2)]
    _check(_run(keys, 102, seeds, 50, None, 1, "nccl"), keys, 102, seeds)


@pytest.mark.parametrize("world", [2, 3])
def test_native_sharded_local_threads(gpu_ctx, world):
    keys = np.stack([head(11, 2, h, 8192)["K"][16:] for h in range(2)])
    seeds = [port().mix_seed(0, 2, h) for h in range(2)]
    _check(_run(keys, 102, seeds, 50, None, world, "local"), keys, 102, seeds)


def test_native_sharded_repair(gpu_ctx):
    rng = np.random.default_rng(3)
    base = rng.standard_normal(128).astype(np.float32)
    keys = rng.standard_normal((300, 128)).astype(np.float32)
    keys[:90] = base
    from oracle.oracle import to_bf16_representable
    keys = to_bf16_representable(keys)[None]
    init = np.array([[0, 1, 2, 150, 151, 200, 250, 299]], np.uint32)
    o = port().kmeans(keys[0], 8, 0, 50, init_rows=init[0])
    assert len(o.repair_iterations) > 0
    _check(_run(keys, 8, None, 50, init, 2, "local"), keys, 8, None, init_rows=init)


def test_native_sharded_max_iters_cap(gpu_ctx):
    keys = np.stack([head(5, 1, 2, 816)["K"][16:]])
    seeds = [port().mix_seed(0, 1, 2)]
    _check(_run(keys, 10, seeds, 2, None, 2, "local"), keys, 10, seeds, max_iters=2)


def test_native_sharded_cpp_host(gpu_ctx):
    """The same protocol from a C++ host through the C-ABI only (no torch):
    worlds 1 (NCCL) and 2-3 (LOCAL threads) vs the C oracle."""
    import subprocess

    from tests.cpp import build as B
    exe = B.build_sharded()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sharded_native: OK" in r.stdout, r.stdout + r.stderr
