"""Sequence-sharded k-means on the B200 kernels.

Two ranks share cuda:0 (gpurun gives one GPU), each with its own context and
its contiguous shard of the keys, the collectives staged through gloo; the
per-shard steps are the CUDA kernels (DeviceShard -> ckv_kmshard.cu, the
tensor-core assignment when C fits).  Results must equal the single-process
CPU oracle bit for bit, as for the unsharded path (tests/test_gpu_kmeans.py).
"""
import numpy as np
import pytest

from tests._dist import run_world
from tests._inputs import head, port
from tests.test_sharded import _check

pytestmark = pytest.mark.gpu


def test_gpu_sharded_kmeans_exact_path(gpu_ctx):
    keys = np.stack([head(7, 0, h, 1040)["K"][16:] for h in range(2)])
    seeds = [port().mix_seed(0, 0, h) for h in range(2)]
    res = run_world(2, "tests._sharded_workers", "kmeans_rank", keys, 13, seeds, 50, None, 0)
    _check(res, keys, 13, seeds)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_gpu_sharded_kmeans_tensor_core_path(gpu_ctx, world):
    # L = 8192: N = 8176 keys, C0 = 102 clusters -> k_assign_tc on every shard
    keys = np.stack([head(11, 2, h, 8192)["K"][16:] for h in range(2)])
    seeds = [port().mix_seed(0, 2, h) for h in range(2)]
    res = run_world(world, "tests._sharded_workers", "kmeans_rank", keys, 102, seeds, 50, None, 0)
    _check(res, keys, 102, seeds)


def test_gpu_sharded_kmeans_repair(gpu_ctx):
    rng = np.random.default_rng(3)
    base = rng.standard_normal(128).astype(np.float32)
    keys = rng.standard_normal((300, 128)).astype(np.float32)
    keys[:90] = base
    from oracle.oracle import to_bf16_representable
    keys = to_bf16_representable(keys)[None]
    init = np.array([[0, 1, 2, 150, 151, 200, 250, 299]], np.uint32)
    res = run_world(2, "tests._sharded_workers", "kmeans_rank", keys, 8, None, 50, init, 0)
    o = port().kmeans(keys[0], 8, 0, 50, init_rows=init[0])
    assert len(o.repair_iterations) > 0
    _check(res, keys, 8, None, init_rows=init)
