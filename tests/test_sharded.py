"""Sequence-sharded k-means protocol on CPU.

world_size 2 and 3 under gloo, each rank holding a contiguous position shard
and running paper_2412_03213_b200.sharded.kmeans_cosine_sharded with the CPU
checker steps (tests/_shard_cpu.py).  The result must equal the single-process
reference restatement (oracle) bit for bit: labels, centroids, iteration
counts, convergence, repair iterations; objective within 1e-9 relative (its
summation order differs across shards).  The GPU version of the same test
(DeviceShard, the CUDA kernels) is tests/test_gpu_sharded.py.
"""
import numpy as np
import pytest

from tests._dist import run_world
from tests._inputs import head, port


def _check(results, keys, C_, seeds, max_iters=50, init_rows=None):
    U = keys.shape[0]
    for u in range(U):
        o = port().kmeans(keys[u], C_, seeds[u] if seeds is not None else 0, max_iters,
                          init_rows=None if init_rows is None else init_rows[u])
        labels = np.concatenate([r["labels"][u] for r in results])
        assert np.array_equal(labels, o.labels), f"unit {u}: labels differ"
        for r in results:  # every rank holds the same centroids
            assert np.array_equal(r["centroids"][u].view(np.uint32), o.centroids.view(np.uint32))
            assert int(r["iters"][u]) == o.iterations_used
            assert bool(r["converged"][u]) == o.converged
            assert list(r["reps"][u]) == list(o.repair_iterations)
            np.testing.assert_allclose(r["obj"][u], o.objective_history, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_kmeans_matches_reference(world):
    keys = np.stack([head(7, 0, h, 1040)["K"][16:] for h in range(2)])  # N = 1024
    seeds = [port().mix_seed(0, 0, h) for h in range(2)]
    res = run_world(world, "tests._sharded_workers", "kmeans_rank", keys, 13, seeds, 50, None,
                    None)
    assert [r["lo"] for r in res] == [1024 * k // world for k in range(world)]
    _check(res, keys, 13, seeds)


def test_sharded_kmeans_max_iters_cap():
    keys = np.stack([head(5, 1, 2, 816)["K"][16:]])
    seeds = [port().mix_seed(0, 1, 2)]
    res = run_world(2, "tests._sharded_workers", "kmeans_rank", keys, 10, seeds, 2, None, None)
    _check(res, keys, 10, seeds, max_iters=2)


def test_sharded_kmeans_empty_cluster_repair():
    # 24 copies of one key: two init centroids on it tie, every copy goes to
    # the lower id, the other cluster is empty and gets repaired from the
    # largest cluster's farthest member, which may live on either shard
    rng = np.random.default_rng(3)
    base = rng.standard_normal(128).astype(np.float32)
    keys = rng.standard_normal((60, 128)).astype(np.float32)
    keys[:24] = base
    from oracle.oracle import to_bf16_representable
    keys = to_bf16_representable(keys)[None]
    init = np.array([[0, 1, 30, 31, 45, 50]], np.uint32)
    res = run_world(2, "tests._sharded_workers", "kmeans_rank", keys, 6, None, 50, init, None)
    o = port().kmeans(keys[0], 6, 0, 50, init_rows=init[0])
    assert len(o.repair_iterations) > 0, "the fixture must force a repair"
    _check(res, keys, 6, None, init_rows=init)


def test_sharded_kmeans_validation():
    zero = np.zeros((1, 40, 128), np.float32)
    with pytest.raises(RuntimeError, match="degenerate input"):
        run_world(2, "tests._sharded_workers", "kmeans_rank", zero, 3, [1], 50, None, None)
    keys = np.stack([head(7, 0, 0, 80)["K"][16:]])
    with pytest.raises(RuntimeError, match="need 1 <= C <= N"):
        run_world(2, "tests._sharded_workers", "kmeans_rank", keys, 65, [1], 50, None, None)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_decode_sizes_and_trim_shares(world):
    """Host side of the sharded decode step under gloo: the all-gathered
    global sizes equal build_index's over the whole head, every rank's prefix
    is the members on lower shards, and the per-rank shares of a trimmed
    cluster (k_select_scored's clamp(allow - prefix, 0, local)) reassemble the
    reference's lowest-position trim."""
    rng = np.random.default_rng(world)
    C_, n = 37, 1000
    labels = rng.integers(0, C_, (2, n)).astype(np.int32)
    res = run_world(world, "tests._sharded_workers", "sizes_rank", labels, C_)
    for u in range(2):
        sizes, _, sorted_ids = port().build_index(labels[u], C_)
        for r in res:
            assert np.array_equal(r["g"][u], sizes)
        acc = np.zeros(C_, np.int64)
        for r in res:
            assert np.array_equal(r["p"][u], acc)
            acc += r["lsize"][u]
        for c in range(C_):
            for allow in (0, 1, int(sizes[c]) // 2, int(sizes[c])):
                allow = min(allow, int(sizes[c]))
                take = [min(max(allow - int(r["p"][u][c]), 0), int(r["lsize"][u][c])) for r in res]
                assert sum(take) == allow
                # shard s's share = its lowest-position members of c, in rank order
                members = np.nonzero(labels[u] == c)[0]
                got = np.concatenate([members[(members >= k * n // world) &
                                              (members < (k + 1) * n // world)][:take[k]]
                                      for k in range(world)])
                assert np.array_equal(got, members[:allow])
    slices = [r["slice"] for r in res]
    assert all(s[0] * world >= C_ for s in slices) and [s[1] for s in slices] == \
        [k * slices[0][0] for k in range(world)]
