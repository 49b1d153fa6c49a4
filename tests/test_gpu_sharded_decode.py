"""Sequence-sharded decode step on the B200 kernels.

Each rank holds a contiguous position shard of the keys and values (rank 0
also the 16 sinks, the last rank the recency window).  Sharded k-means ->
centroid-sharded exact scoring -> all-gather -> global budgeted top-k ->
local sparse attention -> LSE merge.  Checked against the single-process
oracle on the whole head: ranked clusters, n_taken, trimmed_from_last and
the reassembled I_T bit-exact; output and weights within the attention
tolerance of DESIGN.md §5.
"""
import numpy as np
import pytest

from tests._dist import run_world
from tests._inputs import head, port

pytestmark = pytest.mark.gpu


def _assemble(res, key, h, n_taken):
    """Global I_T order from the ranks' shares: each taken cluster's slices
    in rank (= position) order, then rank 0's sinks, then the recency."""
    parts = []
    for i in range(n_taken):
        for r in res:
            parts.append(r[key][h][r["off"][h][i]:r["off"][h][i + 1]])
    for r in res:
        nt, cl = int(r["n_tokens"][h]), int(r["off"][h][n_taken])
        parts.append(r[key][h][cl:nt])
    return np.concatenate(parts)


@pytest.mark.parametrize("world,L,budget,full_rank,exact", [
    (1, 1040, 256, True, False), (2, 1040, 256, True, False), (3, 2064, 300, True, True),
    (2, 2064, 5000, True, False), (1, 1040, 256, False, False), (2, 2064, 300, False, False),
    (3, 4112, 1000, False, False), (2, 2064, 5000, False, False), (2, 4112, 700, False, True)])
def test_gpu_sharded_decode_matches_reference(gpu_ctx, world, L, budget, full_rank, exact):
    from oracle.oracle import ClusterConfig as OCfg
    G, U, n_rec = 2, 2, 5
    hs = [head(9, 0, u, L, T=64) for u in range(U)]
    K = np.stack([x["K"] for x in hs])
    V = np.stack([x["V"] for x in hs])
    Kr = np.stack([x["dK"][:n_rec] for x in hs])
    Vr = np.stack([x["dV"][:n_rec] for x in hs])
    Q = np.stack([hs[u]["Q"][7 + 20 * g] for u in range(U) for g in range(G)])
    seeds = [port().mix_seed(0, 0, u) for u in range(U)]
    C0 = port().prefill_cluster_count(L, OCfg())
    res = run_world(world, "tests._sharded_workers", "decode_rank", K, V, Q, Kr, Vr, C0, seeds,
                    G, budget, 0, full_rank, exact)
    for u in range(U):
        o = port().cluster_prefill(K[u], OCfg(seed=seeds[u]))
        assert all(int(r["iters"][u]) == o.iterations_used for r in res)
        Kall = np.concatenate([K[u], Kr[u]])
        Vall = np.concatenate([V[u], Vr[u]])
        for g in range(G):
            h = u * G + g
            sel = port().select_tokens(Q[h], o.centroids, o.labels, 16, budget,
                                       recency=np.arange(L, L + n_rec, dtype=np.uint32))
            for r in res:
                assert int(r["n_taken"][h]) == sel.n_clusters_taken
                assert int(r["trimmed"][h]) == sel.trimmed_from_last
                nr = C0 if full_rank else sel.n_clusters_taken
                assert np.array_equal(r["ranked"][h][:nr], sel.ranked_clusters[:nr])
            ids = _assemble(res, "ids", h, sel.n_clusters_taken)
            assert np.array_equal(ids, sel.token_ids), f"I_T differs for q head {h}"
            oo, ow = port().approx_attention(Q[h], Kall, Vall, sel.token_ids)
            w = _assemble(res, "w", h, sel.n_clusters_taken)
            assert np.abs(w - ow).max() <= 1e-6 + 2e-5 * ow.max()
            for r in res:
                assert np.abs(r["out"][h] - oo).max() <= 2e-5 * np.abs(Vall).max()
