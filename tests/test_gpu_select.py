"""K5 build_index, K6 select, K8 cache parity (integer outputs bit-exact)."""
import numpy as np
import pytest

from oracle.oracle import ClusterConfig as OCfg
from tests._inputs import head, port

pytestmark = pytest.mark.gpu


def _model(labels, cents, sink=0):
    from paper_2412_03213_b200 import api
    labels = np.asarray(labels, np.int32)
    cents = np.asarray(cents, np.float32).reshape(-1, 128)
    return api.ClusterModel(cents.shape[0], cents, labels, sink)


def test_index_fig6_kat(gpu_ctx):
    """SPEC.md:208 / Fig. 6."""
    from paper_2412_03213_b200 import api
    m = _model([2, 0, 1, 1, 1, 2], np.zeros((3, 128)))
    ix = api.build_index(m)
    assert list(ix.sizes) == [1, 3, 2]
    assert list(ix.sorted_token_ids) == [1, 2, 3, 4, 0, 5]
    assert list(ix.cluster_start) == [0, 1, 4, 6]


@pytest.mark.parametrize("n,C,frac_neg", [(1000, 7, 0.1), (36000, 457, 0.01), (5000, 3000, 0.0)])
def test_index_random_vs_oracle(gpu_ctx, n, C, frac_neg):
    from paper_2412_03213_b200 import api
    rng = np.random.default_rng(n)
    lab = rng.integers(0, C, n).astype(np.int32)
    lab[rng.random(n) < frac_neg] = -1
    lab[:16] = -1
    ix = api.build_index(_model(lab, np.zeros((C, 128))))
    s, st, srt = port().build_index(lab, C)
    assert np.array_equal(ix.sizes, s)
    assert np.array_equal(ix.cluster_start, st)
    assert np.array_equal(ix.sorted_token_ids, srt)


def test_select_fig6_and_trim_kats(gpu_ctx):
    """SPEC.md:228 (budget matches the 2nd prefix sum) and SPEC.md:230 trim."""
    from paper_2412_03213_b200 import api
    # clusters 0,1,2 with sizes [1,3,2]; q scores order: c0 > c2 > c1
    cents = np.zeros((3, 128), np.float32)
    cents[0, 0], cents[2, 0], cents[1, 0] = 3.0, 2.0, 1.0
    m = _model([2, 0, 1, 1, 1, 2], cents)
    ix = api.build_index(m)
    q = np.zeros(128, np.float32)
    q[0] = 1.0
    r = api.select_tokens(q, m, ix, 3)
    assert r.n_clusters_taken == 2 and r.trimmed_from_last == 0
    assert list(r.token_ids) == [1, 0, 5]
    # trim: A(4) then B(4) with budget 6 -> B keeps its 2 lowest positions
    lab = [0, 1, 0, 1, 0, 1, 0, 1]
    cents = np.zeros((2, 128), np.float32)
    cents[0, 0], cents[1, 0] = 2.0, 1.0
    m = _model(lab, cents)
    ix = api.build_index(m)
    r = api.select_tokens(q, m, ix, 6)
    assert r.n_clusters_taken == 2 and r.trimmed_from_last == 2
    assert list(r.token_ids) == [0, 2, 4, 6, 1, 3]


def test_select_ties_lowest_id(gpu_ctx):
    from paper_2412_03213_b200 import api
    cents = np.ones((5, 128), np.float32)
    m = _model([4, 3, 2, 1, 0, 0], cents)
    ix = api.build_index(m)
    r = api.select_tokens(np.ones(128, np.float32), m, ix, 2)
    assert list(r.ranked_clusters) == [0, 1, 2, 3, 4]
    assert list(r.token_ids) == [4, 5]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_select_near_ties_vs_oracle(gpu_ctx, seed):
    """Clusters in near-tied triples (copies a few ulps apart): their score
    bounds overlap, so the selection must take the exact f64 path for those
    and still match the oracle's ranking bit for bit; budgets land inside
    the triples.  Random clusters elsewhere take the disjoint-bounds path."""
    from paper_2412_03213_b200 import api
    rng = np.random.default_rng(40 + seed)
    base = rng.standard_normal((60, 128)).astype(np.float32)
    cents = np.repeat(base, 3, axis=0)
    for r in range(1, cents.shape[0], 3):
        j = rng.integers(0, 128, 3)
        cents[r, j] = np.nextafter(cents[r, j], np.float32(np.inf))
        cents[r + 1, j] = np.nextafter(cents[r + 1, j], np.float32(-np.inf))
    C = cents.shape[0]
    n = 6000
    lab = rng.integers(0, C, n).astype(np.int32)
    m = _model(lab, cents)
    ix = api.build_index(m)
    for t in range(6):
        q = base[rng.integers(0, 60)] + 0.05 * rng.standard_normal(128).astype(np.float32)
        for budget in (17, 100, 333):
            r = port().select_tokens(q, cents, lab, 0, budget, np.zeros(0, np.uint32))
            g = api.select_tokens(q, m, ix, budget)  # exhaustive (full ranking)
            assert np.array_equal(g.ranked_clusters, r.ranked_clusters)
            # the decode path's fast selection (candidate set + bounds)
            f = api._select(gpu_ctx, q, m, ix, budget, (), full_rank=False)[0]
            for x in (g, f):
                k = x.n_clusters_taken
                assert k == r.n_clusters_taken
                assert np.array_equal(x.ranked_clusters[:k], r.ranked_clusters[:k])
                assert x.trimmed_from_last == r.trimmed_from_last
                assert np.array_equal(x.token_ids, r.token_ids)


@pytest.mark.parametrize("budget", [1, 64, 1024, 5000])
def test_select_vs_oracle_config_a(gpu_ctx, budget):
    from paper_2412_03213_b200 import api
    h = head(7, 0, 2, 4096, T=64)
    seed = port().mix_seed(0, 0, 2)
    o = port().cluster_prefill(h["K"], OCfg(seed=seed))
    m = _model(o.labels, o.centroids, o.sink_count)
    ix = api.build_index(m)
    rec = np.arange(4096, 4096 + 37, dtype=np.uint32)
    for t in range(0, 64, 9):
        q = h["Q"][t]
        g = api.select_tokens(q, m, ix, budget, rec)
        r = port().select_tokens(q, o.centroids, o.labels, o.sink_count, budget, rec)
        assert np.array_equal(g.ranked_clusters, r.ranked_clusters)
        assert g.n_clusters_taken == r.n_clusters_taken
        assert g.trimmed_from_last == r.trimmed_from_last
        assert np.array_equal(g.token_ids, r.token_ids)
        sc = api.score_clusters(q, m)
        assert np.array_equal(sc.view(np.uint64), port().score_clusters(q, o.centroids).view(np.uint64))


def test_cache_sequence_vs_oracle(gpu_ctx):
    from paper_2412_03213_b200 import api
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 200, 400).astype(np.uint32)
    for R in (1, 2, 3):
        g = api.ClusterCache(R, 128, c_cap=512)
        o = port().cache(R)
        for t in range(40):
            sel = np.sort(rng.choice(400, rng.integers(0, 30), replace=False)).astype(np.uint32)
            gh, gm = g.lookup_and_update(sel, sizes)
            oh, om = o.lookup_and_update(sel, sizes)
            assert np.array_equal(gh, oh) and np.array_equal(gm, om)
        c = g.counters()
        oc = o.counters()
        assert [c["clusters_requested"], c["clusters_hit"], c["tokens_transferred"],
                c["bytes_transferred"]] == [int(x) for x in oc]
    with pytest.raises(ValueError):
        api.ClusterCache(0, 128)


def test_select_budget_zero_vs_oracle(gpu_ctx):
    """Budget 0 takes no cluster (selection.hpp:91 breaks at once): I_T is
    the sinks then the recency, the full ranking is still returned."""
    from paper_2412_03213_b200 import api
    h = head(7, 0, 1, 2048, T=8)
    seed = port().mix_seed(0, 0, 1)
    o = port().cluster_prefill(h["K"], OCfg(seed=seed))
    m = _model(o.labels, o.centroids, o.sink_count)
    ix = api.build_index(m)
    rec = np.arange(2048, 2048 + 5, dtype=np.uint32)
    g = api.select_tokens(h["Q"][3], m, ix, 0, rec)
    r = port().select_tokens(h["Q"][3], o.centroids, o.labels, o.sink_count, 0, rec)
    assert g.n_clusters_taken == r.n_clusters_taken == 0 and g.trimmed_from_last == 0
    assert np.array_equal(g.token_ids, r.token_ids)
    assert np.array_equal(g.ranked_clusters, r.ranked_clusters)


def test_select_capacity_checks(gpu_ctx):
    """The C-ABI rejects a token / row buffer too small for min(B, p_cap) +
    sinks + recency, and a cache narrower than the selection's c_cap, before
    any kernel could write out of range (CKV_EINVAL)."""
    import ctypes as C

    import torch

    from paper_2412_03213_b200 import _native as N
    dev = gpu_ctx.device
    n_q, c_cap, p_cap, B = 2, 64, 512, 100
    z = lambda n, dt=torch.int32: torch.zeros(n, dtype=dt, device=dev)
    q, cents = z(n_q * 128, torch.float32), z(n_q * c_cap * 128, torch.float32)
    ncl, sizes, starts, srt = z(n_q), z(n_q * c_cap), z(n_q * (c_cap + 1)), z(n_q * p_cap)
    outs = [z(n_q) for _ in range(3)]
    ranked = z(n_q * c_cap)
    for sel_cap, ok in ((B + 16 + 4, True), (B + 16 + 3, False)):
        tok = z(n_q * sel_cap)
        sd = N.SelectDesc(n_q, 1, B, 16, p_cap, c_cap, sel_cap, 600, 604, 0, 0)
        rc = N.lib().ckv_select(gpu_ctx.h, C.byref(sd), q.data_ptr(), cents.data_ptr(),
                                ncl.data_ptr(), sizes.data_ptr(), starts.data_ptr(),
                                srt.data_ptr(), tok.data_ptr(), None, None,
                                *[o.data_ptr() for o in outs], ranked.data_ptr(), None, None)
        assert (rc == N.CKV_OK) == ok, (sel_cap, rc)
    cache = C.c_void_p()
    N.check(N.lib().ckv_cache_create(gpu_ctx.h, n_q, c_cap // 2, 1, 128, C.byref(cache)))
    try:
        sd = N.SelectDesc(n_q, 1, B, 16, p_cap, c_cap, B + 20, 600, 604, 0, 0)
        rc = N.lib().ckv_select(gpu_ctx.h, C.byref(sd), q.data_ptr(), cents.data_ptr(),
                                ncl.data_ptr(), sizes.data_ptr(), starts.data_ptr(),
                                srt.data_ptr(), None, None, None, *[o.data_ptr() for o in outs],
                                ranked.data_ptr(), None, cache)
        assert rc == N.CKV_EINVAL
    finally:
        N.lib().ckv_cache_destroy(cache)
    torch.cuda.synchronize()


def test_cache_invalidate_on_recluster_vs_oracle(gpu_ctx):
    """cache.hpp:65-76: retired ids leave every retained set; later lookups
    (hits, misses, counters) match the reference's ClusterCache."""
    from paper_2412_03213_b200 import api
    rng = np.random.default_rng(3)
    sizes = rng.integers(1, 90, 300).astype(np.uint32)
    for R in (1, 2, 3):
        g = api.ClusterCache(R, 128, c_cap=320)
        o = port().cache(R)
        for t in range(30):
            sel = np.sort(rng.choice(300, rng.integers(1, 25), replace=False)).astype(np.uint32)
            gh, gm = g.lookup_and_update(sel, sizes)
            oh, om = o.lookup_and_update(sel, sizes)
            assert np.array_equal(gh, oh) and np.array_equal(gm, om), (R, t)
            if t % 3 == 1:
                dead = rng.choice(300, 40, replace=False).astype(np.uint32)
                g.invalidate_on_recluster(dead)
                o.invalidate_on_recluster(dead)
        c = g.counters()
        assert [c["clusters_requested"], c["clusters_hit"], c["tokens_transferred"],
                c["bytes_transferred"]] == [int(x) for x in o.counters()]
