"""CPU-only: the C restatement (oracle/ckv_oracle.c) is pinned against the
compiled reference (oracle/_ref) and the committed golden fixtures."""
import os

import numpy as np
import pytest

from oracle.oracle import ClusterConfig, to_bf16_representable

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_mt19937_64_known_answer(port):
    import ctypes as C
    from oracle.oracle import Oracle
    lib = port.lib

    class MT(C.Structure):
        _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_uint32)]
    g = MT()
    lib.orc_mt64_seed.argtypes = [C.POINTER(MT), C.c_uint64]
    lib.orc_mt64_next.argtypes = [C.POINTER(MT)]
    lib.orc_mt64_next.restype = C.c_uint64
    lib.orc_mt64_seed(C.byref(g), 5489)
    for _ in range(9999):
        lib.orc_mt64_next(C.byref(g))
    # C++ standard [rand.predef]: 10000th output of default-constructed mt19937_64
    assert lib.orc_mt64_next(C.byref(g)) == 9981545732273789042


def test_spec_kats(port):
    cfg = ClusterConfig()
    assert port.prefill_cluster_count(32016, cfg) == 400
    assert port.prefill_cluster_count(96, cfg) == 1
    assert port.prefill_cluster_count(16, cfg) == 0
    s, st, srt = port.build_index(np.array([2, 0, 1, 1, 1, 2], np.int32), 3)
    assert list(s) == [1, 3, 2] and list(srt) == [1, 2, 3, 4, 0, 5] and list(st) == [0, 1, 4, 6]


def test_generator_port_vs_reference(port, ref):
    for seed in (0, 7, 99):
        a = port.generate_head(seed, 300, 20)
        b = ref.generate_head(seed, 300, 20)
        for f in ("prompt_keys", "prompt_values", "decode_queries", "decode_keys", "decode_values"):
            assert np.array_equal(getattr(a, f), getattr(b, f))


@pytest.mark.parametrize("L,seed", [(600, 1), (1500, 2), (2048, 3)])
def test_kmeans_select_attention_port_vs_reference(port, ref, L, seed):
    tr = port.generate_head(port.mix_seed(7, 0, seed), L, 32)
    K, V = to_bf16_representable(tr.prompt_keys), to_bf16_representable(tr.prompt_values)
    cfg = ClusterConfig(seed=port.mix_seed(0, 0, seed))
    a, b = port.cluster_prefill(K, cfg), ref.cluster_prefill(K, cfg)
    assert a.iterations_used == b.iterations_used and a.converged == b.converged
    assert np.array_equal(a.labels, b.labels)
    assert np.array_equal(a.centroids, b.centroids)
    assert np.array_equal(a.objective_history, b.objective_history)
    rec = np.arange(L, L + 5, dtype=np.uint32)
    for t in (0, 13):
        q = to_bf16_representable(tr.decode_queries[t])
        sa = port.select_tokens(q, a.centroids, a.labels, a.sink_count, 256, rec)
        sb = ref.select_tokens(q, b.centroids, b.labels, b.sink_count, 256, rec)
        assert np.array_equal(sa.ranked_clusters, sb.ranked_clusters)
        assert np.array_equal(sa.token_ids, sb.token_ids)
        assert sa.trimmed_from_last == sb.trimmed_from_last
        ids = sa.token_ids[sa.token_ids < L]
        oa, wa = port.approx_attention(q, K, V, ids)
        ob, wb = ref.approx_attention(q, K, V, ids)
        assert np.array_equal(oa, ob) and np.array_equal(wa, wb)


@pytest.mark.parametrize("n,C_", [(16384, 205), (9000, 403)])
def test_threaded_assign_port_vs_reference(port, ref, n, C_):
    """The port's multi-threaded, 4-chain-interleaved cosine assignment (the
    path large checks take, n*C >= 2^21) equals the reference's sequential
    AssignScorer (clustering.hpp:104-115) — C odd and not a multiple of 4
    exercises the tail chain."""
    tr = port.generate_head(port.mix_seed(7, 3, n), n + 16, 4)
    K = to_bf16_representable(tr.prompt_keys[16:])
    a, b = port.kmeans(K, C_, 5, 2), ref.kmeans(K, C_, 5, 2)
    assert a.iterations_used == b.iterations_used == 2
    assert np.array_equal(a.labels, b.labels)
    assert np.array_equal(a.centroids.view(np.uint32), b.centroids.view(np.uint32))


def test_repair_and_decode_batch_port_vs_reference(port, ref):
    rng = np.random.default_rng(5)
    base = rng.standard_normal((6, 128)).astype(np.float32)
    K = to_bf16_representable(base[rng.integers(0, 6, 64)] +
                              0.01 * rng.standard_normal((64, 128)).astype(np.float32))
    for s in range(4):
        a, b = port.kmeans(K, 40, s), ref.kmeans(K, 40, s)
        assert np.array_equal(a.labels, b.labels) and np.array_equal(a.centroids, b.centroids)
        assert list(a.repair_iterations) == list(b.repair_iterations)
    tr = port.generate_head(3, 500, 330)
    cfg = ClusterConfig(seed=11)
    a = port.cluster_prefill(tr.prompt_keys, cfg)
    x = port.cluster_decode_batch(a.centroids, a.labels, tr.decode_keys[:320], cfg)
    y = ref.cluster_decode_batch(a.centroids, a.labels, tr.decode_keys[:320], cfg)
    assert all(np.array_equal(p, q) for p, q in zip(x, y))


def test_cache_port_vs_reference(port, ref):
    rng = np.random.default_rng(1)
    sizes = rng.integers(1, 50, 100).astype(np.uint32)
    for R in (1, 2):
        a, b = port.cache(R), ref.cache(R)
        for _ in range(30):
            sel = np.sort(rng.choice(100, 10, replace=False)).astype(np.uint32)
            ha, hb = a.lookup_and_update(sel, sizes), b.lookup_and_update(sel, sizes)
            assert all(np.array_equal(p, q) for p, q in zip(ha, hb))
            dead = rng.choice(100, 6, replace=False).astype(np.uint32)
            a.invalidate_on_recluster(dead)
            b.invalidate_on_recluster(dead)
        assert np.array_equal(a.counters(), b.counters())


def test_golden_fixtures(port):
    """Fixtures produced by the compiled reference (tests/golden/make_golden.py)."""
    path = os.path.join(GOLD, "golden_v1.npz")
    g = np.load(path)
    tr = port.generate_head(int(g["gen_seed"]), int(g["gen_L"]), int(g["gen_T"]))
    assert np.array_equal(tr.prompt_keys, g["gen_prompt_keys"])
    assert np.array_equal(tr.decode_queries, g["gen_decode_queries"])
    K = g["km_keys"]
    cfg = ClusterConfig(seed=int(g["km_seed"]))
    m = port.cluster_prefill(K, cfg)
    assert m.iterations_used == int(g["km_iters"]) and m.converged == bool(g["km_converged"])
    assert np.array_equal(m.labels, g["km_labels"])
    assert np.array_equal(m.centroids, g["km_centroids"])
    assert np.array_equal(m.objective_history, g["km_objective"])
    s = port.select_tokens(g["sel_q"], m.centroids, m.labels, m.sink_count, int(g["sel_budget"]),
                           g["sel_recency"])
    assert np.array_equal(s.ranked_clusters, g["sel_ranked"])
    assert np.array_equal(s.token_ids, g["sel_token_ids"])
    assert s.n_clusters_taken == int(g["sel_taken"]) and s.trimmed_from_last == int(g["sel_trimmed"])
    o, w = port.approx_attention(g["sel_q"], K, g["att_values"], g["att_rows"])
    assert np.array_equal(o, g["att_out"]) and np.array_equal(w, g["att_weights"])
    c = port.cache(2)
    for i in range(g["cache_sel"].shape[0]):
        c.lookup_and_update(g["cache_sel"][i][g["cache_sel"][i] >= 0].astype(np.uint32),
                            g["cache_sizes"])
    assert np.array_equal(c.counters(), g["cache_counters"])
    cc, ll, it = port.cluster_decode_batch(m.centroids, m.labels, g["dec_keys"], cfg)
    assert np.array_equal(cc, g["dec_centroids"]) and np.array_equal(ll, g["dec_labels"])


def test_page_select_port_matches_reference(ref):
    """orc_page_select restates selection.hpp:141-194 bit for bit."""
    from oracle.oracle import Oracle, to_bf16_representable
    P = Oracle("port")
    rng = np.random.default_rng(0)
    for n, B, ps, mm in ((1000, 256, 16, 0), (1000, 256, 16, 1), (37, 100, 7, 1),
                         (4096, 1024, 32, 0), (10, 5, 16, 0), (200, 64, 16, 1)):
        K = to_bf16_representable(rng.standard_normal((n, 128)).astype(np.float32))
        q = to_bf16_representable(rng.standard_normal(128).astype(np.float32))
        assert np.array_equal(P.page_select(q, K, B, ps, mm), ref.page_select(q, K, B, ps, mm))


def test_generate_synthetic_bundle_port_vs_reference(port, ref, tmp_path):
    """orc_generate_synthetic (the whole bundle, per-head sub-seeds) equals
    the reference's generate_synthetic, read back from its own CKVT file."""
    from paper_2412_03213_b200 import trace as T
    p = tmp_path / "b.ckvt"
    assert ref.lib.ref_write_synthetic_trace(str(p).encode(), 8, 7, 300, 20, 128, 2, 3) == 0
    b = T.read_trace(str(p))
    tr = port.generate_synthetic(7, 2, 3, 300, 20)
    for u in range(6):
        for name in T.NAMES:
            assert np.array_equal(getattr(b.traces[u], name), getattr(tr, name)[u]), (u, name)
