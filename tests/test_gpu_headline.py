"""Parity at the shapes the bench times (BASELINE configs[1] and [4]).

north_star asks for indices bit-exact against the CPU oracle "at 32k
context with a 1k budget".  These tests run the SAME entry points and the
same scale-dependent code paths the bench runs — the batched 256-unit
ckv_cluster_prefill (memory-bounded unit batches, 256-tile units, the
fix-up volume of early passes), the session's decode fast path
(k_select_fused: approximate f32 scores, radix cut, candidate proof, exact
f64 re-scoring; no CKV_SEL_FULL_RANK), and at config E's shape the C > 512
multi-range tensor-core assignment and the sharded approximate selection
(k_select_approx at C = 1638, B = 2048) — and compare a sample of units
with the oracle (oracle/, pinned to the compiled reference in
test_oracle.py):

  k-means (clustering.hpp:160-263): labels, centroid bits, iterations,
      convergence and repair passes bit-exact;
  selection (selection.hpp:74-111) + cache (cache.hpp:38-57): the whole
      I_T (ranked taken clusters, trim, sinks, recency) and the hit/miss
      counters bit-exact;
  attention (attention.hpp:20-50): within DESIGN.md §5's tolerance.

Inputs: the bench's own device draw (bench.gen_inputs / fill_kv /
gen_decode) plus heads from the reference generator (trace.hpp:134-198).
"""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import ClusterConfig as OCfg
from tests._inputs import bf16_bits, head, port

pytestmark = pytest.mark.gpu

D = 128


def _f32(bits) -> np.ndarray:
    """bf16 bit patterns (int16/uint16, numpy or torch) -> f32 numpy."""
    if hasattr(bits, "cpu"):
        bits = bits.cpu().numpy()
    return (np.asarray(bits).view(np.uint16).astype(np.uint32) << 16).view(np.float32)


def _prefill(ctx, K, L, seeds, max_iters=50, c_cap=None):
    """ckv_cluster_prefill of every unit of K [U][p_cap][128] (device
    bf16 bits), exactly as bench.py calls it."""
    import torch
    from paper_2412_03213_b200 import _native as N
    U, p_cap = K.shape[0], K.shape[1]
    lib = N.lib()
    c0 = lib.ckv_prefill_cluster_count(L, 80, 16, 0)
    c_cap = c_cap or c0 + 64
    cents = torch.empty((U, c_cap, D), dtype=torch.float32, device=K.device)
    labels = torch.empty((U, p_cap), dtype=torch.int32, device=K.device)
    ncl = torch.empty((U,), dtype=torch.int32, device=K.device)
    info = (N.KMeansInfo * U)()
    reps = np.zeros(U * (max_iters + 1), np.uint32)
    desc = N.PrefillDesc(U, L, p_cap, c_cap, 80, 16, max_iters, 0, 0)
    sv = (C.c_uint64 * U)(*seeds)
    N.check(lib.ckv_cluster_prefill(ctx.h, C.byref(desc), K.data_ptr(), C.cast(sv, C.c_void_p),
                                    cents.data_ptr(), labels.data_ptr(), ncl.data_ptr(),
                                    C.cast(info, C.c_void_p), None, reps.ctypes.data))
    torch.cuda.synchronize()
    return c0, cents, labels, ncl, info, reps.reshape(U, max_iters + 1)


def _check_unit(u, Kf32, seed, c0, cents, labels, ncl, info, reps, max_iters=50):
    o = port().cluster_prefill(Kf32, OCfg(seed=seed, max_iters=max_iters))
    assert o.n_clusters == c0 == int(ncl[u])
    assert info[u].iterations_used == o.iterations_used, u
    assert bool(info[u].converged) == o.converged, u
    assert list(reps[u, : info[u].n_repair]) == list(o.repair_iterations), u
    L = Kf32.shape[0]
    assert np.array_equal(labels[u, :L].cpu().numpy(), o.labels), f"labels differ, unit {u}"
    g = cents[u, :c0].cpu().numpy()
    assert np.array_equal(g.view(np.uint32), o.centroids.view(np.uint32)), f"centroids, unit {u}"
    return o


def test_prefill_32k_all_bench_units(gpu_ctx):
    """Config B prefill: all 256 units (32 layers x 8 kv) of 32k keys in ONE
    ckv_cluster_prefill call, C0 = 409, up to 50 iterations; units 0-1 are
    reference-generator heads, the rest the bench's device draw.  Ten units
    (both generators, first / middle / last of the batch) are replayed to
    convergence by the oracle."""
    import torch

    import bench
    dev = gpu_ctx.device
    U, L, kvh = 256, 32768, 8
    K = torch.empty((U, L, D), dtype=torch.int16, device=dev)
    V = torch.empty_like(K)
    g, centers = bench.gen_inputs(torch, dev, U, 4, L, 0, seed=7)
    bench.fill_kv(torch, dev, g, centers, K, V, L)
    del V
    ref_heads = {u: head(7, u // kvh, u % kvh, L, T=4)["K"] for u in (0, 1)}
    for u, k in ref_heads.items():
        K[u].copy_(torch.from_numpy(bf16_bits(k).view(np.int16)).to(dev))
    P = port()
    seeds = [P.mix_seed(0, u // kvh, u % kvh) for u in range(U)]
    c0, cents, labels, ncl, info, reps = _prefill(gpu_ctx, K, L, seeds)
    assert c0 == 409
    iters = [info[u].iterations_used for u in range(U)]
    assert min(iters) >= 2 and all(info[u].converged for u in range(U))
    for u in (0, 1, 2, 31, 64, 97, 128, 160, 203, 255):
        Kf = ref_heads[u] if u in ref_heads else _f32(K[u])
        _check_unit(u, Kf, seeds[u], c0, cents, labels, ncl, info, reps)


@pytest.mark.parametrize("retention", [1, 2])
def test_session_decode_fast_path_32k(gpu_ctx, retention):
    """Config B decode: a Session of one layer (8 kv units, G = 4 -> 32 q
    heads) at 32k, B = 1024, through the session step the bench times
    (k_select_fused + k_attend, cluster-major store), 8 steps with the
    recency window growing; every q head's I_T, the cache counters and the
    output against select_tokens + ClusterCache + approx_attention over the
    oracle's own prefill model."""
    import torch

    import bench
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200.session import Session
    dev = gpu_ctx.device
    U, G, L, T, B, kvh = 8, 4, 32768, 8, 1024, 8
    s = Session(U, G, L, T, B, retention=retention, cfg=api.ClusterConfig(), kv_heads=kvh,
                flags=N.CKV_SESSION_TOKEN_IDS)
    g, centers = bench.gen_inputs(torch, dev, U, G, L, T, seed=11)
    bench.fill_kv(torch, dev, g, centers, s.K, s.V, L)
    q_all, kn_all, vn_all = bench.gen_decode(torch, dev, g, centers, G, T)
    torch.cuda.synchronize()
    Kf = [_f32(s.K[u, :L]) for u in range(U)]
    Vf = [_f32(s.V[u, :L]) for u in range(U)]
    info = s.prefill()
    P = port()
    models = []
    st = s.state()
    for u in range(U):
        o = P.cluster_prefill(Kf[u], OCfg(seed=P.mix_seed(0, 0, u)))
        assert info[u] == (o.iterations_used, o.converged), u
        assert np.array_equal(st["labels"][u, :L].cpu().numpy(), o.labels), u
        models.append(o)
    caches = [P.cache(retention) for _ in range(U * G)]
    n_ctx = L
    for t in range(T):
        q = q_all[t].cpu().numpy()
        out = s.step(q_all[t], kn_all[t], vn_all[t]).cpu().numpy()
        st = s.state()
        tok = st["token_ids"].cpu().numpy().view(np.uint32)
        ntok = st["n_tokens"].cpu().numpy()
        rec = np.arange(L, n_ctx, dtype=np.uint32)
        for u in range(U):
            o = models[u]
            sizes, _, _ = P.build_index(o.labels, o.n_clusters)
            for r in range(G):
                hq = u * G + r
                sel = P.select_tokens(q[hq], o.centroids, o.labels, 16, B, rec)
                assert np.array_equal(tok[hq, : ntok[hq]], sel.token_ids), (t, u, r)
                caches[hq].lookup_and_update(np.sort(sel.taken_clusters), sizes)
                oo, _ = P.approx_attention(q[hq], Kf[u], Vf[u], sel.token_ids)
                assert np.abs(out[hq] - oo).max() <= 2e-5 * np.abs(Vf[u]).max(), (t, u, r)
        kn, vn = _f32(kn_all[t]), _f32(vn_all[t])
        for u in range(U):
            Kf[u] = np.concatenate([Kf[u], kn[u:u + 1]])
            Vf[u] = np.concatenate([Vf[u], vn[u:u + 1]])
        n_ctx += 1
    gc = s.cache_counters()
    for hq in range(U * G):
        assert np.array_equal(gc[hq], caches[hq].counters()), hq


def test_prefill_128k_config_e_shape(gpu_ctx):
    """Config E prefill shape: N = 131056, C0 = 1638 (> 512: multi-range
    tensor-core assignment + k_assign_merge + fix-up), capped at 3
    iterations (4 assignment passes), two units in one call (a reference-
    generator head and a device-drawn one), both against the oracle."""
    import torch

    import bench
    dev = gpu_ctx.device
    L = 131072
    K = torch.empty((2, L, D), dtype=torch.int16, device=dev)
    V = torch.empty_like(K)
    g, centers = bench.gen_inputs(torch, dev, 2, 8, L, 0, seed=5)
    bench.fill_kv(torch, dev, g, centers, K, V, L)
    del V
    h0 = head(7, 0, 0, L, T=4)["K"]
    K[0].copy_(torch.from_numpy(bf16_bits(h0).view(np.int16)).to(dev))
    P = port()
    seeds = [P.mix_seed(0, 0, 0), P.mix_seed(0, 0, 1)]
    c0, cents, labels, ncl, info, reps = _prefill(gpu_ctx, K, L, seeds, max_iters=3)
    assert c0 == 1638
    for u, Kf in ((0, h0), (1, _f32(K[1]))):
        assert info[u].iterations_used == 3 and not info[u].converged
        _check_unit(u, Kf, seeds[u], c0, cents, labels, ncl, info, reps, max_iters=3)


def test_sharded_select_config_e_shape(gpu_ctx):
    """Config E decode shape on the sequence-sharded path at world 1 (what
    bench --config E runs per rank): sharded k-means of a 128k head (3
    iterations, C0 = 1638), then ShardedDecoder steps at B = 2048, G = 8
    through the default approximate scorer (k_score_range_f32 ->
    k_select_approx: radix cut on f32 scores with rigorous bounds, exact f64
    re-scoring near the cut).  n_taken, trim and the whole I_T bit-exact
    against select_tokens on the oracle's model; output within tolerance."""
    import torch

    from paper_2412_03213_b200.sharded import DeviceShard, ShardedDecoder, kmeans_cosine_sharded
    dev = gpu_ctx.device
    L, G, B, n_rec = 131072, 8, 2048, 7
    N_ = L - 16
    h = head(7, 0, 3, L, T=64)
    P = port()
    seed = P.mix_seed(0, 0, 3)
    o = P.cluster_prefill(h["K"], OCfg(seed=seed, max_iters=3))
    Kst = np.concatenate([h["K"], h["dK"][:n_rec]])[None]
    Vst = np.concatenate([h["V"], h["dV"][:n_rec]])[None]
    tK = torch.from_numpy(bf16_bits(Kst).view(np.int16)).to(dev).contiguous()
    tV = torch.from_numpy(bf16_bits(Vst).view(np.int16)).to(dev).contiguous()
    shard = DeviceShard(tK[:, 16:16 + N_], o.n_clusters, ctx=gpu_ctx)
    km = kmeans_cosine_sharded(shard, N_, 0, seeds=[seed], max_iters=3)
    del shard
    assert int(km.iterations_used[0]) == 3
    assert np.array_equal(km.labels[0].cpu().numpy(), o.labels[16:])
    assert np.array_equal(km.centroids[0].cpu().numpy().view(np.uint32),
                          o.centroids.view(np.uint32))
    dec = ShardedDecoder(km, tK, tV, G, B, sink_rows=16, n_rec=n_rec, rec_pos=L, ctx=gpu_ctx)
    Kall, Vall = Kst[0], Vst[0]
    rec = np.arange(L, L + n_rec, dtype=np.uint32)
    for t in (0, 9, 31):
        Q = np.stack([h["Q"][(t + r * 8) % 64] for r in range(G)])
        r = dec.step(torch.from_numpy(Q).to(dev), want_ids=True)
        ids = r["token_ids"].cpu().numpy().view(np.uint32)
        nt = r["n_tokens"].cpu().numpy()
        out = r["out"].cpu().numpy()
        for hq in range(G):
            sel = P.select_tokens(Q[hq], o.centroids, o.labels, 16, B, rec)
            assert int(r["n_taken"][hq]) == sel.n_clusters_taken, (t, hq)
            assert int(r["trimmed"][hq]) == sel.trimmed_from_last, (t, hq)
            # world 1: the rank's share is the whole I_T in the reference order
            assert np.array_equal(ids[hq, : nt[hq]], sel.token_ids), (t, hq)
            oo, _ = P.approx_attention(Q[hq], Kall, Vall, sel.token_ids)
            assert np.abs(out[hq] - oo).max() <= 2e-5 * np.abs(Vall).max(), (t, hq)
