"""End-to-end decode-loop parity: the device session (prefill clustering,
per-step select + cache + attention, append, decode-batch clustering every m
steps) against the oracle replaying simulate_head's ClusterKV branch
(harness.hpp:193-339) for every (unit, q head)."""
import numpy as np
import pytest

from oracle.oracle import ClusterConfig as OCfg
from tests._inputs import bf16_bits, head, port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("f16_scores", [False, True])
def test_session_vs_oracle_decode_loop(gpu_ctx, monkeypatch, f16_scores):
    """f16_scores: the opt-in fp16 centroid copy for the approximate scores
    (CKV_SESSION_F16_SCORES; the copy is refreshed after the prefill and after
    each committed decode batch) must select exactly the same tokens."""
    import torch
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200.session import Session
    if f16_scores:
        monkeypatch.setenv("CKV_SESSION_F16_SCORES", "1")

    layers, kvh, G = 2, 2, 2
    L, T, B, m, R = 700, 45, 96, 20, 2
    U = layers * kvh
    heads = [head(7, u // kvh, u % kvh, L, T) for u in range(U)]
    cfg = api.ClusterConfig(decode_batch=m, c0_divisor=40)
    from paper_2412_03213_b200 import _native as N
    s = Session(U, G, L, T, B, retention=R, cfg=cfg, kv_heads=kvh, flags=N.CKV_SESSION_TOKEN_IDS)
    s.load_prompt_host(np.stack([bf16_bits(h["K"]) for h in heads]),
                       np.stack([bf16_bits(h["V"]) for h in heads]))
    s.prefill()

    # oracle state per unit
    P = port()
    models = []
    for u in range(U):
        o = P.cluster_prefill(heads[u]["K"], OCfg(seed=P.mix_seed(0, u // kvh, u % kvh),
                                                  decode_batch=m, c0_divisor=40))
        models.append([o.centroids, o.labels])
    caches = [P.cache(R) for _ in range(U * G)]
    Kc = [h["K"].copy() for h in heads]
    Vc = [h["V"].copy() for h in heads]
    labeled_end, n_ctx = L, L
    dev = gpu_ctx.device
    for t in range(T):
        # q head (u, r) queries row (t + r*T//G) % T of its unit's trace
        q = np.stack([heads[u]["Q"][(t + r * (T // G)) % T] for u in range(U) for r in range(G)])
        kn = np.stack([bf16_bits(heads[u]["dK"][t]) for u in range(U)])
        vn = np.stack([bf16_bits(heads[u]["dV"][t]) for u in range(U)])
        out = s.step(torch.from_numpy(q).to(dev), torch.from_numpy(kn.view(np.int16)).to(dev),
                     torch.from_numpy(vn.view(np.int16)).to(dev))
        st = s.state()
        tok = st["token_ids"].cpu().numpy().view(np.uint32)
        ntok = st["n_tokens"].cpu().numpy()
        go = out.cpu().numpy()
        rec = np.arange(labeled_end, n_ctx, dtype=np.uint32)
        for u in range(U):
            cents, labels = models[u]
            for r in range(G):
                hq = u * G + r
                sel = P.select_tokens(q[hq], cents, labels, 16, B, rec)
                assert np.array_equal(tok[hq, : ntok[hq]], sel.token_ids), (t, u, r)
                sizes, _, _ = P.build_index(labels, cents.shape[0])
                caches[hq].lookup_and_update(np.sort(sel.taken_clusters), sizes)
                oo, _ = P.approx_attention(q[hq], Kc[u][:n_ctx], Vc[u][:n_ctx], sel.token_ids)
                assert np.abs(go[hq] - oo).max() <= 2e-5 * np.abs(Vc[u][:n_ctx]).max()
        # append + decode-batch clustering (harness.hpp:318-337)
        for u in range(U):
            Kc[u] = np.concatenate([Kc[u], heads[u]["dK"][t:t + 1]])
            Vc[u] = np.concatenate([Vc[u], heads[u]["dV"][t:t + 1]])
        n_ctx += 1
        if n_ctx - labeled_end == m:
            for u in range(U):
                cents, labels = models[u]
                seed = P.mix_seed(0, u // kvh, u % kvh)
                c2, l2, _ = P.cluster_decode_batch(cents, labels, Kc[u][labeled_end:n_ctx],
                                                   OCfg(seed=seed, decode_batch=m))
                models[u] = [c2, l2]
            labeled_end = n_ctx
    # device model after the decode clustering events equals the oracle's
    st = s.state()
    for u in range(U):
        cents, labels = models[u]
        nc = int(st["n_clusters"][u].item())
        assert nc == cents.shape[0]
        assert np.array_equal(st["centroids"][u, :nc].cpu().numpy().view(np.uint32),
                              cents.view(np.uint32))
        assert np.array_equal(st["labels"][u, :labeled_end].cpu().numpy(), labels)
    ctr = s.cache_counters()
    for hq in range(U * G):
        assert [int(x) for x in ctr[hq]] == [int(x) for x in caches[hq].counters()]


def test_session_host_buffer_paths_match_device(gpu_ctx):
    """The host-buffer step (pinned: zero-copy kernels reading q / k / v and
    writing out over PCIe; pageable: staged copies) gives exactly the
    device-buffer step's outputs, step after step (decode batches included)."""
    import torch
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200.session import Session

    U, G, L, T, B = 4, 2, 600, 30, 64
    heads = [head(9, u, 0, L, T) for u in range(U)]
    cfg = api.ClusterConfig(decode_batch=12, c0_divisor=40)
    Kb = np.stack([bf16_bits(h["K"]) for h in heads])
    Vb = np.stack([bf16_bits(h["V"]) for h in heads])
    ss = []
    for _ in range(3):
        s = Session(U, G, L, T, B, retention=2, cfg=cfg, kv_heads=U)
        s.load_prompt_host(Kb, Vb)
        s.prefill()
        ss.append(s)
    dev = gpu_ctx.device
    qp = torch.empty((U * G, 128), dtype=torch.float32).pin_memory()
    kp = torch.empty((U, 128), dtype=torch.int16).pin_memory()
    vp = torch.empty((U, 128), dtype=torch.int16).pin_memory()
    op = torch.empty((U * G, 128), dtype=torch.float32).pin_memory()
    for t in range(T):
        q = np.stack([heads[u]["Q"][(t + r) % T] for u in range(U) for r in range(G)])
        kn = np.stack([bf16_bits(heads[u]["dK"][t]) for u in range(U)]).view(np.int16)
        vn = np.stack([bf16_bits(heads[u]["dV"][t]) for u in range(U)]).view(np.int16)
        o_dev = ss[0].step(torch.from_numpy(q).to(dev), torch.from_numpy(kn).to(dev),
                           torch.from_numpy(vn).to(dev)).cpu().numpy()
        qp.copy_(torch.from_numpy(q)); kp.copy_(torch.from_numpy(kn)); vp.copy_(torch.from_numpy(vn))
        N.check(N.lib().ckv_session_step(ss[1].h, qp.data_ptr(), kp.data_ptr(), vp.data_ptr(),
                                         op.data_ptr(), 0))
        o_pin = op.numpy().copy()
        o_page = np.zeros_like(o_pin)
        qq, kk, vv = q.copy(), kn.copy(), vn.copy()
        N.check(N.lib().ckv_session_step(ss[2].h, qq.ctypes.data, kk.ctypes.data, vv.ctypes.data,
                                         o_page.ctypes.data, 0))
        assert np.array_equal(o_pin, o_dev), t
        assert np.array_equal(o_page, o_dev), t


@pytest.mark.parametrize("delay", [1, 5])
def test_session_async_clustering_vs_oracle(gpu_ctx, delay):
    """The harness's async_clustering (harness.hpp:236-243, 327-329): a
    decode batch formed at step t is clustered on a side stream and joins
    the model at the start of step t + delay; until then its rows stay in
    the recency window.  I_T, outputs, the cache counters and the final model
    against the oracle replaying that schedule."""
    import torch
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200.session import Session

    U, G, L, T, B, m, R = 3, 2, 640, 75, 96, 20, 2
    heads = [head(13, u, 0, L, T) for u in range(U)]
    cfg = api.ClusterConfig(decode_batch=m, c0_divisor=40)
    s = Session(U, G, L, T, B, retention=R, cfg=cfg, kv_heads=U,
                flags=N.CKV_SESSION_TOKEN_IDS, async_delay=delay)
    s.load_prompt_host(np.stack([bf16_bits(h["K"]) for h in heads]),
                       np.stack([bf16_bits(h["V"]) for h in heads]))
    s.prefill()
    P = port()
    seeds = [P.mix_seed(0, 0, u) for u in range(U)]  # unit u = (layer 0, kv head u)
    models = []
    for u in range(U):
        o = P.cluster_prefill(heads[u]["K"], OCfg(seed=seeds[u], decode_batch=m, c0_divisor=40))
        models.append([o.centroids, o.labels])
    caches = [P.cache(R) for _ in range(U * G)]
    Kc = [h["K"].copy() for h in heads]
    Vc = [h["V"].copy() for h in heads]
    labeled_end, n_ctx, pending, queue = L, L, 0, []
    dev = gpu_ctx.device
    for t in range(T):
        while queue and queue[0][0] <= t:  # harness.hpp:237-243
            _, lo, hi = queue.pop(0)
            for u in range(U):
                c2, l2, _ = P.cluster_decode_batch(models[u][0], models[u][1], Kc[u][lo:hi],
                                                   OCfg(seed=seeds[u], decode_batch=m))
                models[u] = [c2, l2]
            labeled_end = hi
        q = np.stack([heads[u]["Q"][(t + r * (T // G)) % T] for u in range(U) for r in range(G)])
        kn = np.stack([bf16_bits(heads[u]["dK"][t]) for u in range(U)])
        vn = np.stack([bf16_bits(heads[u]["dV"][t]) for u in range(U)])
        out = s.step(torch.from_numpy(q).to(dev), torch.from_numpy(kn.view(np.int16)).to(dev),
                     torch.from_numpy(vn.view(np.int16)).to(dev))
        st = s.state()
        tok = st["token_ids"].cpu().numpy().view(np.uint32)
        ntok = st["n_tokens"].cpu().numpy()
        go = out.cpu().numpy()
        rec = np.arange(labeled_end, n_ctx, dtype=np.uint32)
        for u in range(U):
            cents, labels = models[u]
            sizes, _, _ = P.build_index(labels, cents.shape[0])
            for r in range(G):
                hq = u * G + r
                sel = P.select_tokens(q[hq], cents, labels, 16, B, rec)
                assert np.array_equal(tok[hq, : ntok[hq]], sel.token_ids), (t, u, r)
                caches[hq].lookup_and_update(np.sort(sel.taken_clusters), sizes)
                oo, _ = P.approx_attention(q[hq], Kc[u][:n_ctx], Vc[u][:n_ctx], sel.token_ids)
                assert np.abs(go[hq] - oo).max() <= 2e-5 * np.abs(Vc[u][:n_ctx]).max()
        for u in range(U):
            Kc[u] = np.concatenate([Kc[u], heads[u]["dK"][t:t + 1]])
            Vc[u] = np.concatenate([Vc[u], heads[u]["dV"][t:t + 1]])
        n_ctx += 1
        pending += 1
        if pending == m:  # harness.hpp:327-329
            queue.append((t + delay, n_ctx - m, n_ctx))
            pending = 0
    s.stats()  # blocking status check of the last batch
    st = s.state()
    for u in range(U):
        cents, labels = models[u]
        nc = int(st["n_clusters"][u].item())
        assert nc == cents.shape[0]
        assert np.array_equal(st["centroids"][u, :nc].cpu().numpy().view(np.uint32),
                              cents.view(np.uint32))
        assert np.array_equal(st["labels"][u, :labeled_end].cpu().numpy(), labels)
    ctr = s.cache_counters()
    for hq in range(U * G):
        assert [int(x) for x in ctr[hq]] == [int(x) for x in caches[hq].counters()]


def test_session_async_rejects_bad_delay(gpu_ctx):
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200.session import Session
    with pytest.raises(ValueError, match="async"):
        Session(2, 2, 300, 40, 64, cfg=api.ClusterConfig(decode_batch=20, c0_divisor=40),
                kv_heads=2, async_delay=20)


def test_session_layer_mode_matches_batched(gpu_ctx):
    """ckv_session_set_layer_units: one (select, attend) pair per layer slice
    gives the same outputs, token ids and cache counters as the all-units
    launch pair, bit for bit, across a decode-batch event."""
    import torch
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200.session import Session

    layers, kvh, G, L, T, B = 3, 2, 2, 500, 30, 80
    U = layers * kvh
    heads = [head(21, u // kvh, u % kvh, L, T) for u in range(U)]
    cfg = api.ClusterConfig(decode_batch=12, c0_divisor=40)
    ss = []
    for lu in (0, kvh):
        s = Session(U, G, L, T, B, retention=2, cfg=cfg, kv_heads=kvh,
                    flags=N.CKV_SESSION_TOKEN_IDS)
        s.load_prompt_host(np.stack([bf16_bits(h["K"]) for h in heads]),
                           np.stack([bf16_bits(h["V"]) for h in heads]))
        s.prefill()
        s.set_layer_units(lu)
        ss.append(s)
    dev = gpu_ctx.device
    for t in range(T):
        q = np.stack([heads[u]["Q"][(t + r) % T] for u in range(U) for r in range(G)])
        kn = torch.from_numpy(np.stack([bf16_bits(heads[u]["dK"][t]) for u in range(U)]).view(np.int16)).to(dev)
        vn = torch.from_numpy(np.stack([bf16_bits(heads[u]["dV"][t]) for u in range(U)]).view(np.int16)).to(dev)
        qd = torch.from_numpy(q).to(dev)
        o = [s.step(qd, kn, vn).cpu().numpy() for s in ss]
        assert np.array_equal(o[0], o[1]), t
        st = [s.state() for s in ss]
        assert torch.equal(st[0]["n_tokens"], st[1]["n_tokens"])
        nt = st[0]["n_tokens"].cpu().numpy()
        a, b = st[0]["token_ids"].cpu().numpy(), st[1]["token_ids"].cpu().numpy()
        for hq in range(U * G):
            assert np.array_equal(a[hq, :nt[hq]], b[hq, :nt[hq]]), (t, hq)
    assert np.array_equal(ss[0].cache_counters(), ss[1].cache_counters())
    with pytest.raises(ValueError):
        ss[0].set_layer_units(4)  # does not divide 6


@pytest.mark.parametrize("layer_mode", [False, True])
def test_session_attend_only_interleaved_with_steps(gpu_ctx, layer_mode):
    """ckv_session_attend_only between steps (no append: it advances the
    selection -> attention hand-off epoch itself): its output equals the next
    step's for the same q, bit for bit, in both launch modes."""
    import torch
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200.session import Session

    layers, kvh, G, L, T, B = 2, 2, 2, 600, 16, 90
    U = layers * kvh
    heads = [head(33, u // kvh, u % kvh, L, T) for u in range(U)]
    s = Session(U, G, L, T, B, retention=1,
                cfg=api.ClusterConfig(decode_batch=7, c0_divisor=40), kv_heads=kvh)
    s.load_prompt_host(np.stack([bf16_bits(h["K"]) for h in heads]),
                       np.stack([bf16_bits(h["V"]) for h in heads]))
    s.prefill()
    if layer_mode:
        s.set_layer_units(kvh)
    dev = gpu_ctx.device
    for t in range(T):
        q = np.stack([heads[u]["Q"][(t + r) % T] for u in range(U) for r in range(G)])
        qd = torch.from_numpy(q).to(dev)
        kn = torch.from_numpy(np.stack([bf16_bits(heads[u]["dK"][t]) for u in range(U)]).view(np.int16)).to(dev)
        vn = torch.from_numpy(np.stack([bf16_bits(heads[u]["dV"][t]) for u in range(U)]).view(np.int16)).to(dev)
        a = torch.empty((U * G, 128), dtype=torch.float32, device=dev)
        s.attend_only(qd, a)
        if t % 3 == 0:  # two attend-only calls in a row
            s.attend_only(qd, a)
        b = s.step(qd, kn, vn)
        assert torch.equal(a, b), t


def test_session_fused_and_split_select_paths(gpu_ctx):
    """A session of 80 units selects with the fused kernel (one CTA per unit:
    scoring + selection, k_select_fused); its layer mode (8-unit slices)
    selects with the split kernels (k_score_approx over many CTAs per unit,
    then k_select_warp).  Both against select_tokens on the oracle's models."""
    import torch
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200.session import Session

    layers, kvh, G, L, T, B = 10, 8, 2, 400, 4, 64
    U = layers * kvh
    heads = [head(31, u // kvh, u % kvh, L, T) for u in range(U)]
    cfg = api.ClusterConfig(decode_batch=50, c0_divisor=40)
    s = Session(U, G, L, T, B, retention=1, cfg=cfg, kv_heads=kvh, flags=N.CKV_SESSION_TOKEN_IDS)
    s.load_prompt_host(np.stack([bf16_bits(h["K"]) for h in heads]),
                       np.stack([bf16_bits(h["V"]) for h in heads]))
    s.prefill()
    P = port()
    models = [P.cluster_prefill(heads[u]["K"], OCfg(seed=P.mix_seed(0, u // kvh, u % kvh),
                                                     c0_divisor=40)) for u in range(U)]
    Kc = [h["K"].copy() for h in heads]
    dev = gpu_ctx.device
    for t in range(T):
        s.set_layer_units(kvh if t % 2 else 0)
        q = np.stack([heads[u]["Q"][(t + 3 * r) % T] for u in range(U) for r in range(G)])
        kn = np.stack([bf16_bits(heads[u]["dK"][t]) for u in range(U)]).view(np.int16)
        vn = np.stack([bf16_bits(heads[u]["dV"][t]) for u in range(U)]).view(np.int16)
        s.step(torch.from_numpy(q).to(dev), torch.from_numpy(kn).to(dev),
               torch.from_numpy(vn).to(dev))
        st = s.state()
        tok = st["token_ids"].cpu().numpy().view(np.uint32)
        ntok = st["n_tokens"].cpu().numpy()
        rec = np.arange(L, L + t, dtype=np.uint32)
        for u in range(U):
            for r in range(G):
                hq = u * G + r
                sel = P.select_tokens(q[hq], models[u].centroids, models[u].labels, 16, B, rec)
                assert np.array_equal(tok[hq, : ntok[hq]], sel.token_ids), (t, u, r)


@pytest.mark.parametrize("flag,R,layer_mode", [("TIERED", 1, False), ("TIER_HOST", 2, False),
                                               ("TIERED", 2, True)])
def test_session_two_tier_cache_matches_flat(gpu_ctx, flag, R, layer_mode):
    """The physical two-tier cache (ckv_tier.cu): misses copied from the
    backing tier (HBM store or the host-pinned mirror) into the page pool,
    attention over page runs — outputs, I_T and the reference cache
    counters equal the flat session's bit for bit, across decode batches; the
    physical counters are consistent (fetched <= selected, bytes = rows x 512)."""
    import torch
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200.session import Session

    layers, kvh, G, L, T, B = 2, 3, 2, 700, 45, 96
    U = layers * kvh
    heads = [head(41, u // kvh, u % kvh, L, T) for u in range(U)]
    cfg = api.ClusterConfig(decode_batch=15, c0_divisor=40)
    ss = []
    for extra in (0, getattr(N, f"CKV_SESSION_{flag}")):
        s = Session(U, G, L, T, B, retention=R, cfg=cfg, kv_heads=kvh,
                    flags=N.CKV_SESSION_TOKEN_IDS | extra)
        s.load_prompt_host(np.stack([bf16_bits(h["K"]) for h in heads]),
                           np.stack([bf16_bits(h["V"]) for h in heads]))
        s.prefill()
        if layer_mode:
            s.set_layer_units(kvh)
        ss.append(s)
    dev = gpu_ctx.device
    for t in range(T):
        q = torch.from_numpy(np.stack([heads[u]["Q"][(t + 5 * r) % T] for u in range(U)
                                       for r in range(G)])).to(dev)
        kn = torch.from_numpy(np.stack([bf16_bits(heads[u]["dK"][t]) for u in range(U)]).view(np.int16)).to(dev)
        vn = torch.from_numpy(np.stack([bf16_bits(heads[u]["dV"][t]) for u in range(U)]).view(np.int16)).to(dev)
        o = [s.step(q, kn, vn).cpu().numpy() for s in ss]
        assert np.array_equal(o[0], o[1]), t
        st = [s.state() for s in ss]
        assert torch.equal(st[0]["n_tokens"], st[1]["n_tokens"])
    assert np.array_equal(ss[0].cache_counters(), ss[1].cache_counters())
    ts = ss[1].tier_stats()
    assert 0 < ts["clusters_fetched"] <= ts["clusters_selected"]
    assert ts["rows_fetched"] > 0 and ts["bytes_fetched"] == ts["rows_fetched"] * 512
