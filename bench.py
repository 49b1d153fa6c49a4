#!/usr/bin/env python
"""ClusterKV hot-path benchmark on B200 (BASELINE.json configs[1] = config B).

Workload (config B): Llama-3-8B attention shape — 32 layers x 8 kv heads
(256 units), 4 q heads per kv head (1024 q heads), d = 128, 32k prompt,
batch 1, budget B = 1024, R = 1 cluster cache.  Per run:
  prefill : cluster_prefill (cosine k-means, C0 = 409) + build_index for all
            256 units — timed, reported as `prefill`.
  decode  : W warm-up + K timed decode steps through the device session:
            select (+cache) -> sparse attention -> append, every unit, every
            layer, one step = one generated token.  `value` = tokens/s.
  e2e     : the same step through ckv_session_step with HOST q/k/v/out
            buffers (H2D + D2H inside the timed region).
Inputs: synthetic, drawn on device with the reference generator's
distributions (trace.hpp:134-198: unit keys around 8 directional centres,
N(0,1) values, 2*sqrt(d)-scaled drifting queries), rounded to bf16.
The per-step working set (~600 MB) is far above L2 (126 MB): no L2 flush.

Layers are independent units inside one decode step (as in the reference's
run_simulation fan-out, harness.hpp:362-378), so one step issues one select
and one attention launch covering all 32 layers.

--impl reference: the reference's own CPU implementation
(oracle/_ref/libckv_ref.so = /root/reference headers compiled unmodified),
select_tokens + approx_attention on all host threads, same config.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
D = 128


def peaks():
    try:
        p = json.load(open(PEAKS_PATH))
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# --------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md)
# --------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def soak_for(torch, fn, seconds: float) -> None:
    """Keeps the GPU busy for `seconds` (untimed) so the clock sampler sees
    loaded clocks before a short timed region starts."""
    t_end = time.time() + seconds
    while time.time() < t_end:
        for _ in range(10):
            fn()
        torch.cuda.synchronize()


# --------------------------------------------------------------------------
# synthetic inputs on device (distributions of trace.hpp:134-198)
# --------------------------------------------------------------------------
def gen_inputs(torch, dev, U, G, L, T, seed=7, n_centers=8):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    nrm = lambda x: x / x.norm(dim=-1, keepdim=True)
    base = nrm(torch.randn(U, 1, D, device=dev, generator=g))
    centers = nrm(base + 1.0 * torch.randn(U, n_centers, D, device=dev, generator=g))
    return g, centers


def fill_kv(torch, dev, g, centers, K, V, L, chunk=16):
    U = K.shape[0]
    for u0 in range(0, U, chunk):
        u1 = min(U, u0 + chunk)
        idx = torch.randint(0, centers.shape[1], (u1 - u0, L), device=dev, generator=g)
        c = torch.gather(centers[u0:u1], 1, idx[..., None].expand(-1, -1, D))
        k = c + 0.15 * torch.randn(u1 - u0, L, D, device=dev, generator=g)
        k = k / k.norm(dim=-1, keepdim=True)
        K[u0:u1, :L].copy_(k.to(torch.bfloat16).view(torch.int16))
        V[u0:u1, :L].copy_(torch.randn(u1 - u0, L, D, device=dev, generator=g)
                           .to(torch.bfloat16).view(torch.int16))


def gen_decode(torch, dev, g, centers, G, T, drift=0.15, T_gen=256):
    """queries [T, U*G, D] f32 (bf16-representable), new k/v [T, U, D] bf16 bits.

    One drifting query walk of T_gen = 256 steps per kv unit (the trace's
    decode_len); q head r of a group reads walk row (t + r*T_gen/G) % T_gen,
    the GQA mapping of SURVEY §8d."""
    U, NC, _ = centers.shape
    q_scale = 2.0 * math.sqrt(D)
    ar = torch.arange(U, device=dev)
    u = centers[ar, torch.randint(0, NC, (U,), device=dev, generator=g)]
    retarget = max(1, T_gen // (2 * NC))
    walk = []
    tgt = None
    for t in range(T_gen):
        if t % retarget == 0:
            tgt = centers[ar, torch.randint(0, NC, (U,), device=dev, generator=g)]
        u = u + drift * (tgt - u) + 0.25 * drift * torch.randn(U, D, device=dev, generator=g)
        u = u / u.norm(dim=-1, keepdim=True)
        walk.append(q_scale * u)
    walk = torch.stack(walk)  # [T_gen, U, D]
    rows = (torch.arange(T, device=dev)[:, None] + torch.arange(G, device=dev)[None, :] *
            (T_gen // G)) % T_gen  # [T, G]
    q = walk[rows]  # [T, G, U, D]
    q = q.permute(0, 2, 1, 3).reshape(T, U * G, D)
    q = q.to(torch.bfloat16).float().contiguous()
    idx = torch.randint(0, NC, (T, U), device=dev, generator=g)
    c = centers[ar[None, :].expand(T, U), idx]
    kn = c + 0.15 * torch.randn(T, U, D, device=dev, generator=g)
    kn = (kn / kn.norm(dim=-1, keepdim=True)).to(torch.bfloat16).view(torch.int16).contiguous()
    vn = torch.randn(T, U, D, device=dev, generator=g).to(torch.bfloat16).view(torch.int16)
    return q, kn, vn.contiguous()


# --------------------------------------------------------------------------
# CPU legs: the reference compiled unmodified (oracle/_ref), else the port
# --------------------------------------------------------------------------
def cpu_reference_decode(layer_sample, n_threads, G, L, B, sink=16):
    """One full 32-layer decode step on the host = 32 x select_tokens +
    approx_attention over one layer's 8 kv heads (bounded sample: that
    layer's data is reused for every layer).  Returns ms per step."""
    from oracle.oracle import Oracle
    R = Oracle("reference")
    cents, ncl, labels, K, V, qs = layer_sample
    n_kv = len(cents)
    units = n_kv * G
    keep = [cents, labels, K, V]  # keep buffers alive
    ptr = lambda arrs: (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    kv_of = np.repeat(np.arange(n_kv, dtype=np.uint32), G)
    out = np.zeros((units, D), np.float32)
    ms = R.lib.ref_decode_step_cpu(qs, kv_of, units, ptr(cents), ncl, ptr(labels), ptr(K), ptr(V),
                                   n_kv, L, L, D, B, sink, n_threads, out)
    del keep
    return ms


def layer_sample_from_device(torch, sess, U_layer, G, L, q0):
    st = sess.state()
    bf = lambda t: (t.to(torch.int32) << 16).view(torch.float32)
    cents, ncl, labels, K, V = [], [], [], [], []
    for u in range(U_layer):
        n = int(st["n_clusters"][u].item())
        cents.append(np.ascontiguousarray(st["centroids"][u, :n].cpu().numpy()))
        ncl.append(n)
        labels.append(np.ascontiguousarray(st["labels"][u, :L].cpu().numpy()))
        # the store is cluster-major after prefill: scatter back to positions
        srt = st["sorted_ids"][u, : L - 16].to(torch.int64)
        for store, dst in ((sess.K, K), (sess.V, V)):
            pos = torch.empty((L, D), dtype=torch.int16, device=store.device)
            pos[:16] = store[u, :16]
            pos[srt] = store[u, 16:L]
            dst.append(np.ascontiguousarray(bf(pos).cpu().numpy()))
    qs = np.ascontiguousarray(q0[: U_layer * G].cpu().numpy())
    return cents, np.array(ncl, np.uint32), labels, K, V, qs


def host_sample_reference(L, n_kv, G, T=256, max_iters=3):
    """Inputs for --impl reference without touching our kernels: the
    reference's own generator + its own cluster_prefill (iterations capped
    for the bounded sample; decode-step cost does not depend on them)."""
    from oracle.oracle import ClusterConfig, Oracle, to_bf16_representable
    import concurrent.futures as cf
    R = Oracle("reference")

    def one(h):
        tr = R.generate_head(R.mix_seed(7, 0, h), L, T)
        K = to_bf16_representable(tr.prompt_keys)
        m = R.cluster_prefill(K, ClusterConfig(seed=R.mix_seed(0, 0, h), max_iters=max_iters))
        q = to_bf16_representable(np.stack([tr.decode_queries[(r * (T // G)) % T] for r in range(G)]))
        return m, K, to_bf16_representable(tr.prompt_values), q

    with cf.ThreadPoolExecutor(max_workers=min(n_kv, os.cpu_count() or 1)) as ex:
        res = list(ex.map(one, range(n_kv)))
    cents = [np.ascontiguousarray(r[0].centroids) for r in res]
    ncl = np.array([r[0].n_clusters for r in res], np.uint32)
    labels = [np.ascontiguousarray(r[0].labels) for r in res]
    K = [r[1] for r in res]
    V = [r[2] for r in res]
    qs = np.ascontiguousarray(np.concatenate([r[3] for r in res]))
    return cents, ncl, labels, K, V, qs


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle.oracle import Oracle, build, ref_available
    if not ref_available():
        try:
            build(ref=True)
        except Exception:
            pass
    kind = "reference" if ref_available() else "port"
    if kind != "reference":
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libckv_ref.so not built (needs /root/reference)"}))
        return
    L, B, G, layers, n_kv = args.L, args.budget, 4, 32, 8
    cores = int(Oracle("reference").lib.ref_hardware_concurrency())
    sample = host_sample_reference(L, n_kv, G)
    for _ in range(args.warmup):
        cpu_reference_decode(sample, cores, G, L, B)
    times = []
    for _ in range(args.steps):
        t = sum(cpu_reference_decode(sample, cores, G, L, B) for _ in range(layers))
        times.append(t)
    ms = float(np.mean(times))
    tps = 1000.0 / ms
    line = {"impl": "reference", "metric": "decode tokens/s (select+gather+attend, 32k ctx, B=1024)",
            "value": tps, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
            "config": {"workload": "config B decode step: 32 layers x 8 kv x 4 q heads, 32k ctx, "
                                   "B=1024, batch 1", "global_batch": 1, "seq_len": L},
            "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": cores, "kind": kind,
                             "sample": "one layer (8 kv heads, 32 q heads, reference generator, "
                                       "reference cluster_prefill capped at 3 iterations) "
                                       "reused for all 32 layers; select_tokens + "
                                       "approx_attention per q head on std::async workers"},
            "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------------------
# secondary workloads (BASELINE.json configs[2..4]); the headline is config B
# --------------------------------------------------------------------------
def _events(torch, n):
    return [torch.cuda.Event(enable_timing=True) for _ in range(n)]


def _max_over_ranks(torch, dev, world, vals):
    """Max over ranks of per-rank device-timed values (NCCL on the device;
    host tensors under gloo, i.e. CKV_BENCH_SHARE_GPU)."""
    if world == 1:
        return list(vals)
    import torch.distributed as dist
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor(vals, device=dev if on_dev else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_world(n: int) -> None:
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run with N local ranks (one per GPU, 127.0.0.1
    rendezvous).  Fails loudly when fewer than N GPUs are visible, unless
    CKV_BENCH_SHARE_GPU=1 (test mode: every rank on cuda:0, gloo)."""
    if os.environ.get("CKV_BENCH_SHARE_GPU") != "1":
        import torch
        vis = torch.cuda.device_count()
        if vis < n:
            raise SystemExit(f"bench.py --gpus {n}: only {vis} visible GPU(s); "
                             "one rank per GPU is required")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def rank_device(local: int) -> int:
    """CUDA device of this rank: LOCAL_RANK, or 0 for every rank in the
    shared-GPU test mode."""
    return 0 if os.environ.get("CKV_BENCH_SHARE_GPU") == "1" else local


def unique_kv_rows(torch, run_row, run_off, run_cnt, group, p_cap):
    """Unique (kv unit, store row) pairs read by one attention launch, from
    the I_T run lists: the q heads of a GQA group share their unit's rows
    through L2, so unique rows (not the per-head sum) are the algorithmic
    bytes."""
    n_q, run_cap = run_row.shape
    live = torch.arange(run_cap, device=run_row.device)[None] < run_cnt.to(torch.int64)[:, None]
    lens = ((run_off[:, 1:] - run_off[:, :-1]).to(torch.int64) * live).flatten()
    total = int(lens.sum().item())
    if total == 0:
        return 0, 0
    rid = torch.repeat_interleave(torch.arange(n_q * run_cap, device=run_row.device), lens)
    first = torch.repeat_interleave(torch.cumsum(lens, 0) - lens, lens)
    rows = run_row.flatten().to(torch.int64)[rid] + (torch.arange(total, device=rid.device) - first)
    key = (rid // run_cap // group) * p_cap + rows
    return int(torch.unique(key).numel()), total


def ncu_traffic(kernel: str):
    """DRAM bytes of one launch of `kernel` from the newest committed ncu
    --set full summary (tools/profile_summary.py); None if absent."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_decode_kernels.json")))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))
        for k, v in d.items():
            if k.startswith(kernel) and v.get("dram_traffic_bytes"):
                return float(v["dram_traffic_bytes"])
    except Exception:
        return None
    return None


def run_config_D(torch, dev, ctx, args):
    """configs[3]: 32k prompt + 4096 generated tokens, decode-batch clustering
    every 320 steps (harness.hpp:325-333), cluster cache R = 1 and 2.  Every
    step goes through ckv_session_step (select + attend + append + the
    clustering event when due); per-step CUDA events split event steps from
    the rest."""
    from paper_2412_03213_b200.api import ClusterConfig
    from paper_2412_03213_b200.session import Session
    U, G, L, B, T = args.layers * args.kv_heads, args.group, args.L, args.budget, args.gen_tokens
    g, centers = gen_inputs(torch, dev, U, G, L, T, seed=11)
    q_all, kn_all, vn_all = gen_decode(torch, dev, g, centers, G, T)
    out = torch.empty((U * G, D), dtype=torch.float32, device=dev)
    res = {"workload": f"config D: {args.layers} layers x {args.kv_heads} kv x {G} q heads, "
                       f"{L} prompt + {T} generated, B={B}, decode-batch clustering every 320 steps",
           "tokens": T}
    from paper_2412_03213_b200 import _native as N
    # flat (every cluster HBM-resident), async clustering, and the physical
    # two-tier cache: backing tier in HBM (secondary store) or host-pinned
    # memory (the offload setting, misses over PCIe), R = 1 and 2
    variants = ((1, 0, 0, ""), (2, 0, 0, ""), (1, 8, 0, ""),
                (1, 0, N.CKV_SESSION_TIERED, "_tier_hbm"), (2, 0, N.CKV_SESSION_TIERED, "_tier_hbm"),
                (1, 0, N.CKV_SESSION_TIER_HOST, "_tier_host"),
                (2, 0, N.CKV_SESSION_TIER_HOST, "_tier_host"))
    flat_us = {}
    # warm-up: a small session per mode runs decode-batch events first, so the
    # timed runs do not pay one-time kernel loading / attribute setup
    gw = torch.Generator(device=dev)
    gw.manual_seed(13)
    for _, delay, tflag, _ in variants:
        ws = Session(args.kv_heads, G, 1024, 12, 64, retention=2,
                     cfg=ClusterConfig(decode_batch=4, c0_divisor=40), kv_heads=args.kv_heads,
                     ctx=ctx, async_delay=min(delay, 3), flags=tflag)
        fill_kv(torch, dev, gw, centers[: args.kv_heads], ws.K, ws.V, 1024)
        ws.prefill()
        for t in range(12):
            ws.step(q_all[t, : args.kv_heads * G], kn_all[t, : args.kv_heads],
                    vn_all[t, : args.kv_heads], out[: args.kv_heads * G])
        del ws
    torch.cuda.synchronize()
    for R, delay, tflag, tname in variants:
        sess = Session(U, G, L, T, B, retention=R, cfg=ClusterConfig(), kv_heads=args.kv_heads,
                       ctx=ctx, async_delay=delay, flags=tflag)
        gk = torch.Generator(device=dev)
        gk.manual_seed(12)
        fill_kv(torch, dev, gk, centers, sess.K, sess.V, L)
        sess.prefill()
        ev = _events(torch, T + 1)
        ev[0].record()
        for t in range(T):
            sess.step(q_all[t], kn_all[t], vn_all[t], out)
            ev[t + 1].record()
        torch.cuda.synchronize()
        ms = np.array([ev[t].elapsed_time(ev[t + 1]) for t in range(T)])
        st = sess.stats()
        m = 320
        # synchronous: the step that completes a batch clusters and commits
        # it; async (harness.hpp:236-243): that step launches the k-means on
        # the side stream, the step `delay` later commits it
        ev_steps = np.array([bool((t + 1) % m == 0 or
                                  (delay and (t + 1 - delay) % m == 0 and t >= delay))
                             for t in range(T)], dtype=bool)
        ctr = sess.cache_counters().astype(np.float64)
        key = f"R{R}" + (f"_async{delay}" if delay else "") + tname
        res[key] = {
            "hit_rate": float(ctr[:, 1].sum() / max(1.0, ctr[:, 0].sum())),
            "miss_tokens_per_q_head_step": float(ctr[:, 2].sum() / (U * G * T)),
            "step_us_mean": float(ms.mean() * 1e3),
            "step_us_plain": float(ms[~ev_steps].mean() * 1e3),
            "step_us_event": float(ms[ev_steps].mean() * 1e3) if ev_steps.any() else None,
            "clustering_events": int(ev_steps.sum()),
            "clustering_us_per_event": float((ms[ev_steps].mean() - ms[~ev_steps].mean()) * 1e3)
            if ev_steps.any() else None,
            "amortised_overhead_us_per_step": float((ms.sum() - ms[~ev_steps].mean() * T) / T * 1e3),
            "labeled_end": int(st.labeled_end), "n_ctx": int(st.n_ctx),
            "tokens_per_s": float(1000.0 / ms.mean()),
        }
        if delay:
            res[key]["async_delay"] = delay
        if not tflag and not delay:
            flat_us[R] = float(ms.mean() * 1e3)
        if tflag:
            ts = sess.tier_stats()
            extra = float(ms.mean() * 1e3) - flat_us.get(R, float("nan"))
            res[key]["tier"] = {
                "backing": "host-pinned (PCIe)" if tflag == N.CKV_SESSION_TIER_HOST else "HBM",
                "pool_rows_per_unit": ts["pool_rows_per_unit"],
                "rows_fetched_per_step": ts["rows_fetched"] / T,
                "bytes_fetched_per_step": ts["bytes_fetched"] / T,
                "physical_hit_rate": 1.0 - ts["clusters_fetched"] / max(1, ts["clusters_selected"]),
                "transfer_us_per_step": extra,
                "transfer_gbs": ts["bytes_fetched"] / T / (extra * 1e-6) / 1e9 if extra > 0 else None}
        del sess
        torch.cuda.synchronize()
    del q_all, kn_all, vn_all
    return res


def run_quality(torch, dev, ctx, args, budgets=(128, 256, 512, 1024, 2048), T=32):
    """Selection quality vs budget: the GPU port of the
    reference harness's run_simulation + sweep (paper_2412_03213_b200/
    quality.py, pinned to the compiled reference in tests/test_gpu_quality.py)
    on one layer (8 kv heads) of the bench's synthetic 32k draw, T decode
    steps each: mean recall against the exact top-B, output error against
    full attention, cluster-cache hit rate."""
    from paper_2412_03213_b200 import quality as Q
    from paper_2412_03213_b200.trace import HeadTrace, TraceBundle
    U, L = args.kv_heads, args.L
    g, centers = gen_inputs(torch, dev, U, 1, L, T, seed=21)
    K = torch.empty((U, L, D), dtype=torch.int16, device=dev)
    V = torch.empty_like(K)
    fill_kv(torch, dev, g, centers, K, V, L)
    q, kn, vn = gen_decode(torch, dev, g, centers, 1, T)  # [T, U, D]
    f32 = lambda b: ((b.to(torch.int32) & 0xffff) << 16).view(torch.float32).cpu().numpy()
    Kf, Vf, dKf, dVf = f32(K), f32(V), f32(kn.transpose(0, 1)), f32(vn.transpose(0, 1))
    Qf = q.transpose(0, 1).contiguous().cpu().numpy()
    bundle = TraceBundle(1, U, [HeadTrace(Kf[u], Vf[u], Qf[u], dKf[u], dVf[u]) for u in range(U)])
    t0 = time.perf_counter()
    reps = Q.sweep(bundle, Q.PolicyConfig(), "budget", list(budgets), ctx=ctx)
    return {"workload": f"{U} kv heads (one layer), {L} ctx, {T} decode steps per budget; "
                        "quality.run_simulation (reference harness semantics, GPU metrics)",
            "budget": list(budgets),
            "mean_recall": [r.summary.mean_recall for r in reps],
            "mean_l2_rel": [r.summary.mean_l2_rel for r in reps],
            "mean_cos_sim": [r.summary.mean_cos_sim for r in reps],
            "hit_rate": [r.summary.hit_rate for r in reps],
            "sweep_ms": (time.perf_counter() - t0) * 1e3}


def run_config_C(args, rank, world, torch, dev, ctx, hbm):
    """configs[2]: Llama-3-8B shape, 32k context, B = 2048, global batch 32,
    batch-sharded over the ranks (strong scaling: 32 / world sequences each).
    Decode steps through ckv_session_step on HBM-resident inputs."""
    from paper_2412_03213_b200.api import ClusterConfig
    from paper_2412_03213_b200.session import Session
    batch_total = 32
    if batch_total % world:
        raise SystemExit("config C needs world | 32")
    batch = batch_total // world
    G, L, B = 4, args.L, 2048
    U = batch * args.layers * args.kv_heads
    T = args.warmup + args.steps + 2
    sess = Session(U, G, L, T, B, retention=1, cfg=ClusterConfig(), kv_heads=args.kv_heads,
                   ctx=ctx)
    if args.trace:  # a CKVT file's heads instead of the synthetic draw
        from paper_2412_03213_b200 import trace as TR
        tb = TR.read_trace(args.trace)
        Kt, Vt, Qt, dKt, dVt = TR.to_device(tb, dev, decode_kv=True)
        if Kt.shape[0] != U or Kt.shape[1] != L:
            raise SystemExit(f"--trace: need {U} heads of L = {L} (pass --layers/--kv-heads/--L); "
                             f"the file has {Kt.shape[0]} heads of L = {Kt.shape[1]}")
        sess.K[:, :L].copy_(Kt)
        sess.V[:, :L].copy_(Vt)
        Tt = Qt.shape[1]
        rows = (torch.arange(T, device=dev)[:, None] + torch.arange(G, device=dev)[None, :] *
                max(1, Tt // G)) % Tt  # the GQA row offset of SURVEY §8d
        q_all = Qt[:, rows].permute(1, 0, 2, 3).reshape(T, U * G, D).contiguous()
        kn_all = dKt[:, torch.arange(T, device=dev) % Tt].permute(1, 0, 2).contiguous()
        vn_all = dVt[:, torch.arange(T, device=dev) % Tt].permute(1, 0, 2).contiguous()
        del Kt, Vt, Qt, dKt, dVt
    else:
        g, centers = gen_inputs(torch, dev, U, G, L, T, seed=7 + rank)
        fill_kv(torch, dev, g, centers, sess.K, sess.V, L)
        q_all, kn_all, vn_all = gen_decode(torch, dev, g, centers, G, T)
    torch.cuda.synchronize()
    e = _events(torch, 2)
    e[0].record()
    info = sess.prefill()
    e[1].record()
    torch.cuda.synchronize()
    prefill_ms = e[0].elapsed_time(e[1])
    out = torch.empty((U * G, D), dtype=torch.float32, device=dev)
    t = 0
    for _ in range(args.warmup):
        sess.step(q_all[t], kn_all[t], vn_all[t], out)
        t += 1
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    with ClockSampler(int(str(dev).split(":")[-1])) as clk:
        soak_out = torch.empty_like(out)
        soak_for(torch, lambda: sess.attend_only(q_all[0], soak_out), 0.4)
        e[0].record()
        for _ in range(args.steps):
            sess.step(q_all[t], kn_all[t], vn_all[t], out)
            t += 1
        e[1].record()
        torch.cuda.synchronize()
    step_ms = e[0].elapsed_time(e[1]) / args.steps
    st = sess.state()
    ntok = int(st["n_tokens"].to(torch.int64).sum().item())
    ncl = int(st["n_clusters"].to(torch.int64).sum().item())
    # the last step's selection as runs (one untimed select) -> unique rows
    from paper_2412_03213_b200 import _native as N
    n_q, c_cap, sel_cap = U * G, st["c_cap"], st["sel_cap"]
    stats = sess.stats()
    sd = N.SelectDesc(n_q, G, B, 16, sess.p_cap, c_cap, sel_cap, stats.labeled_end, stats.n_ctx,
                      0, 16)
    ptrs = [C.c_void_p() for _ in range(8)]
    cc, scap = C.c_uint32(), C.c_uint32()
    N.lib().ckv_session_state(sess.h, *[C.byref(p) for p in ptrs], C.byref(cc), C.byref(scap))
    rr = torch.zeros((n_q, c_cap + 2), dtype=torch.int32, device=dev)
    ro = torch.zeros((n_q, c_cap + 3), dtype=torch.int32, device=dev)
    rc_ = torch.zeros(n_q, dtype=torch.int32, device=dev)
    runs = N.Runs(rr.data_ptr(), ro.data_ptr(), rc_.data_ptr(), c_cap + 2)
    tmp = [torch.zeros(n_q, dtype=torch.int32, device=dev) for _ in range(3)]
    rk = torch.zeros((n_q, c_cap), dtype=torch.int32, device=dev)
    N.check(N.lib().ckv_select(ctx.h, C.byref(sd), q_all[t - 1].data_ptr(), ptrs[0], ptrs[2],
                               ptrs[3], ptrs[4], ptrs[5], None, None, C.byref(runs),
                               tmp[0].data_ptr(), tmp[1].data_ptr(), tmp[2].data_ptr(),
                               rk.data_ptr(), None, None))
    uniq, _ = unique_kv_rows(torch, rr, ro, rc_, G, sess.p_cap)
    n_runs = int(rc_.sum().item())
    step_bytes = uniq * D * 2 * 2 + ncl * D * 4 + ncl * 8 + n_runs * 8 + U * G * D * 8
    step_bytes_nodd = ntok * D * 2 * 2 + ncl * D * 4 + ncl * 8 + n_runs * 8 + U * G * D * 8
    step_ms, prefill_ms = _max_over_ranks(torch, dev, world, [step_ms, prefill_ms])
    gbs = step_bytes / (step_ms * 1e-3) / 1e9
    return {"metric": "decode tokens/s (select+gather+attend, 32k ctx, B=2048, batch 32)",
            "value": batch_total * 1000.0 / step_ms, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16 KV, f32/f64 math",
            "data": "synthetic (device draw with trace.hpp generator distributions, bf16)",
            "config": {"workload": f"config C: Llama-3-8B shape, {args.layers} layers x "
                                   f"{args.kv_heads} kv x {G} q heads, {L} ctx, B={B}, "
                                   f"batch {batch_total} ({batch} per GPU), R=1",
                       "global_batch": batch_total, "seq_len": L,
                       "parallelism": f"batch-sharded x{world}",
                       "l2": f"per-step working set ~{step_bytes / 1e9:.0f} GB >> L2"},
            "step_roofline": {"achieved_gbs": gbs, "frac": gbs / hbm,
                              "bytes_per_step": step_bytes,
                              "bytes_rule": "unique (kv unit, row) K+V rows + f32 centroids + "
                                            "sizes/starts + runs + q/out",
                              "bytes_per_step_no_dedupe": step_bytes_nodd},
            "prefill": {"ms": prefill_ms, "units": U,
                        "iters_max": max(i for i, _ in info)},
            "clocks": clk.summary()}


def run_config_E(args, rank, world, torch, dev, ctx, hbm):
    """configs[4]: Llama-3-70B shape (80 layers x 8 kv x 8 q heads), 128k
    context, B = 2048, one sequence SEQUENCE-sharded over the ranks
    (paper_2412_03213_b200/sharded.py): sharded k-means with all-reduced f64
    centroid sums, then decode steps with centroid-sharded scoring, an
    all-gather of the scores for the global top-k, local sparse attention
    and an LSE merge.  Timing: prefill = the whole sharded k-means; a step =
    ShardedDecoder.step (score + all-gather + select + attend + merge) at a
    fixed context (no append)."""
    from paper_2412_03213_b200.sharded import (Comm, DeviceShard, ShardedDecoder,
                                               kmeans_cosine_sharded, shard_range)
    layers, kvh, G, L, B = 80, 8, 8, args.L_E, 2048
    U = layers * kvh
    N = L - 16
    lo, hi = shard_range(N, world, rank)
    sink_rows = 16 if rank == 0 else 0
    rows = sink_rows + hi - lo
    comm = Comm()
    K = torch.empty((U, rows, D), dtype=torch.int16, device=dev)
    V = torch.empty_like(K)
    g, centers = gen_inputs(torch, dev, U, G, L, 0, seed=7)  # centres shared by all ranks
    g.manual_seed(100 + rank)
    fill_kv(torch, dev, g, centers, K, V, rows)
    C0 = int(N_lib().ckv_prefill_cluster_count(L, 80, 16, 0))
    seeds = [int(N_lib().ckv_mix_seed(0, u // kvh, u % kvh)) for u in range(U)]
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    # the sharded k-means through the native C++ driver (ckv_kmeans_sharded,
    # NCCL collectives; rank 0's NCCL id reaches the others over the process
    # group) — CKV_E_PY=1 runs sharded.py's torch.distributed host instead
    native = os.environ.get("CKV_E_PY") is None
    if native:
        from paper_2412_03213_b200.sharded import NativeComm, kmeans_cosine_native
        nid = [NativeComm.nccl_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(nid, src=0)
        ncomm = NativeComm(ctx, world, rank, nccl_id=nid[0])
    e = _events(torch, 2)
    # one untimed call (first-use scratch allocations of tens of GB), then the
    # median of CKV_E_PREFILL_REPS timed calls (single calls spread 2.5-3.2 s)
    reps = max(1, int(os.environ.get("CKV_E_PREFILL_REPS", "3")))
    prefill_all = []
    for r in range(reps + 1):
        if world > 1:
            dist.barrier()
        e[0].record()
        if native:
            km = kmeans_cosine_native(K[:, sink_rows:], C0, N, lo, ncomm, seeds=seeds)
        else:
            shard = DeviceShard(K[:, sink_rows:], C0, ctx=ctx)
            km = kmeans_cosine_sharded(shard, N, lo, seeds=seeds, comm=comm)
            del shard
        e[1].record()
        torch.cuda.synchronize()
        if r > 0:
            prefill_all.append(e[0].elapsed_time(e[1]))
    prefill_ms = float(np.median(prefill_all))
    if native:
        ncomm.close()
    dec = ShardedDecoder(km, K, V, G, B, comm, sink_rows=sink_rows, ctx=ctx)
    T = args.warmup + args.steps
    ar = torch.arange(U, device=dev)
    qs = []
    for _ in range(T):
        c = centers[ar.repeat_interleave(G), torch.randint(0, centers.shape[1], (U * G,),
                                                            device=dev, generator=g)]
        qq = c + 0.15 * torch.randn(U * G, D, device=dev, generator=g)
        qs.append((2.0 * math.sqrt(D) * qq / qq.norm(dim=-1, keepdim=True))
                  .to(torch.bfloat16).float().contiguous())
    for t in range(args.warmup):
        dec.step(qs[t])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(int(str(dev).split(":")[-1])) as clk:
        soak_for(torch, lambda: dec.step(qs[0]), 0.4)
        if world > 1:
            dist.barrier()
        e[0].record()
        for t in range(args.warmup, T):
            dec.step(qs[t])
        e[1].record()
        torch.cuda.synchronize()
    step_ms = e[0].elapsed_time(e[1]) / args.steps
    ntok = int(dec.n_tokens.to(torch.int64).sum().item())
    uniq, _ = unique_kv_rows(torch, dec.run_row, dec.run_off, dec.run_cnt, G, dec.p_cap)
    n_runs = int(dec.run_cnt.sum().item())
    # this rank's bytes: unique KV rows + its centroid slice + the gathered
    # f64 scores + global sizes / prefix / local index + runs + q / out
    rest = U * dec.slice * D * 4 + U * G * C0 * 8 + U * C0 * 4 * 4 + n_runs * 8 + U * G * D * 8
    step_bytes = uniq * D * 2 * 2 + rest
    step_bytes_nodd = ntok * D * 2 * 2 + rest
    iters = km.iterations_used
    passes = int(sum(int(i) + 1 for i in iters))
    flops = 2.0 * (hi - lo) * C0 * D * passes
    step_ms, prefill_ms = _max_over_ranks(torch, dev, world, [step_ms, prefill_ms])
    gbs = step_bytes / (step_ms * 1e-3) / 1e9
    return {"metric": "decode select+attend us/step (70B shape, 128k ctx, B=2048, "
                      "sequence-sharded)",
            "value": step_ms * 1e3, "unit": "us/step", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16 KV, f32/f64 math",
            "data": "synthetic (device draw with trace.hpp generator distributions, bf16)",
            "config": {"workload": f"config E: Llama-3-70B shape, {layers} layers x {kvh} kv x "
                                   f"{G} q heads, {L} ctx, B={B}, one sequence "
                                   f"sequence-sharded x{world}",
                       "global_batch": 1, "seq_len": L, "parallelism": f"sequence-sharded x{world}"},
            "tokens_per_s": 1000.0 / step_ms,
            "step_roofline_rank0": {"achieved_gbs": gbs, "frac": gbs / hbm,
                                    "bytes_per_step": step_bytes,
                                    "bytes_per_step_no_dedupe": step_bytes_nodd},
            "prefill": {"ms": prefill_ms, "ms_all": [round(x, 1) for x in prefill_all],
                        "timing": f"median of {reps} calls after one untimed call",
                        "units": U, "C0": C0, "iters_min": int(min(iters)),
                        "iters_max": int(max(iters)), "passes": passes,
                        "assign_tflops_rank0": flops / (prefill_ms * 1e-3) / 1e12,
                        "host": "ckv_kmeans_sharded (C++ driver, NCCL)" if native
                                else "sharded.py (torch.distributed)"},
            "clocks": clk.summary()}


def run_config_A(args, torch, dev, ctx):
    """configs[0]: the reference's own CPU-runnable case — one layer of the
    Llama-3-8B shape (8 kv / 32 q heads), 4k prompt, cosine k-means (C0 = 51),
    then decode steps at B = 1024.  The same synthetic heads (drawn on the
    device with the reference generator's distributions, trace.hpp:134-198,
    rounded to bf16) run through our session on the GPU and — copied to the
    host — through the compiled reference (oracle/_ref) on all host threads:
    prefill (cluster_prefill of every head) and one decode step
    (select_tokens + approx_attention of every q head)."""
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200.api import ClusterConfig
    from paper_2412_03213_b200.session import Session
    n_kv, G, L, B = 8, 4, 4096, 1024
    steps = args.steps
    T = steps + args.warmup + 2
    g, centers = gen_inputs(torch, dev, n_kv, G, L, T, seed=7)
    K = torch.empty((n_kv, L, D), dtype=torch.int16, device=dev)
    V = torch.empty_like(K)
    fill_kv(torch, dev, g, centers, K, V, L)
    q_all, kn_all, vn_all = gen_decode(torch, dev, g, centers, G, T)
    seeds = [int(N.lib().ckv_mix_seed(0, 0, h)) for h in range(n_kv)]
    # ---- GPU ------------------------------------------------------------------
    gpu_prefill = []
    for rep in range(4):  # the session re-lays its store: a fresh one per prefill
        sess = Session(n_kv, G, L, T, B, retention=1, cfg=ClusterConfig(), kv_heads=n_kv,
                       ctx=ctx)
        sess.K[:, :L].copy_(K)
        sess.V[:, :L].copy_(V)
        e = _events(torch, 2)
        e[0].record()
        sess.prefill()
        e[1].record()
        torch.cuda.synchronize()
        if rep:
            gpu_prefill.append(e[0].elapsed_time(e[1]))
    out = torch.empty((n_kv * G, D), dtype=torch.float32, device=dev)
    for t in range(args.warmup):
        sess.step(q_all[t], kn_all[t], vn_all[t], out)
    e = _events(torch, 2)
    torch.cuda.synchronize()
    with ClockSampler(int(str(dev).split(":")[-1])) as clk:
        soak_out = torch.empty_like(out)
        soak_for(torch, lambda: sess.attend_only(q_all[0], soak_out), 0.4)
        e[0].record()
        for t in range(steps):
            sess.step(q_all[args.warmup + t], kn_all[args.warmup + t], vn_all[args.warmup + t],
                      out)
        e[1].record()
        torch.cuda.synchronize()
    gpu_step = e[0].elapsed_time(e[1]) / steps
    gp = float(np.median(gpu_prefill))
    # ---- CPU reference (the cpu_baseline leg) -----------------------------------
    from oracle.oracle import ClusterConfig as OCfg
    from oracle.oracle import Oracle, build, ref_available
    if not ref_available():
        build(ref=True)
    R = Oracle("reference")
    cores = int(R.lib.ref_hardware_concurrency())
    f32 = lambda t16: np.ascontiguousarray((t16.to(torch.int32) << 16).view(torch.float32).cpu().numpy())
    Kh, Vh = f32(K), f32(V)
    seeds_np = np.array(seeds, np.uint64)
    kptr = (C.c_void_p * n_kv)(*[Kh[h].ctypes.data for h in range(n_kv)])
    passes = np.zeros(1, np.uint64)
    cpu_prefill = float(np.median([R.lib.ref_prefill_cpu(kptr, n_kv, L, D, seeds_np, 50, cores,
                                                         passes) for _ in range(3)]))
    models = [R.cluster_prefill(Kh[h], OCfg(seed=seeds[h])) for h in range(n_kv)]
    sample = ([np.ascontiguousarray(m.centroids) for m in models],
              np.array([m.n_clusters for m in models], np.uint32),
              [np.ascontiguousarray(m.labels) for m in models], list(Kh), list(Vh),
              np.ascontiguousarray(q_all[0].cpu().numpy()))
    cpu_decode_reps = [cpu_reference_decode(sample, cores, G, L, B) for _ in range(6)]
    cpu_step = float(np.median(cpu_decode_reps[1:]))  # one layer = one step here
    return {"metric": "config A: prefill ms and decode step us (1 layer, 8 kv / 32 q, 4k, "
                      "B=1024), GPU vs the compiled reference on host threads",
            "value": gpu_step * 1e3, "unit": "us/step", "n_gpus": 1, "steps": steps,
            "warmup": args.warmup, "ms_per_step": gpu_step, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 KV, f32/f64 math",
            "data": "synthetic (device draw with trace.hpp generator distributions, bf16)",
            "config": {"workload": "config A: Llama-3-8B head shape, 1 layer, 8 kv x 4 q heads, "
                                   "4096-token prompt, C0 = 51, B = 1024",
                       "global_batch": 1, "seq_len": L},
            "prefill": {"gpu_ms": gp, "cpu_reference_ms": cpu_prefill,
                        "speedup": cpu_prefill / gp, "passes": int(passes[0])},
            "decode": {"gpu_us": gpu_step * 1e3, "cpu_reference_us": cpu_step * 1e3,
                       "speedup": cpu_step / gpu_step},
            "cpu_baseline": {"value": cpu_step * 1e3, "unit": "us/step", "cores": cores,
                             "kind": "reference",
                             "sample": "the whole config-A step: select_tokens + "
                                       "approx_attention of all 32 q heads (median of 5), and "
                                       "cluster_prefill of all 8 heads (median of 3), on the "
                                       "same bf16 heads copied to the host"},
            "clocks": clk.summary()}


def run_page_baseline(torch, dev, ctx, sess, U, G, L, B, q, hbm, ps=16, kv_heads=8):
    """the page-select baseline (selection.hpp:136-194) on the
    same prompts, same queries, same budget: GPU latency of page select +
    attend over a position-ordered store, and the quality of both selections
    for every q head on the GPU (ckv_metrics.cu): recall against the exact
    top-B (exact_topb, selection.hpp:115-132) and the output error against
    full attention (harness.hpp:228-310)."""
    from paper_2412_03213_b200 import _native as N
    st = sess.state()
    n = L - 16
    n_q = U * G
    # the prompt back in position order (the session's store is cluster-major)
    srt = st["sorted_ids"][:, :n].to(torch.int64)
    Kp = torch.empty((U, L, D), dtype=torch.int16, device=dev)
    Vp = torch.empty_like(Kp)
    for dst, store in ((Kp, sess.K), (Vp, sess.V)):
        dst[:, :16] = store[:, :16]
        dst.scatter_(1, srt[..., None].expand(-1, -1, D), store[:, 16:L])
    n_pages = (L + ps - 1) // ps
    n_sel = min(n_pages, B // ps)
    rmax = torch.empty((U, n_pages, D), dtype=torch.float32, device=dev)
    e = _events(torch, 2)
    e[0].record()
    N.check(N.lib().ckv_page_reps(ctx.h, U, L, L, ps, n_pages, Kp.data_ptr(), rmax.data_ptr(),
                                  None))
    e[1].record()
    torch.cuda.synchronize()
    reps_ms = e[0].elapsed_time(e[1])
    rr = torch.zeros((n_q, n_sel + 1), dtype=torch.int32, device=dev)
    ro = torch.zeros((n_q, n_sel + 2), dtype=torch.int32, device=dev)
    rc = torch.zeros(n_q, dtype=torch.int32, device=dev)
    runs = N.Runs(rr.data_ptr(), ro.data_ptr(), rc.data_ptr(), n_sel + 1)
    ids = torch.zeros((n_q, n_sel * ps), dtype=torch.int32, device=dev)
    nt = torch.zeros(n_q, dtype=torch.int32, device=dev)
    pd = N.PageDesc(n_q, G, L, ps, B, n_pages, n_sel * ps, 0)
    ad = N.AttendDesc(n_q, G, L, n_sel * ps, n_sel * ps)
    out = torch.empty((n_q, D), dtype=torch.float32, device=dev)
    qd = q.contiguous()

    def sel(with_ids=False):
        N.check(N.lib().ckv_page_select(ctx.h, C.byref(pd), qd.data_ptr(), rmax.data_ptr(), None,
                                        C.byref(runs), ids.data_ptr() if with_ids else None,
                                        nt.data_ptr()))

    def att():
        N.check(N.lib().ckv_attend(ctx.h, C.byref(ad), qd.data_ptr(), Kp.data_ptr(), Vp.data_ptr(),
                                   None, C.byref(runs), nt.data_ptr(), out.data_ptr(), None))

    for _ in range(3):
        sel()
        att()
    ev = _events(torch, 3 * 10)
    for i in range(10):
        ev[3 * i].record()
        sel()
        ev[3 * i + 1].record()
        att()
        ev[3 * i + 2].record()
    torch.cuda.synchronize()
    sel_us = float(np.mean([ev[3 * i].elapsed_time(ev[3 * i + 1]) for i in range(10)])) * 1e3
    att_us = float(np.mean([ev[3 * i + 1].elapsed_time(ev[3 * i + 2]) for i in range(10)])) * 1e3
    # recall sample: the first layer's q heads, cluster vs page selection
    sel(True)
    c_cap, sel_cap = st["c_cap"], st["sel_cap"]
    sd = N.SelectDesc(n_q, G, B, 16, sess.p_cap, c_cap, sel_cap, L, L, 0, 16)
    ptrs = [C.c_void_p() for _ in range(8)]
    cc, scap = C.c_uint32(), C.c_uint32()
    N.lib().ckv_session_state(sess.h, *[C.byref(p) for p in ptrs], C.byref(cc), C.byref(scap))
    tok = torch.zeros((n_q, sel_cap), dtype=torch.int32, device=dev)
    ntc = torch.zeros(n_q, dtype=torch.int32, device=dev)
    tmp = [torch.zeros(n_q, dtype=torch.int32, device=dev) for _ in range(2)]
    rk = torch.zeros((n_q, c_cap), dtype=torch.int32, device=dev)
    rr2 = torch.zeros((n_q, c_cap + 2), dtype=torch.int32, device=dev)
    ro2 = torch.zeros((n_q, c_cap + 3), dtype=torch.int32, device=dev)
    rc2 = torch.zeros(n_q, dtype=torch.int32, device=dev)
    runs2 = N.Runs(rr2.data_ptr(), ro2.data_ptr(), rc2.data_ptr(), c_cap + 2)
    N.check(N.lib().ckv_select(ctx.h, C.byref(sd), qd.data_ptr(), ptrs[0], ptrs[2], ptrs[3],
                               ptrs[4], ptrs[5], tok.data_ptr(), None, C.byref(runs2),
                               ntc.data_ptr(), tmp[0].data_ptr(), tmp[1].data_ptr(),
                               rk.data_ptr(), None, None))
    # the cluster selection's attention over the session's cluster-major store
    cl_out = torch.empty((n_q, D), dtype=torch.float32, device=dev)
    adc = N.AttendDesc(n_q, G, sess.p_cap, sel_cap, B + 16)
    N.check(N.lib().ckv_attend(ctx.h, C.byref(adc), qd.data_ptr(), sess.K.data_ptr(),
                               sess.V.data_ptr(), None, C.byref(runs2), ntc.data_ptr(),
                               cl_out.data_ptr(), None))
    # quality of both selections on the device (ckv_metrics.cu), every q head
    from paper_2412_03213_b200.metrics import StepQuality
    sq = StepQuality(Kp, Vp, L, G, B, ctx)
    e = _events(torch, 2)
    e[0].record()
    qc = sq(qd, tok, ntc, cl_out)
    e[1].record()
    torch.cuda.synchronize()
    quality_ms = e[0].elapsed_time(e[1])
    rc_m, lc_m = float(qc["recall"].mean().item()), float(qc["l2_rel"].mean().item())
    qp = sq(qd, ids, nt, out)
    rp_m, lp_m = float(qp["recall"].mean().item()), float(qp["l2_rel"].mean().item())
    del Kp, Vp, rmax, sq
    return {"page_size": ps, "repr": "max", "budget": B,
            "page_select_us": sel_us, "page_attend_us": att_us,
            "page_step_us": sel_us + att_us, "page_reps_ms_once": reps_ms,
            "quality": f"every q head ({n_q}) at the prompt context, sinks included in the "
                       f"cluster selection: recall vs exact top-{B} (exact_topb) and l2_rel vs "
                       "full attention, on the GPU (ckv_metrics.cu)",
            "recall_cluster": rc_m, "recall_page": rp_m,
            "l2_rel_cluster": lc_m, "l2_rel_page": lp_m, "quality_eval_ms": quality_ms}


def N_lib():
    from paper_2412_03213_b200 import _native as N
    return N.lib()


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--L", type=int, default=32768)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--group", type=int, default=4)
    ap.add_argument("--budget", type=int, default=1024)
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--exact-kmeans", action="store_true")
    ap.add_argument("--config", default="B", choices=["A", "B", "C", "D", "E"],
                    help="B = the headline (configs[1], plus a config D block); C / D / E "
                         "print their own line")
    ap.add_argument("--gen-tokens", type=int, default=4096, help="config D generated tokens")
    ap.add_argument("--L-E", type=int, default=131072, help="config E context")
    ap.add_argument("--no-extra", action="store_true", help="skip the config D block")
    ap.add_argument("--trace", default=None,
                    help="a CKVT trace file (trace.hpp format): its heads are the units "
                         "of the decode bench instead of the synthetic draw")
    ap.add_argument("--max-iters", type=int, default=50,
                    help="k-means cap (profiling only; the bench default is the reference's 50)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return spawn_world(args.gpus)  # one process per GPU (torchrun re-exec)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" in os.environ and world != args.gpus and args.impl == "ours":
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    local = rank_device(int(os.environ.get("LOCAL_RANK", "0")))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        if os.environ.get("CKV_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200.api import ClusterConfig, Context
    from paper_2412_03213_b200.session import Session

    hbm, bf16_peak, bf16_sus, peak_kind = peaks()
    if args.config in ("A", "C", "E", "D"):
        ctx = Context(local)
        if args.config == "A":
            line = run_config_A(args, torch, dev, ctx) if rank == 0 else None
        elif args.config == "D":
            line = run_config_D(torch, dev, ctx, args) if rank == 0 else None
        elif args.config == "C":
            line = run_config_C(args, rank, world, torch, dev, ctx, hbm)
        else:
            line = run_config_E(args, rank, world, torch, dev, ctx, hbm)
        if rank == 0:
            print(json.dumps(line))
        if world > 1:
            dist.destroy_process_group()
        return
    U = args.layers * args.kv_heads
    G, L, B = args.group, args.L, args.budget
    T = 2 * (args.warmup + args.steps) + args.e2e_steps + 2
    ctx = Context(local)
    sess_flags = (N.CKV_KM_EXACT_ONLY if args.exact_kmeans else 0) | \
        (0 if os.environ.get("CKV_NO_L2_PERSIST") else N.CKV_SESSION_L2_PERSIST)
    sess = Session(U, G, L, T, B, retention=1, cfg=ClusterConfig(max_iters=args.max_iters),
                   kv_heads=args.kv_heads, flags=sess_flags, ctx=ctx)
    if args.trace:  # a CKVT file's heads instead of the synthetic draw
        from paper_2412_03213_b200 import trace as TR
        tb = TR.read_trace(args.trace)
        Kt, Vt, Qt, dKt, dVt = TR.to_device(tb, dev, decode_kv=True)
        if Kt.shape[0] != U or Kt.shape[1] != L:
            raise SystemExit(f"--trace: need {U} heads of L = {L} (pass --layers/--kv-heads/--L); "
                             f"the file has {Kt.shape[0]} heads of L = {Kt.shape[1]}")
        sess.K[:, :L].copy_(Kt)
        sess.V[:, :L].copy_(Vt)
        Tt = Qt.shape[1]
        rows = (torch.arange(T, device=dev)[:, None] + torch.arange(G, device=dev)[None, :] *
                max(1, Tt // G)) % Tt  # the GQA row offset of SURVEY §8d
        q_all = Qt[:, rows].permute(1, 0, 2, 3).reshape(T, U * G, D).contiguous()
        kn_all = dKt[:, torch.arange(T, device=dev) % Tt].permute(1, 0, 2).contiguous()
        vn_all = dVt[:, torch.arange(T, device=dev) % Tt].permute(1, 0, 2).contiguous()
        del Kt, Vt, Qt, dKt, dVt
    else:
        g, centers = gen_inputs(torch, dev, U, G, L, T, seed=7 + rank)
        fill_kv(torch, dev, g, centers, sess.K, sess.V, L)
        q_all, kn_all, vn_all = gen_decode(torch, dev, g, centers, G, T)
    torch.cuda.synchronize()

    # ---- prefill clustering --------------------------------------------
    # cluster_prefill of all units through the C-ABI (ckv_cluster_prefill) on
    # the prompt keys in HBM: two warm-up calls (first-touch scratch
    # allocation, clock ramp), then the median of 9 timed calls (single calls
    # on the shared boxes sometimes stall on the host for 100+ ms; the list
    # goes to stderr and `ms_all`).  The session's own
    # prefill (the same k-means + build_index + cluster-major relayout) is
    # timed once after it as `session_ms`.
    p_cap = sess.p_cap
    c_cap = N.lib().ckv_prefill_cluster_count(L, 80, 16, 0) + 64
    km_c = torch.empty((U, c_cap, D), dtype=torch.float32, device=dev)
    km_l = torch.empty((U, p_cap), dtype=torch.int32, device=dev)
    km_n = torch.empty((U,), dtype=torch.int32, device=dev)
    seeds = (C.c_uint64 * U)(*[N.lib().ckv_mix_seed(0, u // args.kv_heads, u % args.kv_heads)
                               for u in range(U)])
    km_info = (N.KMeansInfo * U)()
    pdesc = N.PrefillDesc(U, L, p_cap, c_cap, 80, 16, args.max_iters, 0,
                          N.CKV_KM_EXACT_ONLY if args.exact_kmeans else 0)
    km_ms = []
    for rep in range(11):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(N.lib().ckv_cluster_prefill(ctx.h, C.byref(pdesc), sess.K.data_ptr(),
                                            C.cast(seeds, C.c_void_p), km_c.data_ptr(),
                                            km_l.data_ptr(), km_n.data_ptr(),
                                            C.cast(km_info, C.c_void_p), None, None))
        e1.record()
        torch.cuda.synchronize()
        if rep >= 2:
            km_ms.append(e0.elapsed_time(e1))
    prefill_ms = float(np.median(km_ms))
    print(f"[bench] cluster_prefill ms per call: {[round(x, 1) for x in km_ms]}", file=sys.stderr)
    del km_c, km_l, km_n
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    info = sess.prefill()
    e1.record()
    torch.cuda.synchronize()
    session_prefill_ms = e0.elapsed_time(e1)
    iters = [i for i, _ in info]
    C0 = int(sess.state()["n_clusters"][0].item())
    N_ = L - 16
    passes = sum(i + 1 for i in iters)
    assign_flops = 2.0 * N_ * C0 * D * passes

    # ---- decode steps (device-resident inputs) -------------------------
    n_q = U * G
    out = torch.empty((n_q, D), dtype=torch.float32, device=dev)
    t = 0
    for _ in range(args.warmup):
        sess.step(q_all[t], kn_all[t], vn_all[t], out)
        t += 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    soak_out = torch.empty_like(out)

    def soak(seconds):  # keeps the GPU busy so nvidia-smi samples loaded clocks
        t_end = time.time() + seconds
        while time.time() < t_end:
            for _ in range(20):
                sess.attend_only(q_all[0], soak_out)
            torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        soak(0.4)
        l0 = ctx.launches
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(args.steps):
            sess.step(q_all[t], kn_all[t], vn_all[t], out)
            t += 1
        ev[1].record()
        launches = ctx.launches - l0
        torch.cuda.synchronize()
        soak(0.2)
    step_ms = ev[0].elapsed_time(ev[1]) / args.steps
    if world > 1:
        step_ms = _max_over_ranks(torch, dev, world, [step_ms])[0]
        dist.barrier()

    # ---- layer mode: one (select, attend) pair per layer, in layer order --
    # (a decoder's dependency order: layer l+1's queries need layer l's
    # output), vs the layer-batched step above (the harness's independent
    # (layer, head) fan-out, harness.hpp:362-378)
    sess.set_layer_units(args.kv_heads)
    for _ in range(args.warmup):
        sess.step(q_all[t], kn_all[t], vn_all[t], out)
        t += 1
    torch.cuda.synchronize()
    evl = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    evl[0].record()
    for _ in range(args.steps):
        sess.step(q_all[t], kn_all[t], vn_all[t], out)
        t += 1
    evl[1].record()
    torch.cuda.synchronize()
    layer_step_ms = evl[0].elapsed_time(evl[1]) / args.steps
    sess.set_layer_units(0)
    if world > 1:
        layer_step_ms = _max_over_ranks(torch, dev, world, [layer_step_ms])[0]

    # ---- per-kernel timing of one step's select and attend --------------
    st = sess.state()
    sel_cap, c_cap = st["sel_cap"], st["c_cap"]
    ncl = st["n_clusters"].to(torch.int64)
    stats = sess.stats()
    rec_begin, rec_end = stats.labeled_end, stats.n_ctx
    sd = N.SelectDesc(n_q, G, B, 16, sess.p_cap, c_cap, sel_cap, rec_begin, rec_end,
                      N.CKV_SEL_L2_PERSIST if sess_flags & N.CKV_SESSION_L2_PERSIST else 0, 16)
    ad = N.AttendDesc(n_q, G, sess.p_cap, sel_cap, min(B, rec_begin) + 16 + (rec_end - rec_begin))
    st_ptrs = [C.c_void_p() for _ in range(8)]
    cc, scap = C.c_uint32(), C.c_uint32()
    N.lib().ckv_session_state(sess.h, *[C.byref(p) for p in st_ptrs], C.byref(cc), C.byref(scap))
    ranked = torch.empty((n_q, c_cap), dtype=torch.int32, device=dev)
    ntk = torch.empty(n_q, dtype=torch.int32, device=dev)
    trm = torch.empty(n_q, dtype=torch.int32, device=dev)
    rows2 = torch.empty((n_q, sel_cap), dtype=torch.int32, device=dev)
    run_cap = c_cap + 2
    run_row = torch.empty((n_q, run_cap), dtype=torch.int32, device=dev)
    run_off = torch.empty((n_q, run_cap + 1), dtype=torch.int32, device=dev)
    run_cnt = torch.empty(n_q, dtype=torch.int32, device=dev)
    runs = N.Runs(run_row.data_ptr(), run_off.data_ptr(), run_cnt.data_ptr(), run_cap)
    nt2 = torch.empty(n_q, dtype=torch.int32, device=dev)
    qd = q_all[t - 1].contiguous()

    def select(rows_ptr=None):
        N.check(N.lib().ckv_select(ctx.h, C.byref(sd), qd.data_ptr(), st_ptrs[0], st_ptrs[2],
                                   st_ptrs[3], st_ptrs[4], st_ptrs[5], None, rows_ptr,
                                   C.byref(runs), nt2.data_ptr(), ntk.data_ptr(),
                                   trm.data_ptr(), ranked.data_ptr(), None, None))

    # byte accounting from one untimed selection with per-entry rows
    select(rows2.data_ptr())
    ntok = nt2.to(torch.int64)
    nq_tok = int(ntok.sum().item())
    uniq = 0  # unique (kv unit, row) pairs: the q heads of a group share their unit's KV
    for u in range(U):
        rr = torch.cat([rows2[u * G + r, : int(ntok[u * G + r].item())] for r in range(G)])
        uniq += int(torch.unique(rr).numel())
    n_runs = int(run_cnt.sum().item())
    n_cl = int(ncl.sum().item())
    qo_bytes = n_q * D * 8
    attend_bytes_unique = uniq * D * 2 * 2 + n_runs * 8 + qo_bytes
    attend_bytes_perq = nq_tok * D * 2 * 2 + n_runs * 8 + qo_bytes
    select_bytes = n_cl * D * 4 + n_cl * 8 + n_runs * 8 + n_q * D * 4
    step_bytes_unique = attend_bytes_unique + select_bytes
    reps = 10
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(3 * reps)]
    for i in range(reps):
        evs[3 * i].record()
        select()
        evs[3 * i + 1].record()
        N.check(N.lib().ckv_attend(ctx.h, C.byref(ad), qd.data_ptr(), sess.K.data_ptr(),
                                   sess.V.data_ptr(), None, C.byref(runs), nt2.data_ptr(),
                                   out.data_ptr(), None))
        evs[3 * i + 2].record()
    torch.cuda.synchronize()
    sel_ms = float(np.mean([evs[3 * i].elapsed_time(evs[3 * i + 1]) for i in range(2, reps)]))
    att_ms = float(np.mean([evs[3 * i + 1].elapsed_time(evs[3 * i + 2]) for i in range(2, reps)]))

    page_block = None
    if not args.no_extra and world == 1:
        try:
            page_block = run_page_baseline(torch, dev, ctx, sess, U, G, L, B, q_all[t - 1], hbm,
                                           kv_heads=args.kv_heads)
        except Exception as ex:  # reported, never silently dropped
            page_block = {"failed": repr(ex)}

    # ---- e2e through the public step API with host buffers --------------
    qh = torch.empty((n_q, D), dtype=torch.float32).pin_memory()
    kh = torch.empty((U, D), dtype=torch.int16).pin_memory()
    vh = torch.empty((U, D), dtype=torch.int16).pin_memory()
    oh = torch.empty((n_q, D), dtype=torch.float32).pin_memory()
    e2e_times = []
    for _ in range(args.e2e_steps):
        if t >= T:
            break
        qh.copy_(q_all[t].cpu())
        kh.copy_(kn_all[t].cpu())
        vh.copy_(vn_all[t].cpu())
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        N.check(N.lib().ckv_session_step(sess.h, qh.data_ptr(), kh.data_ptr(), vh.data_ptr(),
                                         oh.data_ptr(), 0))
        b.record()
        torch.cuda.synchronize()
        e2e_times.append(a.elapsed_time(b))
        t += 1
    # median over the steps after the first (a host hiccup in one call of a
    # ~150 us step moves a mean of 10 by several percent)
    e2e_ms = float(np.median(e2e_times[1:] if len(e2e_times) > 1 else e2e_times))
    if world > 1:
        e2e_ms, prefill_ms = _max_over_ranks(torch, dev, world, [e2e_ms, prefill_ms])

    # ---- CPU baseline (rank 0, N=1 only) ---------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle.oracle import Oracle, build, ref_available
            if not ref_available():
                build(ref=True)
            Rr = Oracle("reference")
            cores = int(Rr.lib.ref_hardware_concurrency())
            sample = layer_sample_from_device(torch, sess, args.kv_heads, G, L, q_all[0])
            cpu_reference_decode(sample, cores, G, L, B)
            layer_ms = float(np.median([cpu_reference_decode(sample, cores, G, L, B)
                                        for _ in range(5)]))
            cpu_step_ms = layer_ms * args.layers
            cpu = {"value": 1000.0 / cpu_step_ms, "unit": "tokens/s", "cores": cores,
                   "kind": "reference",
                   "sample": f"one layer ({args.kv_heads} kv / {args.kv_heads * G} q heads, 32k, "
                             f"B={B}) select_tokens+approx_attention x5, median {layer_ms:.2f} ms, "
                             f"scaled x{args.layers} layers; model = the GPU-built clusters "
                             "(bit-identical to the reference's)"}
            # SURVEY §8(d) prefill baseline: the reference's cluster_prefill of
            # the same layer's heads, capped at 2 iterations (3 passes per head),
            # one head per thread: cost per head-pass at 32k
            try:
                kh = [np.ascontiguousarray(k, np.float32) for k in sample[3]]
                nh = len(kh)
                kptr = (C.c_void_p * nh)(*[k.ctypes.data for k in kh])
                seeds_np = np.array([N.lib().ckv_mix_seed(0, 0, h) for h in range(nh)], np.uint64)
                npass = np.zeros(1, np.uint64)
                cms = float(Rr.lib.ref_prefill_cpu(kptr, nh, L, D, seeds_np, 2, cores, npass))
                thr = min(cores, nh)
                gpu_hps = passes / (prefill_ms * 1e-3)
                cpu_hps = int(npass[0]) / (cms * 1e-3)
                cpu["prefill"] = {
                    "head_passes_per_s": cpu_hps, "threads": thr,
                    "ms_per_head_pass_per_thread": cms * thr / max(1, int(npass[0])),
                    "gpu_head_passes_per_s": gpu_hps, "speedup": gpu_hps / cpu_hps,
                    "sample": f"cluster_prefill of {nh} heads (32k, C0={C0}) capped at 2 "
                              f"iterations ({int(npass[0])} head-passes) in {cms:.0f} ms on {thr} "
                              f"threads; GPU: {passes} unit-passes in the {prefill_ms:.1f} ms "
                              "prefill"}
            except Exception as ex:  # the decode baseline above stands
                cpu["prefill"] = {"sample": f"failed: {ex!r}"}
        except Exception as ex:  # reported, never silently replaced
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {ex!r}"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    tps = world * 1000.0 / step_ms
    att_gbs = attend_bytes_unique / (att_ms * 1e-3) / 1e9
    line = {
        "metric": "decode tokens/s (select+gather+attend, 32k ctx, B=1024)",
        "value": tps, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16 KV, f32/f64 math",
        "data": (f"CKVT trace {os.path.basename(args.trace)} (bf16-rounded)" if args.trace else
                 "synthetic (device draw with trace.hpp generator distributions, bf16)"),
        "config": {"workload": f"config B: Llama-3-8B shape, {args.layers} layers x "
                               f"{args.kv_heads} kv x {G} q heads, {L} ctx, B={B}, batch 1/GPU, "
                               "R=1 cache; all layers of a step in one select + one attend launch",
                   "global_batch": world, "seq_len": L, "parallelism": f"batch-sharded x{world}",
                   "l2": "per-step working set ~0.6 GB >> 126 MB L2 (no flush needed); "
                         "the 54 MB of centroids sit in a persisting L2 window "
                         "(CKV_SESSION_L2_PERSIST; CKV_NO_L2_PERSIST=1 disables)"},
        "select_attend_us_per_step": step_ms * 1e3,
        "roofline": {"bound": "hbm", "kernel": "k_attend", "achieved": att_gbs, "peak": hbm,
                     "unit": "GB/s", "frac": att_gbs / hbm, "traffic": ncu_traffic("k_attend"),
                     "traffic_source": "ncu --set full dram__bytes_read.sum + "
                                       "dram__bytes_write.sum of one k_attend launch of this "
                                       "workload, newest profiles/r*_decode_kernels.json",
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": attend_bytes_unique,
                     "bytes_rule": "unique (kv unit, row) K+V bf16 rows + I_T runs + q/out",
                     "launch_us": att_ms * 1e3},
        "step_roofline": {"achieved_gbs": step_bytes_unique / (step_ms * 1e-3) / 1e9,
                          "frac": step_bytes_unique / (step_ms * 1e-3) / 1e9 / hbm,
                          "bytes_per_step": step_bytes_unique,
                          "bytes_per_step_no_dedupe": attend_bytes_perq + select_bytes},
        "kernels_us": {"k_select": sel_ms * 1e3, "k_attend": att_ms * 1e3},
        "per_layer": {"ms_per_step": layer_step_ms, "tokens_per_s": world * 1000.0 / layer_step_ms,
                      "us_per_layer": layer_step_ms * 1e3 / args.layers,
                      "vs_layer_batched": layer_step_ms / step_ms,
                      "step_roofline_frac": step_bytes_unique / (layer_step_ms * 1e-3) / 1e9 / hbm,
                      "mode": f"{args.layers} sequential (select, attend) launch pairs per step, "
                              f"{args.kv_heads} kv units each (ckv_session_set_layer_units)"},
        "prefill": {"ms": prefill_ms, "session_ms": session_prefill_ms,
                    "timing": "ckv_cluster_prefill of all units, median of 9 after 2 warm-ups",
                    "ms_all": [round(x, 2) for x in km_ms],
                    "units": U, "C0": C0, "iters_min": min(iters),
                    "iters_max": max(iters), "passes": passes,
                    "assign_tflops": assign_flops / (prefill_ms * 1e-3) / 1e12,
                    "frac_of_bf16_peak": assign_flops / (prefill_ms * 1e-3) / 1e12 /
                    (bf16_sus or bf16_peak)},
        "e2e": {"value": world * 1000.0 / e2e_ms, "unit": "tokens/s",
                "h2d_bytes_per_step": n_q * D * 4 + 2 * U * D * 2,
                "d2h_bytes_per_step": n_q * D * 4,
                "timing": f"median of {max(1, len(e2e_times) - 1)} ckv_session_step calls, "
                          "each synchronous (host call to result in pinned host memory)"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if page_block is not None:
        line["page_baseline"] = page_block
    if not args.no_extra and world == 1:
        try:
            line["quality"] = run_quality(torch, dev, ctx, args)
        except Exception as ex:  # reported, never silently dropped
            line["quality"] = {"failed": repr(ex)}
    if not args.no_extra and world == 1:
        del sess
        torch.cuda.synchronize()
        try:
            line["config_D"] = run_config_D(torch, dev, ctx, args)
        except Exception as ex:  # reported, never silently dropped
            line["config_D"] = {"failed": repr(ex)}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
