"""GPU decode-loop quality driver: the reference harness's
ClusterKV simulation (run_simulation / simulate_head, harness.hpp:155-410)
and its parameter sweep (harness.hpp:428-475), at GPU speed.

Every (layer, head) of a TraceBundle is one unit of a device Session (group
1: each trace head brings its own decode queries, as simulate_head does).
Per decode step t the session runs the serving path — select (+ cluster
cache) -> sparse attention -> append, decode-batch clustering every m steps,
synchronous or async (harness.hpp:236-243, 318-337) — and the metric
kernels (ckv_metrics.cu) score it the way simulate_head does per row:

  recall   |I_T ∩ exact_topb(q, ctx, min(B, n_ctx))| / min(B, n_ctx)
           (selection.hpp:115-132, attention.hpp:70-93), bit-exact;
  l2_rel, cos_sim   output_error(approx, full_attention) (attention.hpp:
           53-60, 101-131), f32 attention against the f64 reference
           (DESIGN.md §5 tolerance);
  clusters_hit / requested / tokens_transferred   the step's cluster-cache
           counter deltas (harness.hpp:250-258), bit-exact.

RunSummary aggregates like run_simulation (means over rows, hit rate over
all requests, transferred tokens/bytes, the k-means iteration histogram).
Checked against the compiled reference's own run_simulation in
tests/test_gpu_quality.py.  Only the ClusterKV policy with its recency
window runs on the GPU path (the page-select baseline has its own kernels,
api.page_select); Oracle/Greedy/Random/Full are harness ablations.
"""
from __future__ import annotations

import ctypes as C
import time
from collections import Counter
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._native import ValidationError, check, lib
from .api import ClusterConfig, Context
from .session import Session
from .trace import TraceBundle

D = 128


@dataclass
class PolicyConfig:
    """harness.hpp:52-70, the fields of the ClusterKV policy."""

    budget: int = 1024
    cluster: ClusterConfig = field(default_factory=ClusterConfig)
    retention: int = 1
    recency_window: bool = True
    async_clustering: bool = False
    async_delay: int = 8

    def validate(self) -> None:  # harness.hpp:64-69
        if self.budget < 1:
            raise ValidationError(1, "PolicyConfig: budget must be >= 1")
        if self.retention < 1:
            raise ValidationError(1, "PolicyConfig: retention must be >= 1")
        self.cluster.validate()
        if not self.recency_window:
            raise ValidationError(1, "PolicyConfig: the GPU session always keeps the recency "
                                     "window (recency_window = false is a harness ablation)")


@dataclass
class StepRow:
    """harness.hpp:72-84."""

    step: int
    layer: int
    head: int
    recall: float
    l2_rel: float
    cos_sim: float
    clusters_hit: int
    clusters_requested: int
    tokens_transferred: int


@dataclass
class RunSummary:
    """harness.hpp:86-98."""

    policy: str = "clusterkv"
    budget: int = 0
    mean_recall: float = 0.0
    mean_l2_rel: float = 0.0
    mean_cos_sim: float = 0.0
    hit_rate: float = 0.0
    tokens_transferred: int = 0
    bytes_transferred: int = 0
    iteration_histogram: dict = field(default_factory=dict)
    wall_ms: float = 0.0


@dataclass
class RunReport:
    rows: list
    summary: RunSummary


def run_simulation(bundle: TraceBundle, cfg: PolicyConfig, ctx: Context | None = None,
                   rows: bool = True) -> RunReport:
    """run_simulation (harness.hpp:362-410) of the ClusterKV policy on the GPU.
    The bundle's matrices must be bf16-representable (the device store is
    bf16).  rows=False skips the per-row list (the summary
    stays exact)."""
    t0 = time.perf_counter()
    bundle.validate()
    cfg.validate()
    ctx = ctx or Context.default()
    dev = ctx.device
    f0 = bundle.traces[0]
    L, T = f0.prompt_keys.shape[0], f0.decode_queries.shape[0]
    if f0.d != D:
        raise ValidationError(1, "run_simulation: the B200 kernels specialise d = 128")
    U, H = len(bundle.traces), bundle.n_heads
    B = cfg.budget
    cc = cfg.cluster

    def bits(name):  # [U][rows][128] bf16 bit patterns on the device
        x = torch.from_numpy(np.stack([np.asarray(getattr(tr, name), np.float32)
                                       for tr in bundle.traces])).to(dev)
        b = x.to(torch.bfloat16)
        if not torch.equal(b.float(), x):
            raise ValidationError(1, f"run_simulation: {name} is not bf16-representable")
        return b.view(torch.int16).contiguous()

    Kp, Vp = bits("prompt_keys"), bits("prompt_values")
    dK, dV = bits("decode_keys"), bits("decode_values")
    Q = torch.from_numpy(np.stack([np.asarray(tr.decode_queries, np.float32)
                                   for tr in bundle.traces])).to(dev)
    sess = Session(U, 1, L, T, B, retention=cfg.retention, cfg=cc, kv_heads=H,
                   flags=N.CKV_SESSION_TOKEN_IDS, ctx=ctx,
                   async_delay=cfg.async_delay if cfg.async_clustering else 0)
    sess.K[:, :L].copy_(Kp)
    sess.V[:, :L].copy_(Vp)
    info = sess.prefill()
    hist = Counter(it for it, _ in info)
    # position-ordered copy of the context for the metric kernels (the
    # session's own store is cluster-major)
    P = L + T
    Kpos = torch.zeros((U, P, D), dtype=torch.int16, device=dev)
    Vpos = torch.zeros_like(Kpos)
    Kpos[:, :L].copy_(Kp)
    Vpos[:, :L].copy_(Vp)
    del Kp, Vp
    bcap = min(B, P)
    truth = torch.zeros((U, bcap), dtype=torch.int32, device=dev)
    recall = torch.zeros(U, dtype=torch.float64, device=dev)
    l2 = torch.zeros(U, dtype=torch.float64, device=dev)
    cos = torch.zeros(U, dtype=torch.float64, device=dev)
    exact = torch.zeros((U, D), dtype=torch.float32, device=dev)
    out = torch.zeros((U, D), dtype=torch.float32, device=dev)
    rr = torch.zeros((U, 1), dtype=torch.int32, device=dev)
    ro = torch.zeros((U, 2), dtype=torch.int32, device=dev)
    rc = torch.zeros(U, dtype=torch.int32, device=dev)
    fruns = N.Runs(rr.data_ptr(), ro.data_ptr(), rc.data_ptr(), 1)
    fnt = torch.zeros(U, dtype=torch.int32, device=dev)
    st = sess.state()
    sel_cap = st["sel_cap"]
    Lb, h = lib(), ctx.h
    ctr_prev = np.zeros((U, 4), np.uint64)
    rec_rows, recs = [], [[], [], [], [], [], []]
    m = cc.decode_batch
    import os as _os
    dbg = _os.environ.get("CKV_QUALITY_TRACE") is not None
    for t in range(T):
        n_ctx = L + t
        if dbg:
            torch.cuda.synchronize()
            print("[quality] step", t, flush=True)
        q = Q[:, t].contiguous()
        sess.step(q, dK[:, t].contiguous(), dV[:, t].contiguous(), out)
        # quality of this step's selection on the context it saw (n_ctx rows)
        bn = min(B, n_ctx)
        check(Lb.ckv_exact_topb(h, U, 1, n_ctx, P, q.data_ptr(), Kpos.data_ptr(), B,
                                truth.data_ptr(), bcap))
        check(Lb.ckv_recall(h, U, st["token_ids"].data_ptr(), sel_cap, st["n_tokens"].data_ptr(),
                            truth.data_ptr(), bcap, bn, recall.data_ptr()))
        check(Lb.ckv_full_runs(h, U, n_ctx, C.byref(fruns), fnt.data_ptr()))
        ad = N.AttendDesc(U, 1, P, n_ctx, n_ctx)
        check(Lb.ckv_attend(h, C.byref(ad), q.data_ptr(), Kpos.data_ptr(), Vpos.data_ptr(), None,
                            C.byref(fruns), fnt.data_ptr(), exact.data_ptr(), None))
        check(Lb.ckv_output_error(h, U, out.data_ptr(), exact.data_ptr(), l2.data_ptr(),
                                  cos.data_ptr()))
        ctr = sess.cache_counters()
        d = (ctr - ctr_prev).astype(np.int64)
        ctr_prev = ctr
        for k, x in enumerate((recall, l2, cos)):
            recs[k].append(x.cpu().numpy().copy())
        recs[3].append(d[:, 1])
        recs[4].append(d[:, 0])
        recs[5].append(d[:, 2])
        # append (harness.hpp:318-320) to the position-ordered copy
        Kpos[:, n_ctx].copy_(dK[:, t])
        Vpos[:, n_ctx].copy_(dV[:, t])
        if (t + 1) % m == 0 and T - (t + 1) >= 0:  # a decode batch was formed this step
            if not cfg.async_clustering or t + cfg.async_delay < T:
                # the reference records a batch's iterations when it is
                # applied (harness.hpp:240, 332); async batches still pending
                # at the end never are
                hist.update(int(x) for x in sess.batch_iterations())
    torch.cuda.synchronize()
    R = np.stack(recs[0], 1), np.stack(recs[1], 1), np.stack(recs[2], 1)
    hits, reqs, toks = np.stack(recs[3], 1), np.stack(recs[4], 1), np.stack(recs[5], 1)
    if rows:
        for u in range(U):
            for t in range(T):
                rec_rows.append(StepRow(t, u // H, u % H, float(R[0][u, t]), float(R[1][u, t]),
                                        float(R[2][u, t]), int(hits[u, t]), int(reqs[u, t]),
                                        int(toks[u, t])))
    s = RunSummary(budget=B)
    n_rows = U * T
    s.mean_recall = float(R[0].sum() / n_rows)
    s.mean_l2_rel = float(R[1].sum() / n_rows)
    s.mean_cos_sim = float(R[2].sum() / n_rows)
    s.hit_rate = float(hits.sum() / reqs.sum()) if reqs.sum() else 0.0
    s.tokens_transferred = int(ctr_prev[:, 2].sum())
    s.bytes_transferred = int(ctr_prev[:, 3].sum())
    s.iteration_histogram = dict(sorted(hist.items()))
    s.wall_ms = (time.perf_counter() - t0) * 1e3
    del sess
    return RunReport(rec_rows, s)


def sweep(bundle: TraceBundle, base: PolicyConfig, axis: str, values, ctx=None,
          rows: bool = False) -> list:
    """harness.hpp:449-475: one full run per value; axes "budget",
    "retention" and "c0" (the prefill cluster count through c0_divisor's
    override, ClusterConfig.c0_override)."""
    if len(values) == 0:
        raise ValidationError(1, "sweep: empty value list")
    out = []
    for v in values:
        cfg = PolicyConfig(**{**base.__dict__})
        cfg.cluster = ClusterConfig(**{**base.cluster.__dict__})
        if axis == "budget":
            cfg.budget = int(v)
        elif axis == "retention":
            cfg.retention = int(v)
        elif axis == "c0":
            cfg.cluster.c0_override = int(v)
        else:
            raise ValidationError(1, f"unknown sweep axis: {axis}")
        out.append(run_simulation(bundle, cfg, ctx, rows=rows))
    return out
