"""Python mirror of the reference hot-path API, running on the B200 kernels.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/clusterkv/{clustering,selection,attention,
cache}.hpp, so parity tests read like tests of the reference itself.  Every
call goes through the C-ABI (include/ckv_cuda.h) into libckv_b200.so; torch
is used only to own device memory and the stream (plumbing).

Inputs follow the reference's f32 `Matrix` convention (numpy float32,
row-major).  The device KV store is bf16: keys / values must be
bf16-representable or ValidationError is raised — the one
documented deviation from the reference's accepted input domain.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from ._native import ValidationError, check, lib

D = 128
COSINE, L2, INNER_PRODUCT = 0, 1, 2


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class Context:
    """One ckv_ctx bound to torch's current stream on `device`."""

    _default: "Context | None" = None

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("the ClusterKV hot path needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        self.stream = stream or torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        check(lib().ckv_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.h = h

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(torch.cuda.current_device())
        return cls._default

    def sync(self):
        check(lib().ckv_ctx_sync(self.h))

    @property
    def launches(self) -> int:
        return int(lib().ckv_ctx_launch_count(self.h))

    def __del__(self):
        try:
            lib().ckv_ctx_destroy(self.h)
        except Exception:
            pass


# --------------------------------------------------------------------------
# reference types (clustering.hpp:20-55, selection.hpp:18-69,
# attention.hpp:11-14)
# --------------------------------------------------------------------------
@dataclass
class ClusterConfig:
    c0_divisor: int = 80
    c_plus: int = 4
    decode_batch: int = 320
    sink_tokens: int = 16
    max_iters: int = 50
    seed: int = 0
    c0_override: int = 0
    metric: int = COSINE

    def validate(self) -> None:  # clustering.hpp:30-35
        if self.c0_divisor < 1:
            raise ValidationError(1, "ClusterConfig: c0_divisor must be >= 1")
        if self.c_plus < 1:
            raise ValidationError(1, "ClusterConfig: c_plus must be >= 1")
        if self.decode_batch < 1:
            raise ValidationError(1, "ClusterConfig: decode_batch must be >= 1")
        if self.max_iters < 1:
            raise ValidationError(1, "ClusterConfig: max_iters must be >= 1")


@dataclass
class ClusterModel:
    n_clusters: int = 0
    centroids: np.ndarray = field(default_factory=lambda: np.zeros((0, D), np.float32))
    labels: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    sink_count: int = 0
    converged: bool = False
    iterations_used: int = 0
    objective_history: list = field(default_factory=list)
    repair_iterations: list = field(default_factory=list)
    invocation_iterations: list = field(default_factory=list)

    def n_positions(self) -> int:
        return int(len(self.labels))


@dataclass
class ClusterIndex:
    sizes: np.ndarray
    sorted_token_ids: np.ndarray
    cluster_start: np.ndarray

    def labeled_total(self) -> int:
        return int(len(self.sorted_token_ids))

    def cluster_slice(self, c: int) -> np.ndarray:
        s = int(self.cluster_start[c])
        return self.sorted_token_ids[s: s + int(self.sizes[c])]


@dataclass
class SelectionResult:
    ranked_clusters: np.ndarray
    n_clusters_taken: int
    token_ids: np.ndarray
    trimmed_from_last: int
    budget: int

    def taken_clusters(self) -> np.ndarray:
        return self.ranked_clusters[: self.n_clusters_taken]


@dataclass
class AttentionOutput:
    out: np.ndarray
    weights: np.ndarray


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------
def _to_bf16_device(ctx: Context, x: np.ndarray, what: str) -> torch.Tensor:
    x = np.ascontiguousarray(x, np.float32)
    src = torch.from_numpy(x).to(ctx.device)
    dst = torch.empty(src.shape, dtype=torch.int16, device=ctx.device)
    exact = C.c_int(0)
    check(lib().ckv_f32_to_bf16(ctx.h, src.data_ptr(), dst.data_ptr(), src.numel(),
                                C.byref(exact)))
    if not exact.value:
        if not np.all(np.isfinite(x)):
            return dst  # non-finite inputs are rejected by the kernel-side checks
        raise ValidationError(1, f"{what}: values must be bf16-representable "
                                 "(the B200 KV store is bf16; SURVEY §8a N1)")
    return dst


def _check_d(m: np.ndarray, what: str) -> None:
    if m.ndim != 2 or m.shape[1] != D:
        raise ValidationError(1, f"{what}: the B200 kernels specialise d = {D}")


# --------------------------------------------------------------------------
# clustering (clustering.hpp:157-332)
# --------------------------------------------------------------------------
def kmeans_cosine(keys: np.ndarray, n_clusters: int, seed: int, max_iters: int = 50,
                  metric: int = COSINE, init_rows: Sequence[int] | None = None,
                  ctx: Context | None = None, flags: int = N.CKV_KM_OBJECTIVE) -> ClusterModel:
    """kmeans_cosine (clustering.hpp:160-263) on one B200."""
    ctx = ctx or Context.default()
    keys = np.ascontiguousarray(keys, np.float32)
    _check_d(keys, "kmeans")
    n = keys.shape[0]
    if n_clusters < 1 or n_clusters > n:
        raise ValidationError(1, "kmeans: need 1 <= C <= N")
    if metric != COSINE:
        raise ValidationError(1, "kmeans: the B200 path implements the cosine metric only")
    if init_rows is not None and len(init_rows) != 0:
        if len(init_rows) != n_clusters:
            raise ValidationError(1, "kmeans: init_rows size must equal C")
        rows = np.ascontiguousarray(init_rows, np.uint32)
        if rows.max() >= n:
            raise ValidationError(1, "kmeans: init_rows out of range")
    else:
        rows = np.zeros(n_clusters, np.uint32)
        check(lib().ckv_kmeans_init_rows(n, n_clusters, seed, rows.ctypes.data))
    kb = _to_bf16_device(ctx, keys, "kmeans")
    d_rows = torch.from_numpy(rows.view(np.int32)).to(ctx.device)
    cents = torch.empty((n_clusters, D), dtype=torch.float32, device=ctx.device)
    labels = torch.empty(n, dtype=torch.int32, device=ctx.device)
    desc = N.KMeansDesc(1, n, n_clusters, max_iters, n * D, n_clusters, n, flags)
    info = N.KMeansInfo()
    obj = np.zeros(max_iters + 1, np.float64)
    rep = np.zeros(max_iters + 1, np.uint32)
    check(lib().ckv_kmeans(ctx.h, C.byref(desc), kb.data_ptr(), d_rows.data_ptr(),
                           cents.data_ptr(), labels.data_ptr(), C.byref(info), obj.ctypes.data,
                           rep.ctypes.data))
    m = ClusterModel(n_clusters, cents.cpu().numpy(), labels.cpu().numpy(), 0,
                     bool(info.converged), int(info.iterations_used),
                     list(obj[: info.n_objective]), list(rep[: info.n_repair]),
                     [int(info.iterations_used)])
    return m


def prefill_cluster_count(prompt_len: int, cfg: ClusterConfig) -> int:
    """clustering.hpp:267-274."""
    return int(lib().ckv_prefill_cluster_count(prompt_len, cfg.c0_divisor, cfg.sink_tokens,
                                               cfg.c0_override))


def cluster_prefill(keys: np.ndarray, cfg: ClusterConfig, ctx: Context | None = None,
                    flags: int = N.CKV_KM_OBJECTIVE) -> ClusterModel:
    """clustering.hpp:278-305."""
    cfg.validate()
    keys = np.ascontiguousarray(keys, np.float32)
    _check_d(keys, "cluster_prefill")
    L = keys.shape[0]
    if L <= cfg.sink_tokens:
        return ClusterModel(0, np.zeros((0, D), np.float32), np.full(L, -1, np.int32), L, True, 0)
    sink = cfg.sink_tokens
    m = kmeans_cosine(keys[sink:], prefill_cluster_count(L, cfg), cfg.seed, cfg.max_iters,
                      cfg.metric, None, ctx, flags)
    m.sink_count = sink
    m.labels = np.concatenate([np.full(sink, -1, np.int32), m.labels])
    return m


def cluster_decode_batch(model: ClusterModel, new_keys: np.ndarray, cfg: ClusterConfig,
                         ctx: Context | None = None) -> None:
    """clustering.hpp:310-332 — mutates `model` in place."""
    new_keys = np.ascontiguousarray(new_keys, np.float32)
    if new_keys.shape[0] == 0:
        return
    cfg.validate()
    c = min(cfg.c_plus, new_keys.shape[0])
    seed = int(lib().ckv_mix_seed(cfg.seed, 0xDECADE, model.n_positions()))
    sub = kmeans_cosine(new_keys, c, seed, cfg.max_iters, cfg.metric, None, ctx)
    base = model.n_clusters
    model.centroids = np.concatenate([model.centroids.reshape(-1, D), sub.centroids])
    model.n_clusters += c
    model.labels = np.concatenate([model.labels, sub.labels + base]).astype(np.int32)
    model.iterations_used += sub.iterations_used
    model.converged = model.converged and sub.converged
    model.objective_history = sub.objective_history
    model.invocation_iterations.append(sub.iterations_used)


# --------------------------------------------------------------------------
# index + selection (selection.hpp:16-111)
# --------------------------------------------------------------------------
def build_index(model: ClusterModel, ctx: Context | None = None) -> ClusterIndex:
    """selection.hpp:29-48."""
    ctx = ctx or Context.default()
    Cn, P = model.n_clusters, model.n_positions()
    lab = torch.from_numpy(np.ascontiguousarray(model.labels, np.int32)).to(ctx.device) \
        if P else torch.zeros(1, dtype=torch.int32, device=ctx.device)
    ncl = torch.tensor([Cn], dtype=torch.int32, device=ctx.device)
    sizes = torch.zeros(max(Cn, 1), dtype=torch.int32, device=ctx.device)
    starts = torch.zeros(Cn + 1, dtype=torch.int32, device=ctx.device)
    srt = torch.zeros(max(P, 1), dtype=torch.int32, device=ctx.device)
    check(lib().ckv_build_index(ctx.h, 1, P, max(P, 1), max(Cn, 1), lab.data_ptr(),
                                ncl.data_ptr(), sizes.data_ptr(), starts.data_ptr(),
                                srt.data_ptr()))
    st = starts.cpu().numpy().view(np.uint32)
    total = int(st[Cn])
    return ClusterIndex(sizes.cpu().numpy().view(np.uint32)[:Cn],
                        srt.cpu().numpy().view(np.uint32)[:total], st)


class _DeviceModel:
    """Device copy of (centroids, index) for one unit."""

    def __init__(self, ctx: Context, model: ClusterModel, index: ClusterIndex):
        dev = ctx.device
        Cn = model.n_clusters
        self.C = Cn
        self.c_cap = max(Cn, 1)
        self.p_cap = max(model.n_positions(), 1)
        cents = np.zeros((self.c_cap, D), np.float32)
        if Cn:
            cents[:Cn] = np.asarray(model.centroids, np.float32).reshape(Cn, D)
        self.cents = torch.from_numpy(cents).to(dev)
        self.ncl = torch.tensor([Cn], dtype=torch.int32, device=dev)
        sz = np.zeros(self.c_cap, np.uint32)
        sz[:Cn] = index.sizes
        self.sizes = torch.from_numpy(sz.view(np.int32)).to(dev)
        stt = np.zeros(self.c_cap + 1, np.uint32)
        stt[: Cn + 1] = index.cluster_start[: Cn + 1]
        self.starts = torch.from_numpy(stt.view(np.int32)).to(dev)
        srt = np.zeros(self.p_cap, np.uint32)
        srt[: index.labeled_total()] = index.sorted_token_ids
        self.sorted = torch.from_numpy(srt.view(np.int32)).to(dev)


def score_clusters(q: np.ndarray, model: ClusterModel, ctx: Context | None = None) -> np.ndarray:
    """selection.hpp:51-57 (computed by the select kernel's exact f64 chains)."""
    ctx = ctx or Context.default()
    index = ClusterIndex(np.zeros(model.n_clusters, np.uint32), np.zeros(0, np.uint32),
                         np.zeros(model.n_clusters + 1, np.uint32))
    return _select(ctx, q, model, index, 1, (), want_scores=True)[1]


def _select(ctx, q, model, index, budget, recency, want_scores=False, full_rank=True):
    """full_rank=False: the decode path's selection (no full ranking: only
    the taken clusters' ranks are written)."""
    dm = _DeviceModel(ctx, model, index)
    dev = ctx.device
    q = np.ascontiguousarray(q, np.float32).reshape(1, D)
    rec = np.ascontiguousarray(recency, np.uint32) if len(recency) else np.zeros(0, np.uint32)
    sel_cap = min(dm.p_cap, budget) + model.sink_count + 1
    qd = torch.from_numpy(q).to(dev)
    tok = torch.zeros(sel_cap, dtype=torch.int32, device=dev)
    ntok = torch.zeros(1, dtype=torch.int32, device=dev)
    ntk = torch.zeros(1, dtype=torch.int32, device=dev)
    trm = torch.zeros(1, dtype=torch.int32, device=dev)
    rnk = torch.zeros(dm.c_cap, dtype=torch.int32, device=dev)
    sc = torch.zeros(dm.c_cap, dtype=torch.float64, device=dev) if want_scores else None
    desc = N.SelectDesc(1, 1, budget, model.sink_count, dm.p_cap, dm.c_cap, sel_cap, 0, 0,
                        (N.CKV_SEL_FULL_RANK if full_rank else 0) |
                        (N.CKV_SEL_SCORES if want_scores else 0), 0)
    check(lib().ckv_select(ctx.h, C.byref(desc), qd.data_ptr(), dm.cents.data_ptr(),
                           dm.ncl.data_ptr(), dm.sizes.data_ptr(), dm.starts.data_ptr(),
                           dm.sorted.data_ptr(), tok.data_ptr(), None, None, ntok.data_ptr(),
                           ntk.data_ptr(), trm.data_ptr(), rnk.data_ptr(), _ptr(sc), None))
    n = int(ntok.item())
    ids = np.concatenate([tok.cpu().numpy().view(np.uint32)[:n], rec]).astype(np.uint32)
    res = SelectionResult(rnk.cpu().numpy().view(np.uint32)[: model.n_clusters],
                          int(ntk.item()), ids, int(trm.item()), budget)
    scores = sc.cpu().numpy()[: model.n_clusters] if want_scores else None
    return res, scores


def select_tokens(q: np.ndarray, model: ClusterModel, index: ClusterIndex, budget: int,
                  recency: Sequence[int] = (), ctx: Context | None = None) -> SelectionResult:
    """selection.hpp:74-111.  The recency span is appended verbatim after the
    sinks, as the reference does (selection.hpp:109)."""
    ctx = ctx or Context.default()
    return _select(ctx, q, model, index, budget, recency)[0]


# --------------------------------------------------------------------------
# attention (attention.hpp:63-69)
# --------------------------------------------------------------------------
def approx_attention(q: np.ndarray, keys: np.ndarray, values: np.ndarray,
                     selected: Sequence[int], ctx: Context | None = None) -> AttentionOutput:
    ctx = ctx or Context.default()
    if len(selected) == 0:
        raise ValidationError(1, "approx_attention: empty selection")
    keys = np.ascontiguousarray(keys, np.float32)
    values = np.ascontiguousarray(values, np.float32)
    _check_d(keys, "approx_attention")
    sel = np.ascontiguousarray(selected, np.uint32)
    if sel.max() >= keys.shape[0]:
        raise ValidationError(1, "approx_attention: selected id out of range")
    kb = _to_bf16_device(ctx, keys, "approx_attention keys")
    vb = _to_bf16_device(ctx, values, "approx_attention values")
    dev = ctx.device
    qd = torch.from_numpy(np.ascontiguousarray(q, np.float32).reshape(1, D)).to(dev)
    ids = torch.from_numpy(sel.view(np.int32)).to(dev)
    nt = torch.tensor([len(sel)], dtype=torch.int32, device=dev)
    out = torch.empty((1, D), dtype=torch.float32, device=dev)
    w = torch.empty(len(sel), dtype=torch.float32, device=dev)
    desc = N.AttendDesc(1, 1, keys.shape[0], len(sel), len(sel))
    check(lib().ckv_attend(ctx.h, C.byref(desc), qd.data_ptr(), kb.data_ptr(), vb.data_ptr(),
                           ids.data_ptr(), None, nt.data_ptr(), out.data_ptr(), w.data_ptr()))
    return AttentionOutput(out.cpu().numpy()[0], w.cpu().numpy())


# --------------------------------------------------------------------------
# page-select baseline (selection.hpp:136-194)
# --------------------------------------------------------------------------
PAGE_MAX, PAGE_MAXMIN = 0, 1  # PageRepr


def page_select(q: np.ndarray, keys: np.ndarray, budget: int, page_size: int,
                repr: int = PAGE_MAX, ctx: Context | None = None) -> np.ndarray:
    """selection.hpp:141-194: the ids of the top min(n_pages, budget /
    page_size) pages by their representative score, ascending."""
    ctx = ctx or Context.default()
    if page_size < 1:
        raise ValidationError(1, "page_select: page_size must be >= 1")
    keys = np.ascontiguousarray(keys, np.float32)
    _check_d(keys, "page_select")
    n = keys.shape[0]
    n_pages = (n + page_size - 1) // page_size
    n_sel = min(n_pages, budget // page_size)
    if n_sel == 0:
        return np.zeros(0, np.uint32)
    kb = _to_bf16_device(ctx, keys, "page_select keys")
    dev = ctx.device
    rmax = torch.empty((n_pages, D), dtype=torch.float32, device=dev)
    rmin = torch.empty((n_pages, D), dtype=torch.float32, device=dev) if repr else None
    check(lib().ckv_page_reps(ctx.h, 1, n, n, page_size, n_pages, kb.data_ptr(),
                              rmax.data_ptr(), _ptr(rmin)))
    qd = torch.from_numpy(np.ascontiguousarray(q, np.float32).reshape(1, D)).to(dev)
    rr = torch.zeros((1, n_sel + 1), dtype=torch.int32, device=dev)
    ro = torch.zeros((1, n_sel + 2), dtype=torch.int32, device=dev)
    rc = torch.zeros(1, dtype=torch.int32, device=dev)
    runs = N.Runs(rr.data_ptr(), ro.data_ptr(), rc.data_ptr(), n_sel + 1)
    ids = torch.zeros((1, n_sel * page_size), dtype=torch.int32, device=dev)
    nt = torch.zeros(1, dtype=torch.int32, device=dev)
    desc = N.PageDesc(1, 1, n, page_size, budget, n_pages, n_sel * page_size, int(repr))
    check(lib().ckv_page_select(ctx.h, C.byref(desc), qd.data_ptr(), rmax.data_ptr(), _ptr(rmin),
                                C.byref(runs), ids.data_ptr(), nt.data_ptr()))
    k = int(nt.item())
    return ids[0, :k].cpu().numpy().view(np.uint32).copy()


# --------------------------------------------------------------------------
# cluster cache (cache.hpp:25-93)
# --------------------------------------------------------------------------
class ClusterCache:
    def __init__(self, retention: int, head_dim: int, c_cap: int = 1 << 16,
                 ctx: Context | None = None):
        self.ctx = ctx or Context.default()
        if retention < 1:
            raise ValidationError(1, "ClusterCache: retention must be >= 1")
        h = C.c_void_p()
        check(lib().ckv_cache_create(self.ctx.h, 1, c_cap, retention, head_dim, C.byref(h)))
        self.h = h
        self._retention = retention

    def __del__(self):
        try:
            lib().ckv_cache_destroy(self.h)
        except Exception:
            pass

    def lookup_and_update(self, selected: Sequence[int], sizes: Sequence[int]):
        dev = self.ctx.device
        sel = np.ascontiguousarray(selected, np.uint32)
        sz = np.ascontiguousarray(sizes, np.uint32)
        n = len(sel)
        ds = torch.from_numpy(sel.view(np.int32)).to(dev) if n else \
            torch.zeros(1, dtype=torch.int32, device=dev)
        dz = torch.from_numpy(sz.view(np.int32)).to(dev) if len(sz) else \
            torch.zeros(1, dtype=torch.int32, device=dev)
        hit = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        miss = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        counts = np.zeros(2, np.uint32)
        check(lib().ckv_cache_lookup(self.ctx.h, self.h, 0, ds.data_ptr(), n, dz.data_ptr(),
                                     hit.data_ptr(), miss.data_ptr(), counts.ctypes.data))
        return (hit.cpu().numpy().view(np.uint32)[: counts[0]],
                miss.cpu().numpy().view(np.uint32)[: counts[1]])

    def counters(self) -> dict:
        out = np.zeros(4, np.uint64)
        check(lib().ckv_cache_counters(self.h, out.ctypes.data))
        return dict(clusters_requested=int(out[0]), clusters_hit=int(out[1]),
                    tokens_transferred=int(out[2]), bytes_transferred=int(out[3]))

    def hit_rate(self) -> float:
        c = self.counters()
        if c["clusters_requested"] == 0:
            raise ValidationError(1, "ClusterCache: hit_rate with zero requests")
        return c["clusters_hit"] / c["clusters_requested"]

    def invalidate_on_recluster(self, retired: Sequence[int], fresh: Sequence[int] = ()):
        r = np.ascontiguousarray(retired, np.uint32)
        if len(r):
            check(lib().ckv_cache_invalidate(self.ctx.h, self.h, 0, r.ctypes.data, len(r)))

    def retention(self) -> int:
        return self._retention
