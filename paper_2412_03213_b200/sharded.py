"""Sequence-sharded ClusterKV path (BASELINE config E).

One very long head (70B shape, 128k context) is split into contiguous
position shards, one per rank (one process per GPU, torch.distributed over
NCCL/NVLink for the collectives).  This module is the host side of the
protocol declared in include/ckv_cuda.h ("sequence-sharded k-means"): it runs
the reference's kmeans_cosine loop (clustering.hpp:160-263) with the per-shard
device steps of ckv_kmshard.cu and one collective between them:

  per iteration: all-reduce SUM of the f64 centroid partial sums [C x 128]
                 and of the counts [C]; all-reduce MAX of a "changed" flag;
                 an all-gather of (distance, row) per empty-cluster repair.

f64 sums of bf16 keys are exact in any order, so every rank
ends with centroids, labels and iteration counts bit-identical to the
single-process reference, for any number of shards.

The local steps sit behind a small interface (`ShardSteps`): `DeviceShard`
binds the CUDA kernels through the C-ABI (the product path); the CPU tests
bind a checker built from the oracle (tests/_shard_cpu.py) to exercise this
protocol with gloo at world_size 2.  There is no CPU fallback here: nothing
in this module computes a k-means step itself.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Protocol

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from ._native import ValidationError, check, lib

D = 128


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous position shard [lo, hi) of rank `rank`."""
    return n * rank // world, n * (rank + 1) // world


# --------------------------------------------------------------------------
# collectives
# --------------------------------------------------------------------------
class Comm:
    """The collectives of the sharded path over torch.distributed.

    NCCL reduces device buffers in place over NVLink/NVSwitch.  gloo (the CPU
    tests, or several ranks sharing one GPU) only takes host tensors, so
    device buffers are staged through the host.  world_size 1 (no process
    group) makes every collective the identity.
    """

    def __init__(self, group=None):
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0
        self.stage = self.on and dist.get_backend(group) == "gloo"

    def all_reduce(self, t: torch.Tensor, op: str = "sum") -> None:
        if self.world == 1:
            return
        rop = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX}[op]
        x = t.cpu() if (self.stage and t.is_cuda) else t
        dist.all_reduce(x, op=rop, group=self.group)
        if x is not t:
            t.copy_(x)

    def all_gather(self, t: torch.Tensor) -> list[torch.Tensor]:
        if self.world == 1:
            return [t]
        x = t.cpu() if (self.stage and t.is_cuda) else t
        out = [torch.empty_like(x) for _ in range(self.world)]
        dist.all_gather(out, x.contiguous(), group=self.group)
        return out


# --------------------------------------------------------------------------
# per-shard steps
# --------------------------------------------------------------------------
class ShardSteps(Protocol):
    """One rank's device steps (ckv_kmshard_* in include/ckv_cuda.h)."""

    n_units: int
    n_local: int
    C: int
    sums: torch.Tensor       # [U][C][128] f64
    counts: torch.Tensor     # [U][C] int32
    stat: torch.Tensor       # [U][4] int32: changed, non-finite, non-zero row, 0
    objective: torch.Tensor  # [U] f64

    def validate(self) -> None: ...
    def init(self, rows: np.ndarray, row_lo: int) -> None: ...
    def set_active(self, active: np.ndarray) -> None: ...
    def update(self, from_init: bool) -> None: ...
    def assign(self, pass_: int) -> None: ...
    def empty(self) -> np.ndarray: ...
    def farthest(self, unit: int, cluster: int) -> tuple[float, int]: ...
    def move(self, unit: int, local_row: int, cluster: int) -> None: ...
    def finish(self, pass_: int, want_objective: bool) -> None: ...
    def partial_sums(self) -> None: ...
    def result(self, iters: np.ndarray) -> tuple[torch.Tensor, torch.Tensor]: ...


class DeviceShard:
    """ShardSteps on the B200 kernels (ckv_kmshard.cu) through the C-ABI.

    keys: device int16/bf16-bits tensor [n_units, n_local, 128] (this rank's
    contiguous position shard of every unit); rows must be contiguous, the
    unit stride is free, so it may be a view into the rank's KV store.
    """

    def __init__(self, keys: torch.Tensor, C_: int, ctx=None, exact_only: bool = False):
        from .api import Context
        if not keys.is_cuda:
            raise ValueError("DeviceShard: keys must be a CUDA tensor (no CPU fallback)")
        self.ctx = ctx or Context.default()
        if keys.stride(2) != 1 or keys.stride(1) != D:
            keys = keys.contiguous()
        self.keys = keys
        U, n, d = self.keys.shape
        if d != D:
            raise ValidationError(N.CKV_EINVAL, "head dim must be 128")
        self.n_units, self.n_local, self.C = U, n, C_
        dev = keys.device
        self.sums = torch.zeros((U, C_, D), dtype=torch.float64, device=dev)
        self.counts = torch.zeros((U, C_), dtype=torch.int32, device=dev)
        self.stat = torch.zeros((U, 4), dtype=torch.int32, device=dev)
        self.objective = torch.zeros((U,), dtype=torch.float64, device=dev)
        desc = N.KmShardDesc(U, n, C_, N.CKV_KM_EXACT_ONLY if exact_only else 0,
                             self.keys.stride(0))
        bufs = N.KmShardBufs(self.sums.data_ptr(), self.counts.data_ptr(),
                             self.stat.data_ptr(), self.objective.data_ptr())
        h = C.c_void_p()
        check(lib().ckv_kmshard_create(self.ctx.h, C.byref(desc), self.keys.data_ptr(),
                                       C.byref(bufs), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().ckv_kmshard_destroy(self.h)
        except Exception:
            pass

    def validate(self):
        check(lib().ckv_kmshard_validate(self.h))

    def init(self, rows, row_lo):
        r = np.ascontiguousarray(rows, np.uint32)
        check(lib().ckv_kmshard_init(self.h, r.ctypes.data_as(C.c_void_p), row_lo))

    def set_active(self, active):
        a = np.ascontiguousarray(active, np.int32)
        check(lib().ckv_kmshard_set_active(self.h, a.ctypes.data_as(C.c_void_p)))

    def update(self, from_init):
        check(lib().ckv_kmshard_update(self.h, int(from_init)))

    def assign(self, pass_):
        check(lib().ckv_kmshard_assign(self.h, pass_))

    def empty(self):
        out = np.zeros(self.n_units, np.int32)
        check(lib().ckv_kmshard_empty(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def farthest(self, unit, cluster):
        d, r = C.c_double(), C.c_int64()
        check(lib().ckv_kmshard_farthest(self.h, unit, cluster, C.byref(d), C.byref(r)))
        return d.value, r.value

    def move(self, unit, local_row, cluster):
        check(lib().ckv_kmshard_move(self.h, unit, local_row, cluster))

    def finish(self, pass_, want_objective):
        check(lib().ckv_kmshard_finish(self.h, pass_, int(want_objective)))

    def partial_sums(self):
        check(lib().ckv_kmshard_partial_sums(self.h))

    def result(self, iters):
        it = np.ascontiguousarray(iters, np.uint32)
        cents = torch.empty((self.n_units, self.C, D), dtype=torch.float32,
                            device=self.keys.device)
        labels = torch.empty((self.n_units, self.n_local), dtype=torch.int32,
                             device=self.keys.device)
        check(lib().ckv_kmshard_result(self.h, it.ctypes.data_as(C.c_void_p), cents.data_ptr(),
                                       labels.data_ptr()))
        self.ctx.sync()
        return cents, labels


# --------------------------------------------------------------------------
# the protocol (kmeans_cosine, clustering.hpp:160-263, sharded)
# --------------------------------------------------------------------------
@dataclass
class ShardedKMeansResult:
    """ClusterModel fields of every unit; labels cover this rank's shard."""

    n_clusters: int
    centroids: torch.Tensor         # [U][C][128] f32, identical on every rank
    labels: torch.Tensor            # [U][n_local] int32, this shard's positions
    row_lo: int                     # global row of labels[:, 0]
    iterations_used: np.ndarray     # [U]
    converged: np.ndarray           # [U] bool
    repair_iterations: list = field(default_factory=list)   # per unit
    objective_history: list = field(default_factory=list)   # per unit


def _init_rows(n_total: int, C_: int, seeds) -> np.ndarray:
    rows = np.zeros((len(seeds), C_), np.uint32)
    for u, s in enumerate(seeds):
        check(lib().ckv_kmeans_init_rows(n_total, C_, int(s),
                                         rows[u].ctypes.data_as(C.c_void_p)))
    return rows


def _repair(shard: ShardSteps, comm: Comm, row_lo: int, n_local: int,
            active: np.ndarray) -> np.ndarray:
    """repair_empty_clusters (clustering.hpp:128-153) over the global counts.

    Every rank holds the same all-reduced counts, so every rank takes the
    same decisions; the victim (the member of the largest cluster farthest
    from its centroid, first in position order on ties) is found by one
    all-gather of each shard's local candidate per repair."""
    U, C_ = shard.n_units, shard.C
    n_rep = np.zeros(U, np.int64)
    empty = shard.empty()
    for u in np.nonzero((empty != 0) & (active != 0))[0]:
        counts = shard.counts[u].cpu().numpy().astype(np.int64)
        for c in range(C_):
            if counts[c] > 0:
                continue
            largest = int(np.argmax(counts))  # first maximum
            if counts[largest] <= 1:
                continue
            d, r = shard.farthest(int(u), largest)
            mine = torch.tensor([d, float(row_lo + r) if r >= 0 else -1.0], dtype=torch.float64)
            best_d, victim = -1.0, -1
            for t in comm.all_gather(mine):
                dd, gg = float(t[0]), int(t[1])
                if gg >= 0 and (dd > best_d or (dd == best_d and gg < victim)):
                    best_d, victim = dd, gg
            if victim < 0:
                victim = 0  # no member beat distance -1: the reference keeps victim = 0
            if row_lo <= victim < row_lo + n_local:
                shard.move(int(u), victim - row_lo, c)
            counts[largest] -= 1
            counts[c] += 1
            n_rep[u] += 1
        shard.counts[u].copy_(torch.from_numpy(counts.astype(np.int32)))
    return n_rep


def kmeans_cosine_sharded(shard: ShardSteps, n_total: int, row_lo: int, seeds=None,
                          max_iters: int = 50, init_rows: np.ndarray | None = None,
                          comm: Comm | None = None,
                          want_objective: bool = False) -> ShardedKMeansResult:
    """kmeans_cosine (clustering.hpp:160-263) of n_units heads whose n_total
    keys are position-sharded over the ranks of `comm`; this rank holds rows
    [row_lo, row_lo + shard.n_local).  seeds[u] (or init_rows[u]) as the
    reference.  Raises ValidationError under the reference's predicates."""
    comm = comm or Comm()
    U, C_, n_local = shard.n_units, shard.C, shard.n_local
    if not 1 <= C_ <= n_total:
        raise ValidationError(N.CKV_EINVAL, "kmeans: need 1 <= C <= N")
    if max_iters < 1:
        raise ValidationError(N.CKV_EINVAL, "ClusterConfig: max_iters must be >= 1")
    shard.validate()
    comm.all_reduce(shard.stat, "max")
    st = shard.stat.cpu().numpy()
    if st[:, 1].any():
        raise ValidationError(N.CKV_EINVAL, "kmeans: keys must be finite")
    if not st[:, 2].all():
        raise ValidationError(N.CKV_EINVAL, "kmeans: degenerate input, all keys zero-norm")
    if init_rows is not None:
        rows = np.asarray(init_rows, np.uint32).reshape(U, -1)
        if rows.shape[1] != C_:
            raise ValidationError(N.CKV_EINVAL, "kmeans: init_rows size must equal C")
    else:
        rows = _init_rows(n_total, C_, seeds)

    shard.init(rows, row_lo)
    comm.all_reduce(shard.sums)
    shard.update(True)
    active = np.ones(U, np.int32)
    iters = np.zeros(U, np.uint32)
    converged = np.zeros(U, bool)
    rep_hist = [[] for _ in range(U)]
    obj_hist = [[] for _ in range(U)]

    def assign_pass(t: int) -> None:
        shard.assign(t)
        comm.all_reduce(shard.counts)
        reps = _repair(shard, comm, row_lo, n_local, active)
        shard.finish(t, want_objective)
        if t > 0:
            comm.all_reduce(shard.stat, "max")
        if want_objective:
            comm.all_reduce(shard.objective)
        objs = shard.objective.cpu().numpy() if want_objective else None
        for u in np.nonzero(active)[0]:
            if reps[u] > 0:
                rep_hist[u].append(t)
            if want_objective:
                obj_hist[u].append(float(objs[u]))

    assign_pass(0)
    for t in range(1, max_iters + 1):
        shard.partial_sums()
        comm.all_reduce(shard.sums)
        shard.update(False)
        assign_pass(t)
        changed = shard.stat[:, 0].cpu().numpy()
        for u in np.nonzero(active)[0]:
            if not changed[u]:
                converged[u], iters[u], active[u] = True, t, 0
            elif t == max_iters:
                iters[u], active[u] = t, 0
        if not active.any():
            break
        shard.set_active(active)
    cents, labels = shard.result(iters)
    return ShardedKMeansResult(C_, cents, labels, row_lo, iters, converged, rep_hist, obj_hist)


# --------------------------------------------------------------------------
# the decode step (select_tokens + approx_attention, sharded)
# --------------------------------------------------------------------------
def global_sizes(comm: Comm, lsize: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """From each rank's local cluster sizes [U][C]: the global sizes (what
    build_index over the whole head gives, selection.hpp:29-48) and this
    rank's prefix = members of each cluster on lower-ranked shards, which
    decides its share of a trimmed cluster (the reference keeps the lowest
    positions, selection.hpp:98-101).  One all-gather per prefill."""
    per_rank = [t.to(lsize.device) for t in comm.all_gather(lsize)]
    gsize = torch.stack(per_rank).sum(0).to(torch.int32).contiguous()
    prefix = (torch.stack(per_rank[: comm.rank]).sum(0).to(torch.int32)
              if comm.rank > 0 else torch.zeros_like(lsize)).contiguous()
    return gsize, prefix


def score_slice(C_: int, world: int, rank: int) -> tuple[int, int]:
    """Rank `rank` scores clusters [c_lo, c_lo + slice) (equal slices so the
    all-gathered buffer is [world][n_q][slice]; cluster c sits in rank
    c // slice at offset c % slice)."""
    slice_ = (C_ + world - 1) // world
    return slice_, rank * slice_


class ShardedDecoder:
    """One rank's share of the sequence-sharded decode step.

    Built from this rank's k-means result and its KV shard: the shard's
    clustered rows (global positions sink_tokens + row_lo ...), plus the
    sinks on the rank that holds positions [0, sink_tokens) and the recency
    window [rec_pos, rec_pos + n_rec) on the rank that holds it.  The local
    store is re-laid cluster-major by the LOCAL index, so every rank's share
    of a selected cluster is one contiguous run.

    step(q): ckv_score_range on this rank's centroid slice -> all-gather of
    the f64 scores -> ckv_select_scored (global ranking, budget and trim;
    this rank's share of I_T) -> ckv_attend_partial -> all-gather of
    (out, lse) -> ckv_attend_merge.  Every rank returns the same output.
    """

    def __init__(self, km: ShardedKMeansResult, K_store: torch.Tensor, V_store: torch.Tensor,
                 group: int, budget: int, comm: Comm | None = None, sink_rows: int = 0,
                 n_rec: int = 0, rec_pos: int = 0, sink_tokens: int = 16, ctx=None):
        """K_store / V_store: device bf16-bits [U][p_cap][128] in position
        order — rows [0, sink_rows) the sinks this rank holds, then its
        n_local shard rows, then n_rec recency rows.  Re-laid cluster-major IN
        PLACE (the decoder keeps them)."""
        from .api import Context
        self.ctx = ctx or Context.default()
        self.comm = comm or Comm()
        dev = K_store.device
        U, n_local = km.labels.shape
        self.U, self.G, self.n_q, self.C, self.B = U, group, U * group, km.n_clusters, budget
        self.sink_rows, self.n_rec, self.rec_pos = sink_rows, n_rec, rec_pos
        n_rows = sink_rows + n_local + n_rec
        if K_store.shape != V_store.shape or K_store.shape[0] != U or K_store.shape[1] < n_rows \
                or not K_store.is_contiguous() or not V_store.is_contiguous():
            raise ValueError("ShardedDecoder: K/V store must be contiguous [U][>= rows][128]")
        self.p_cap = int(K_store.shape[1])
        labels = torch.full((U, self.p_cap), -1, dtype=torch.int32, device=dev)
        labels[:, sink_rows:sink_rows + n_local] = km.labels.to(dev)
        C_ = self.C
        ncl = torch.full((U,), C_, dtype=torch.int32, device=dev)
        self.lsize = torch.zeros((U, C_), dtype=torch.int32, device=dev)
        self.lstart = torch.zeros((U, C_ + 1), dtype=torch.int32, device=dev)
        self.lsorted = torch.zeros((U, self.p_cap), dtype=torch.int32, device=dev)
        check(lib().ckv_build_index(self.ctx.h, U, n_rows, self.p_cap, C_, labels.data_ptr(),
                                    ncl.data_ptr(), self.lsize.data_ptr(),
                                    self.lstart.data_ptr(), self.lsorted.data_ptr()))
        del labels
        self.K, self.V = K_store, V_store
        check(lib().ckv_relayout_kv(self.ctx.h, U, self.p_cap, self.K.data_ptr(),
                                    self.V.data_ptr(), self.K.data_ptr(), self.V.data_ptr(),
                                    self.lsorted.data_ptr(), sink_rows, sink_rows + n_local,
                                    n_rows))
        # global sizes and the members on lower-ranked shards, once per prefill
        self.gsize, self.prefix = global_sizes(self.comm, self.lsize)
        self.cents = km.centroids.to(dev).contiguous()
        self.slice, self.c_lo = score_slice(C_, self.comm.world, self.comm.rank)
        self.pos_base = sink_tokens + km.row_lo - self.sink_rows
        self.sel_cap = budget + self.sink_rows + self.n_rec
        run_cap = C_ + 2
        nq = self.n_q
        self.run_row = torch.zeros((nq, run_cap), dtype=torch.int32, device=dev)
        self.run_off = torch.zeros((nq, run_cap + 1), dtype=torch.int32, device=dev)
        self.run_cnt = torch.zeros((nq,), dtype=torch.int32, device=dev)
        self.runs = N.Runs(self.run_row.data_ptr(), self.run_off.data_ptr(),
                           self.run_cnt.data_ptr(), run_cap)
        self.n_tokens = torch.zeros((nq,), dtype=torch.int32, device=dev)
        self.n_taken = torch.zeros((nq,), dtype=torch.int32, device=dev)
        self.trimmed = torch.zeros((nq,), dtype=torch.int32, device=dev)
        self.ranked = torch.zeros((nq, C_), dtype=torch.int32, device=dev)
        self.my_scores = torch.zeros((nq, self.slice), dtype=torch.float64, device=dev)
        self.my_approx = torch.zeros((2, nq, self.slice), dtype=torch.float32, device=dev)
        self.out_loc = torch.zeros((nq, D), dtype=torch.float32, device=dev)
        self.lse = torch.zeros((nq,), dtype=torch.float32, device=dev)
        self.sdesc = N.ShardSelectDesc(nq, group, budget, C_, C_, self.slice, self.comm.world,
                                       self.p_cap, self.sel_cap, self.sink_rows, self.sink_rows,
                                       self.sink_rows + n_local, rec_pos, self.n_rec,
                                       self.pos_base, 0)
        self.adesc = N.AttendDesc(nq, group, self.p_cap, self.sel_cap, self.sel_cap)

    def step(self, q: torch.Tensor, want_ids: bool = False, want_weights: bool = False,
             full_rank: bool = False, exact_scores: bool = False) -> dict:
        """One decode step for every q head; q: device f32 [n_q][128].

        The all-gathered scores are approximate f32 values with rigorous bounds
        (ckv_score_range_approx; the selection re-scores the few clusters near
        the budget cut exactly), or, with exact_scores, the exact f64 scores
        (ckv_score_range) — the same selection either way."""
        L, h = lib(), self.ctx.h
        q = q.contiguous()
        dev = q.device
        ids = (torch.zeros((self.n_q, self.sel_cap), dtype=torch.int32, device=dev)
               if want_ids else None)
        self.sdesc.flags = N.CKV_SEL_FULL_RANK if full_rank else 0
        common = (self.gsize.data_ptr(), self.lsize.data_ptr(), self.lstart.data_ptr(),
                  self.prefix.data_ptr(), self.lsorted.data_ptr(), C.byref(self.runs),
                  None if ids is None else ids.data_ptr(), self.n_tokens.data_ptr(),
                  self.n_taken.data_ptr(), self.trimmed.data_ptr(), self.ranked.data_ptr())
        if exact_scores:
            check(L.ckv_score_range(h, self.U, self.G, q.data_ptr(), self.cents.data_ptr(),
                                    self.C, self.C, self.c_lo, self.slice,
                                    self.my_scores.data_ptr()))
            scores = torch.stack([t.to(dev) for t in self.comm.all_gather(self.my_scores)])
            check(L.ckv_select_scored(h, C.byref(self.sdesc), scores.data_ptr(), *common))
        else:
            check(L.ckv_score_range_approx(h, self.U, self.G, q.data_ptr(), self.cents.data_ptr(),
                                           self.C, self.C, self.c_lo, self.slice,
                                           self.my_approx.data_ptr()))
            scores = torch.stack([t.to(dev) for t in self.comm.all_gather(self.my_approx)])
            check(L.ckv_select_approx(h, C.byref(self.sdesc), scores.data_ptr(), q.data_ptr(),
                                      self.cents.data_ptr(), *common))
        w = (torch.zeros((self.n_q, self.sel_cap), dtype=torch.float32, device=dev)
             if want_weights else None)
        check(L.ckv_attend_partial(h, C.byref(self.adesc), q.data_ptr(), self.K.data_ptr(),
                                   self.V.data_ptr(), C.byref(self.runs),
                                   self.n_tokens.data_ptr(), self.out_loc.data_ptr(),
                                   self.lse.data_ptr(), None if w is None else w.data_ptr()))
        outs = torch.stack([t.to(dev) for t in self.comm.all_gather(self.out_loc)]).contiguous()
        lses = torch.stack([t.to(dev) for t in self.comm.all_gather(self.lse)]).contiguous()
        out = torch.empty((self.n_q, D), dtype=torch.float32, device=dev)
        check(L.ckv_attend_merge(h, self.n_q, self.comm.world, self.comm.rank, outs.data_ptr(),
                                 lses.data_ptr(), out.data_ptr(),
                                 None if w is None else w.data_ptr(), self.n_tokens.data_ptr(),
                                 self.sel_cap))
        return dict(out=out, token_ids=ids, weights=w, n_tokens=self.n_tokens,
                    n_taken=self.n_taken, trimmed=self.trimmed, ranked=self.ranked,
                    run_off=self.run_off, run_cnt=self.run_cnt)


# --------------------------------------------------------------------------
# the native driver (ckv_comm.cu): the same protocol in C++ over NCCL, no
# torch.distributed — what a C/C++ host of the drop-in calls
# --------------------------------------------------------------------------
class NativeComm:
    """A ckv_comm: NCCL (one rank per GPU; rank 0 makes the id with
    `nccl_id()` and the caller distributes it) or LOCAL (the ranks are
    threads of this process sharing `local_group(world)`: several ranks on
    one GPU)."""

    def __init__(self, ctx=None, world: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                 group=None):
        from .api import Context
        self.ctx = ctx or Context.default()
        self.world, self.rank = world, rank
        h = C.c_void_p()
        if group is not None:
            check(lib().ckv_comm_create_local(self.ctx.h, group, rank, C.byref(h)))
        else:
            if nccl_id is None:
                if world != 1:
                    raise ValueError("NativeComm: world > 1 over NCCL needs rank 0's nccl_id")
                nccl_id = NativeComm.nccl_id()
            buf = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
            check(lib().ckv_comm_create_nccl(self.ctx.h, world, rank, buf, C.byref(h)))
        self.h = h

    @staticmethod
    def nccl_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        check(lib().ckv_comm_nccl_id(buf))
        return bytes(buf)

    @staticmethod
    def local_group(world: int):
        g = C.c_void_p()
        check(lib().ckv_local_group_create(world, C.byref(g)))
        return g

    def close(self):
        if self.h:
            lib().ckv_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kmeans_cosine_native(keys: torch.Tensor, C_: int, n_total: int, row_lo: int,
                         comm: NativeComm, seeds=None, init_rows=None, max_iters: int = 50,
                         exact_only: bool = False) -> ShardedKMeansResult:
    """kmeans_cosine_sharded through ckv_kmeans_sharded: this rank's keys
    [U][n_local][128] (device bf16 bits), rows [row_lo, row_lo + n_local) of
    every unit's n_total.  The whole loop runs in C++ (NCCL or LOCAL
    collectives); repair_iterations holds only the number of repair passes
    per unit (the C-ABI's ckv_kmeans_info.n_repair)."""
    if not keys.is_cuda:
        raise ValueError("kmeans_cosine_native: keys must be a CUDA tensor (no CPU fallback)")
    if keys.stride(2) != 1 or keys.stride(1) != D:
        keys = keys.contiguous()
    U, n_local, _ = keys.shape
    desc = N.KmShardDesc(U, n_local, C_, N.CKV_KM_EXACT_ONLY if exact_only else 0,
                         keys.stride(0))
    sd = None if seeds is None else np.ascontiguousarray(seeds, np.uint64)
    ir = None if init_rows is None else np.ascontiguousarray(init_rows, np.uint32).reshape(U, -1)
    cents = torch.empty((U, C_, D), dtype=torch.float32, device=keys.device)
    labels = torch.empty((U, n_local), dtype=torch.int32, device=keys.device)
    info = (N.KMeansInfo * U)()
    check(lib().ckv_kmeans_sharded(comm.h, C.byref(desc), keys.data_ptr(), n_total, row_lo,
                                   None if sd is None else sd.ctypes.data_as(C.c_void_p),
                                   None if ir is None else ir.ctypes.data_as(C.c_void_p),
                                   max_iters, cents.data_ptr(), labels.data_ptr(),
                                   C.cast(info, C.c_void_p)))
    iters = np.array([i.iterations_used for i in info], np.uint32)
    conv = np.array([bool(i.converged) for i in info])
    reps = [int(i.n_repair) for i in info]
    return ShardedKMeansResult(C_, cents, labels, row_lo, iters, conv, reps, [])
