"""ctypes bindings for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two interchangeable backends with one numpy-facing API:

* ``Oracle("port")``      — oracle/libckv_oracle.so, the plain-C restatement
  (oracle/ckv_oracle.c) of the reference hot path.  Always buildable (gcc).
* ``Oracle("reference")`` — oracle/_ref/libckv_ref.so, the unmodified
  reference headers (/root/reference/proj/include/clusterkv/*.hpp) behind a
  C-ABI wrapper (oracle/ref_capi.cpp).  Built only where /root/reference
  exists; the built .so travels to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module.  The product path (paper_2412_03213_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libckv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libckv_ref.so")
REF_INC = "/root/reference/proj/include"

f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def build(ref: bool | None = None) -> None:
    """make -C oracle (port always; reference when its sources are present)."""
    targets = ["all"]
    if ref or (ref is None and os.path.isdir(REF_INC)):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class OracleError(ValueError):
    """Mirrors ckv::ValidationError."""


@dataclass
class ClusterConfig:
    """clustering.hpp:20-36 defaults."""
    c0_divisor: int = 80
    c_plus: int = 4
    decode_batch: int = 320
    sink_tokens: int = 16
    max_iters: int = 50
    seed: int = 0
    c0_override: int = 0
    metric: int = 0  # 0 cosine, 1 l2, 2 inner product

    def packed(self) -> np.ndarray:
        return np.array([self.c0_divisor, self.c_plus, self.decode_batch, self.sink_tokens,
                         self.max_iters, self.c0_override, self.metric], dtype=np.uint32)


class _OrcCfg(C.Structure):
    _fields_ = [("c0_divisor", C.c_uint32), ("c_plus", C.c_uint32),
                ("decode_batch", C.c_uint32), ("sink_tokens", C.c_uint32),
                ("max_iters", C.c_uint32), ("seed", C.c_uint64),
                ("c0_override", C.c_uint32), ("metric", C.c_int32)]


class _OrcInfo(C.Structure):
    _fields_ = [("n_clusters", C.c_uint32), ("iterations_used", C.c_uint32),
                ("converged", C.c_int32), ("n_objective", C.c_uint32),
                ("n_repair", C.c_uint32)]


class _OrcSpec(C.Structure):
    _fields_ = [("n_centers", C.c_uint32), ("center_spread", C.c_float),
                ("intra_spread", C.c_float), ("query_drift", C.c_float),
                ("seed", C.c_uint64), ("prompt_len", C.c_uint32),
                ("decode_len", C.c_uint32), ("d", C.c_uint32),
                ("n_layers", C.c_uint32), ("n_heads", C.c_uint32)]


@dataclass
class KMeansResult:
    centroids: np.ndarray
    labels: np.ndarray
    converged: bool
    iterations_used: int
    objective_history: np.ndarray
    repair_iterations: np.ndarray
    sink_count: int = 0
    n_clusters: int = 0


@dataclass
class Selection:
    ranked_clusters: np.ndarray
    n_clusters_taken: int
    token_ids: np.ndarray
    trimmed_from_last: int
    budget: int

    @property
    def taken_clusters(self) -> np.ndarray:
        return self.ranked_clusters[: self.n_clusters_taken]


@dataclass
class Trace:
    prompt_keys: np.ndarray
    prompt_values: np.ndarray
    decode_queries: np.ndarray
    decode_keys: np.ndarray
    decode_values: np.ndarray


def _cfg_struct(cfg: ClusterConfig) -> _OrcCfg:
    return _OrcCfg(cfg.c0_divisor, cfg.c_plus, cfg.decode_batch, cfg.sink_tokens,
                   cfg.max_iters, cfg.seed, cfg.c0_override, cfg.metric)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            build(ref=(kind == "reference"))
        self.lib = C.CDLL(path)
        self._bind()

    # -- binding ---------------------------------------------------------
    def _bind(self):
        L = self.lib
        if self.kind == "port":
            L.orc_last_error.restype = C.c_char_p
            L.orc_mix_seed.restype = C.c_uint64
            L.orc_mix_seed.argtypes = [C.c_uint64] * 3
            L.orc_kmeans.argtypes = [f32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                     C.c_uint32, C.c_int, C.c_void_p, C.c_uint32, f32p, i32p,
                                     f64p, u32p, C.POINTER(_OrcInfo)]
            L.orc_kmeans_init_rows.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p]
            L.orc_assign.argtypes = [f32p, C.c_uint32, C.c_uint32, C.c_int, f32p, C.c_uint32,
                                     i32p]
            L.orc_cosine_distance.restype = C.c_double
            L.orc_cosine_distance.argtypes = [f32p, f32p, C.c_uint32]
            L.orc_prefill_cluster_count.restype = C.c_uint32
            L.orc_prefill_cluster_count.argtypes = [C.c_uint32, C.POINTER(_OrcCfg)]
            L.orc_cluster_prefill.argtypes = [f32p, C.c_uint32, C.c_uint32, C.POINTER(_OrcCfg),
                                              f32p, i32p, f64p, u32p, C.POINTER(_OrcInfo),
                                              C.POINTER(C.c_uint32)]
            L.orc_cluster_decode_batch.argtypes = [f32p, C.POINTER(C.c_uint32), i32p,
                                                   C.POINTER(C.c_uint32), f32p, C.c_uint32,
                                                   C.c_uint32, C.POINTER(_OrcCfg),
                                                   C.POINTER(C.c_uint32), C.POINTER(C.c_int32)]
            L.orc_build_index.argtypes = [i32p, C.c_uint32, C.c_uint32, u32p, u32p, u32p]
            L.orc_score_clusters.argtypes = [f32p, f32p, C.c_uint32, C.c_uint32, f64p]
            L.orc_select_tokens.restype = C.c_uint32
            L.orc_select_tokens.argtypes = [f32p, f32p, C.c_uint32, C.c_uint32, u32p, u32p, u32p,
                                            C.c_uint32, C.c_uint32, u32p, C.c_uint32, u32p,
                                            C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), u32p]
            L.orc_exact_topb.argtypes = [f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32, u32p]
            L.orc_page_select.restype = C.c_uint32
            L.orc_page_select.argtypes = [f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_int, u32p]
            L.orc_attention_over.argtypes = [f32p, f32p, f32p, C.c_uint32, u32p, C.c_uint32,
                                             f32p, C.c_void_p]
            L.orc_cache_new.restype = C.c_void_p
            L.orc_cache_new.argtypes = [C.c_uint32, C.c_uint32]
            L.orc_cache_free.argtypes = [C.c_void_p]
            L.orc_cache_lookup_and_update.argtypes = [C.c_void_p, u32p, C.c_uint32, u32p, u32p,
                                                      C.POINTER(C.c_uint32), u32p,
                                                      C.POINTER(C.c_uint32)]
            L.orc_cache_counters.argtypes = [C.c_void_p, u64p]
            L.orc_cache_invalidate.argtypes = [C.c_void_p, u32p, C.c_uint32]
            L.orc_generate_head.argtypes = [C.POINTER(_OrcSpec), C.c_uint64, f32p, f32p, f32p,
                                            f32p, f32p]
            L.orc_generate_synthetic.argtypes = [C.POINTER(_OrcSpec), C.c_uint32, f32p, f32p,
                                                 f32p, f32p, f32p]
        else:
            L.ref_last_error.restype = C.c_char_p
            L.ref_mix_seed.restype = C.c_uint64
            L.ref_mix_seed.argtypes = [C.c_uint64] * 3
            L.ref_generate_head.argtypes = [C.c_uint32, C.c_float, C.c_float, C.c_float,
                                            C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                            f32p, f32p, f32p, f32p, f32p]
            L.ref_kmeans.argtypes = [f32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                     C.c_uint32, C.c_int, C.c_void_p, C.c_uint32, f32p, i32p,
                                     f64p, u32p, u32p]
            L.ref_prefill_cluster_count.restype = C.c_uint32
            L.ref_prefill_cluster_count.argtypes = [C.c_uint32, u32p]
            L.ref_cluster_prefill.argtypes = [f32p, C.c_uint32, C.c_uint32, u32p, C.c_uint64,
                                              f32p, i32p, f64p, u32p, u32p]
            L.ref_cluster_decode_batch.argtypes = [f32p, C.POINTER(C.c_uint32), i32p,
                                                   C.POINTER(C.c_uint32), f32p, C.c_uint32,
                                                   C.c_uint32, u32p, C.c_uint64,
                                                   C.POINTER(C.c_uint32)]
            L.ref_build_index.argtypes = [i32p, C.c_uint32, C.c_uint32, u32p, u32p, u32p]
            L.ref_score_clusters.argtypes = [f32p, f32p, C.c_uint32, C.c_uint32, f64p]
            L.ref_select_tokens.restype = C.c_uint32
            L.ref_select_tokens.argtypes = [f32p, f32p, C.c_uint32, C.c_uint32, i32p, C.c_uint32,
                                            C.c_uint32, C.c_uint32, u32p, C.c_uint32, u32p,
                                            C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), u32p]
            L.ref_approx_attention.argtypes = [f32p, f32p, f32p, C.c_uint32, C.c_uint32, u32p,
                                               C.c_uint32, f32p, C.c_void_p]
            L.ref_cache_new.restype = C.c_void_p
            L.ref_cache_new.argtypes = [C.c_uint32, C.c_uint32]
            L.ref_cache_free.argtypes = [C.c_void_p]
            L.ref_cache_lookup_and_update.argtypes = [C.c_void_p, u32p, C.c_uint32, u32p,
                                                      C.c_uint32, u32p, C.POINTER(C.c_uint32),
                                                      u32p, C.POINTER(C.c_uint32)]
            L.ref_cache_counters.argtypes = [C.c_void_p, u64p]
            L.ref_cache_invalidate.argtypes = [C.c_void_p, u32p, C.c_uint32]
            L.ref_run_simulation_synth.restype = C.c_long
            L.ref_run_simulation_synth.argtypes = (
                [C.c_uint32, C.c_uint64] + [C.c_uint32] * 8 + [C.c_int, C.c_uint32, C.c_int] +
                [f64p, u64p, f64p, u64p, u32p, C.c_uint32])
            L.ref_decode_step_cpu.restype = C.c_double
            L.ref_decode_step_cpu.argtypes = [f32p, u32p, C.c_uint32, C.c_void_p, u32p,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                              C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                              C.c_uint32, C.c_uint32, f32p]
            L.ref_prefill_cpu.restype = C.c_double
            L.ref_prefill_cpu.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, u64p,
                                          C.c_uint32, C.c_uint32, u64p]
            L.ref_hardware_concurrency.restype = C.c_uint
            L.ref_write_synthetic_trace.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64,
                                                    C.c_uint32, C.c_uint32, C.c_uint32,
                                                    C.c_uint32, C.c_uint32]
            L.ref_read_trace_status.argtypes = [C.c_char_p]
            L.ref_page_select.restype = C.c_int64
            L.ref_page_select.argtypes = [f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_int, u32p]

    def _err(self) -> str:
        f = self.lib.orc_last_error if self.kind == "port" else self.lib.ref_last_error
        return f().decode()

    # -- API -------------------------------------------------------------
    def mix_seed(self, seed: int, a: int, b: int = 0) -> int:
        f = self.lib.orc_mix_seed if self.kind == "port" else self.lib.ref_mix_seed
        return int(f(seed, a, b))

    def generate_head(self, sub_seed: int, L: int, T: int, d: int = 128, n_centers: int = 8,
                      center_spread: float = 1.0, intra_spread: float = 0.15,
                      query_drift: float = 0.15) -> Trace:
        pk = np.empty((L, d), np.float32)
        pv = np.empty((L, d), np.float32)
        dq = np.empty((T, d), np.float32)
        dk = np.empty((T, d), np.float32)
        dv = np.empty((T, d), np.float32)
        if self.kind == "port":
            spec = _OrcSpec(n_centers, center_spread, intra_spread, query_drift, 0, L, T, d, 1, 1)
            self.lib.orc_generate_head(C.byref(spec), sub_seed, pk, pv, dq, dk, dv)
        else:
            self.lib.ref_generate_head(n_centers, center_spread, intra_spread, query_drift,
                                       L, T, d, sub_seed, pk, pv, dq, dk, dv)
        return Trace(pk, pv, dq, dk, dv)

    def generate_synthetic(self, seed: int, n_layers: int, n_heads: int, L: int, T: int,
                           d: int = 128, n_threads: int | None = None) -> Trace:
        """All traces, layer-major [n_layers*n_heads, ...] (port backend only)."""
        assert self.kind == "port"
        U = n_layers * n_heads
        pk = np.empty((U, L, d), np.float32)
        pv = np.empty((U, L, d), np.float32)
        dq = np.empty((U, T, d), np.float32)
        dk = np.empty((U, T, d), np.float32)
        dv = np.empty((U, T, d), np.float32)
        spec = _OrcSpec(8, 1.0, 0.15, 0.15, seed, L, T, d, n_layers, n_heads)
        self.lib.orc_generate_synthetic(C.byref(spec), n_threads or os.cpu_count() or 1,
                                        pk, pv, dq, dk, dv)
        return Trace(pk, pv, dq, dk, dv)

    def kmeans(self, keys: np.ndarray, C_: int, seed: int, max_iters: int = 50,
               metric: int = 0, init_rows: np.ndarray | None = None) -> KMeansResult:
        keys = np.ascontiguousarray(keys, np.float32)
        n, d = keys.shape
        cents = np.zeros((max(C_, 1), d), np.float32)
        labels = np.zeros(n, np.int32)
        obj = np.zeros(max_iters + 2, np.float64)
        reps = np.zeros(max_iters + 2, np.uint32)
        ir = None if init_rows is None else np.ascontiguousarray(init_rows, np.uint32)
        ir_ptr = None if ir is None else ir.ctypes.data_as(C.c_void_p)
        n_ir = 0 if ir is None else len(ir)
        if self.kind == "port":
            info = _OrcInfo()
            rc = self.lib.orc_kmeans(keys, n, d, C_, seed, max_iters, metric, ir_ptr, n_ir,
                                     cents, labels, obj, reps, C.byref(info))
            if rc:
                raise OracleError(self._err())
            return KMeansResult(cents[:C_], labels, bool(info.converged), info.iterations_used,
                                obj[: info.n_objective], reps[: info.n_repair], 0, C_)
        info = np.zeros(6, np.uint32)
        rc = self.lib.ref_kmeans(keys, n, d, C_, seed, max_iters, metric, ir_ptr, n_ir, cents,
                                 labels, obj, reps, info)
        if rc:
            raise OracleError(self._err())
        return KMeansResult(cents[:C_], labels, bool(info[2]), int(info[1]), obj[: info[3]],
                            reps[: info[4]], 0, C_)

    def assign(self, keys: np.ndarray, centroids: np.ndarray) -> np.ndarray:
        """AssignScorer::assign (cosine) of every key row (clustering.hpp:70-115)."""
        assert self.kind == "port"
        keys = np.ascontiguousarray(keys, np.float32)
        cents = np.ascontiguousarray(centroids, np.float32)
        out = np.zeros(len(keys), np.int32)
        self.lib.orc_assign(keys, len(keys), keys.shape[1], 0, cents, len(cents), out)
        return out

    def cosine_distance(self, a: np.ndarray, b: np.ndarray) -> float:
        """cosine_distance (clustering.hpp:59-65)."""
        assert self.kind == "port"
        a = np.ascontiguousarray(a, np.float32)
        return float(self.lib.orc_cosine_distance(a, np.ascontiguousarray(b, np.float32),
                                                  len(a)))

    def kmeans_init_rows(self, n: int, C_: int, seed: int) -> np.ndarray:
        assert self.kind == "port"
        out = np.zeros(C_, np.uint32)
        self.lib.orc_kmeans_init_rows(n, C_, seed, out)
        return out

    def prefill_cluster_count(self, L: int, cfg: ClusterConfig) -> int:
        if self.kind == "port":
            s = _cfg_struct(cfg)
            return int(self.lib.orc_prefill_cluster_count(L, C.byref(s)))
        return int(self.lib.ref_prefill_cluster_count(L, cfg.packed()))

    def cluster_prefill(self, keys: np.ndarray, cfg: ClusterConfig) -> KMeansResult:
        keys = np.ascontiguousarray(keys, np.float32)
        L, d = keys.shape
        c0 = max(self.prefill_cluster_count(L, cfg), 1)
        cents = np.zeros((c0, d), np.float32)
        labels = np.zeros(L, np.int32)
        obj = np.zeros(cfg.max_iters + 2, np.float64)
        reps = np.zeros(cfg.max_iters + 2, np.uint32)
        if self.kind == "port":
            info = _OrcInfo()
            sink = C.c_uint32()
            s = _cfg_struct(cfg)
            rc = self.lib.orc_cluster_prefill(keys, L, d, C.byref(s), cents, labels, obj, reps,
                                              C.byref(info), C.byref(sink))
            if rc:
                raise OracleError(self._err())
            nc = info.n_clusters
            return KMeansResult(cents[:nc], labels, bool(info.converged), info.iterations_used,
                                obj[: info.n_objective], reps[: info.n_repair], sink.value, nc)
        info = np.zeros(6, np.uint32)
        rc = self.lib.ref_cluster_prefill(keys, L, d, cfg.packed(), cfg.seed, cents, labels, obj,
                                          reps, info)
        if rc:
            raise OracleError(self._err())
        nc = int(info[0])
        return KMeansResult(cents[:nc], labels, bool(info[2]), int(info[1]), obj[: info[3]],
                            reps[: info[4]], int(info[5]), nc)

    def cluster_decode_batch(self, centroids: np.ndarray, labels: np.ndarray,
                             new_keys: np.ndarray, cfg: ClusterConfig):
        """Returns (centroids', labels', iterations) — the grown model."""
        new_keys = np.ascontiguousarray(new_keys, np.float32)
        rows, d = new_keys.shape
        nc0, np0 = centroids.shape[0], labels.shape[0]
        cents = np.zeros((nc0 + cfg.c_plus, d), np.float32)
        cents[:nc0] = centroids
        lab = np.zeros(np0 + rows, np.int32)
        lab[:np0] = labels
        ncl, npos, it = C.c_uint32(nc0), C.c_uint32(np0), C.c_uint32(0)
        if self.kind == "port":
            s = _cfg_struct(cfg)
            conv = C.c_int32(0)
            rc = self.lib.orc_cluster_decode_batch(cents, C.byref(ncl), lab, C.byref(npos),
                                                   new_keys, rows, d, C.byref(s), C.byref(it),
                                                   C.byref(conv))
        else:
            rc = self.lib.ref_cluster_decode_batch(cents, C.byref(ncl), lab, C.byref(npos),
                                                   new_keys, rows, d, cfg.packed(), cfg.seed,
                                                   C.byref(it))
        if rc:
            raise OracleError(self._err())
        return cents[: ncl.value], lab[: npos.value], int(it.value)

    def build_index(self, labels: np.ndarray, C_: int):
        labels = np.ascontiguousarray(labels, np.int32)
        n = len(labels)
        sizes = np.zeros(max(C_, 1), np.uint32)
        starts = np.zeros(C_ + 1, np.uint32)
        sorted_ids = np.zeros(max(n, 1), np.uint32)
        f = self.lib.orc_build_index if self.kind == "port" else self.lib.ref_build_index
        f(labels, n, C_, sizes, starts, sorted_ids)
        return sizes[:C_], starts, sorted_ids[: int(starts[C_])]

    def score_clusters(self, q: np.ndarray, centroids: np.ndarray) -> np.ndarray:
        q = np.ascontiguousarray(q, np.float32)
        cents = np.ascontiguousarray(centroids, np.float32)
        out = np.zeros(max(cents.shape[0], 1), np.float64)
        f = self.lib.orc_score_clusters if self.kind == "port" else self.lib.ref_score_clusters
        f(q, cents, cents.shape[0], cents.shape[1], out)
        return out[: cents.shape[0]]

    def select_tokens(self, q: np.ndarray, centroids: np.ndarray, labels: np.ndarray,
                      sink_count: int, budget: int,
                      recency: np.ndarray | None = None) -> Selection:
        q = np.ascontiguousarray(q, np.float32)
        cents = np.ascontiguousarray(centroids, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        C_, d = cents.shape
        rec = np.ascontiguousarray(recency if recency is not None else np.zeros(0), np.uint32)
        ranked = np.zeros(max(C_, 1), np.uint32)
        n_labeled = int((labels >= 0).sum())
        out = np.zeros(min(n_labeled, budget) + sink_count + len(rec) + 1, np.uint32)
        nt, tr = C.c_uint32(), C.c_uint32()
        if self.kind == "port":
            sizes, starts, sorted_ids = self.build_index(labels, C_)
            n = self.lib.orc_select_tokens(q, cents, C_, d, np.ascontiguousarray(sizes),
                                           starts, np.ascontiguousarray(sorted_ids)
                                           if len(sorted_ids) else np.zeros(1, np.uint32),
                                           sink_count, budget, rec if len(rec) else
                                           np.zeros(1, np.uint32), len(rec), ranked,
                                           C.byref(nt), C.byref(tr), out)
        else:
            n = self.lib.ref_select_tokens(q, cents, C_, d, labels, len(labels), sink_count,
                                           budget, rec if len(rec) else np.zeros(1, np.uint32),
                                           len(rec), ranked, C.byref(nt), C.byref(tr), out)
        return Selection(ranked[:C_], nt.value, out[:n], tr.value, budget)

    def exact_topb(self, q, keys, budget):
        assert self.kind == "port"
        keys = np.ascontiguousarray(keys, np.float32)
        out = np.zeros(min(budget, keys.shape[0]), np.uint32)
        self.lib.orc_exact_topb(np.ascontiguousarray(q, np.float32), keys, keys.shape[0],
                                keys.shape[1], budget, out)
        return out

    def page_select(self, q, keys, budget: int, page_size: int, maxmin: bool = False):
        """page_select (selection.hpp:141-194): sorted token ids."""
        q = np.ascontiguousarray(q, np.float32)
        keys = np.ascontiguousarray(keys, np.float32)
        n, d = keys.shape
        n_pages = (n + page_size - 1) // page_size if page_size else 0
        out = np.zeros(max(1, min(n_pages, budget // max(page_size, 1)) * max(page_size, 1)),
                       np.uint32)
        if self.kind == "port":
            k = self.lib.orc_page_select(q, keys, n, d, budget, page_size, int(maxmin), out)
            if k == 0xFFFFFFFF:
                raise OracleError(self._err())
        else:
            k = self.lib.ref_page_select(q, keys, n, d, budget, page_size, int(maxmin), out)
            if k < 0:
                raise OracleError(self._err())
        return out[:k]

    def approx_attention(self, q, K, V, rows, want_weights: bool = True):
        q = np.ascontiguousarray(q, np.float32)
        K = np.ascontiguousarray(K, np.float32)
        V = np.ascontiguousarray(V, np.float32)
        rows = np.ascontiguousarray(rows, np.uint32)
        d = K.shape[1]
        out = np.zeros(d, np.float32)
        w = np.zeros(max(len(rows), 1), np.float32)
        wp = w.ctypes.data_as(C.c_void_p) if want_weights else None
        r = rows if len(rows) else np.zeros(1, np.uint32)
        if self.kind == "port":
            rc = self.lib.orc_attention_over(q, K, V, d, r, len(rows), out, wp)
        else:
            rc = self.lib.ref_approx_attention(q, K, V, K.shape[0], d, r, len(rows), out, wp)
        if rc:
            raise OracleError(self._err())
        return out, w[: len(rows)]

    def run_simulation_synth(self, spec: dict, budget: int, retention: int = 1,
                             decode_batch: int = 320, c0_divisor: int = 80,
                             async_clustering: bool = False, async_delay: int = 8,
                             recency_window: bool = True) -> dict:
        """The reference harness (run_simulation, harness.hpp:362-410; ClusterKV
        policy) on generate_synthetic(spec) rounded to bf16.  Reference only."""
        assert self.kind == "reference"
        n_rows = spec["n_layers"] * spec["n_heads"] * spec["T"]
        rows_f = np.zeros((n_rows, 3), np.float64)
        rows_u = np.zeros((n_rows, 6), np.uint64)
        summ_f = np.zeros(4, np.float64)
        summ_u = np.zeros(2, np.uint64)
        hist = np.zeros(64, np.uint32)
        n = self.lib.ref_run_simulation_synth(
            spec["n_centers"], spec["seed"], spec["L"], spec["T"], spec["n_layers"],
            spec["n_heads"], budget, retention, decode_batch, c0_divisor, int(async_clustering),
            async_delay, int(recency_window), rows_f, rows_u, summ_f, summ_u, hist, len(hist))
        if n < 0:
            raise OracleError(self._err())
        return dict(rows_f=rows_f[:n], rows_u=rows_u[:n], summ_f=summ_f, summ_u=summ_u,
                    hist=hist)

    def cache(self, retention: int, d: int = 128) -> "OracleCache":
        return OracleCache(self, retention, d)


class OracleCache:
    """cache.hpp:25-93 ClusterCache."""

    def __init__(self, o: Oracle, retention: int, d: int):
        if retention < 1:
            raise OracleError("ClusterCache: retention must be >= 1")
        self.o = o
        self.h = (o.lib.orc_cache_new if o.kind == "port" else o.lib.ref_cache_new)(retention, d)

    def __del__(self):
        try:
            (self.o.lib.orc_cache_free if self.o.kind == "port" else self.o.lib.ref_cache_free)(self.h)
        except Exception:
            pass

    def lookup_and_update(self, selected, sizes):
        sel = np.ascontiguousarray(selected, np.uint32)
        sizes = np.ascontiguousarray(sizes, np.uint32)
        n = len(sel)
        hit = np.zeros(max(n, 1), np.uint32)
        miss = np.zeros(max(n, 1), np.uint32)
        nh, nm = C.c_uint32(), C.c_uint32()
        s = sel if n else np.zeros(1, np.uint32)
        z = sizes if len(sizes) else np.zeros(1, np.uint32)
        if self.o.kind == "port":
            self.o.lib.orc_cache_lookup_and_update(self.h, s, n, z, hit, C.byref(nh), miss,
                                                   C.byref(nm))
        else:
            self.o.lib.ref_cache_lookup_and_update(self.h, s, n, z, len(sizes), hit, C.byref(nh),
                                                   miss, C.byref(nm))
        return hit[: nh.value], miss[: nm.value]

    def invalidate_on_recluster(self, retired, fresh=()):
        """cache.hpp:65-76: drop retired ids from every retained set."""
        r = np.ascontiguousarray(retired, np.uint32)
        if len(r):
            (self.o.lib.orc_cache_invalidate if self.o.kind == "port"
             else self.o.lib.ref_cache_invalidate)(self.h, r, len(r))

    def counters(self) -> np.ndarray:
        out = np.zeros(4, np.uint64)
        (self.o.lib.orc_cache_counters if self.o.kind == "port"
         else self.o.lib.ref_cache_counters)(self.h, out)
        return out


def to_bf16_representable(x: np.ndarray) -> np.ndarray:
    """Round f32 -> bf16 (RNE) -> f32, SURVEY §8a N1 (identical inputs)."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    r = ((u + rounding) >> 16) << 16
    # NaN/Inf pass through unchanged (not produced by the generator)
    out = r.astype(np.uint32).view(np.float32)
    return out.reshape(x.shape)
