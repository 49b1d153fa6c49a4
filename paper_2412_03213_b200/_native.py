"""ctypes binding of libckv_b200.so (include/ckv_cuda.h).

There is no fallback: if the CUDA library is missing or fails to load, this
module raises, so no caller can silently run anything but the sm_100a path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CKV_LIB: load an experiment build instead (tools/build_variant.py); the
# product build is libckv_b200.so next to this file
LIB_PATH = os.environ.get("CKV_LIB") or os.path.join(_HERE, "libckv_b200.so")

CKV_OK, CKV_EINVAL, CKV_ECUDA, CKV_ENOMEM, CKV_ENCCL = 0, 1, 2, 3, 4
CKV_KM_OBJECTIVE, CKV_KM_EXACT_ONLY, CKV_KM_NO_VALIDATE = 1, 2, 4
CKV_SEL_FULL_RANK, CKV_SEL_SCORES = 1, 2
CKV_SESSION_TOKEN_IDS = 0x100
CKV_SESSION_L2_PERSIST = 0x200
CKV_SESSION_TIERED = 0x800
CKV_SESSION_TIER_HOST = 0x1000
CKV_SEL_L2_PERSIST = 4

vp, u32, u64, i32, f32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32, C.c_float


class KMeansDesc(C.Structure):
    _fields_ = [("n_units", u32), ("n", u32), ("C", u32), ("max_iters", u32),
                ("key_stride", u64), ("c_stride", u32), ("label_stride", u32), ("flags", u32)]


class KMeansInfo(C.Structure):
    _fields_ = [("iterations_used", u32), ("converged", i32), ("n_repair", u32),
                ("n_objective", u32)]


class PrefillDesc(C.Structure):
    _fields_ = [("n_units", u32), ("L", u32), ("p_cap", u32), ("c_cap", u32),
                ("c0_divisor", u32), ("sink_tokens", u32), ("max_iters", u32),
                ("c0_override", u32), ("flags", u32)]


class DecodeClusterDesc(C.Structure):
    _fields_ = [("n_units", u32), ("pos0", u32), ("rows", u32), ("p_cap", u32),
                ("c_cap", u32), ("c_plus", u32), ("max_iters", u32)]


class SelectDesc(C.Structure):
    _fields_ = [("n_q", u32), ("group", u32), ("budget", u32), ("sink_count", u32),
                ("p_cap", u32), ("c_cap", u32), ("sel_cap", u32), ("rec_begin", u32),
                ("rec_end", u32), ("flags", u32), ("row_base", u32)]


class Runs(C.Structure):
    _fields_ = [("row", C.c_void_p), ("off", C.c_void_p), ("count", C.c_void_p),
                ("run_cap", u32)]


class AttendDesc(C.Structure):
    _fields_ = [("n_q", u32), ("group", u32), ("p_cap", u32), ("sel_cap", u32),
                ("max_tokens", u32)]


class SessionDesc(C.Structure):
    _fields_ = [("n_units", u32), ("group", u32), ("prompt_len", u32), ("max_decode", u32),
                ("budget", u32), ("retention", u32), ("c0_divisor", u32), ("c_plus", u32),
                ("decode_batch", u32), ("sink_tokens", u32), ("max_iters", u32),
                ("cluster_seed", u64), ("kv_heads", u32), ("flags", u32),
                ("async_delay", u32), ("c0_override", u32)]


class KmShardDesc(C.Structure):
    _fields_ = [("n_units", u32), ("n_local", u32), ("C", u32), ("flags", u32),
                ("key_stride", u64)]


class KmShardBufs(C.Structure):
    _fields_ = [("sums", vp), ("counts", vp), ("stat", vp), ("objective", vp)]


class ShardSelectDesc(C.Structure):
    _fields_ = [(n, u32) for n in ("n_q", "group", "budget", "C", "c_cap", "slice", "world",
                                   "n_local", "sel_cap", "row_base", "sink_rows", "rec_row",
                                   "rec_pos", "n_rec", "pos_base", "flags")]


class PageDesc(C.Structure):
    _fields_ = [(n, u32) for n in ("n_q", "group", "n", "page_size", "budget", "pages_cap",
                                   "sel_cap", "maxmin")]


class SessionStats(C.Structure):
    _fields_ = [("n_ctx", u32), ("labeled_end", u32), ("steps", u32), ("max_clusters", u32),
                ("launches", u64)]


# every symbol declared in include/ckv_cuda.h, with its ctypes signature
SIGNATURES = {
    "ckv_ctx_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
    "ckv_ctx_destroy": (C.c_int, [vp]),
    "ckv_ctx_sync": (C.c_int, [vp]),
    "ckv_ctx_stream": (vp, [vp]),
    "ckv_last_error": (C.c_char_p, []),
    "ckv_ctx_launch_count": (u64, [vp]),
    "ckv_malloc": (C.c_int, [vp, C.POINTER(vp), C.c_size_t]),
    "ckv_free": (C.c_int, [vp, vp]),
    "ckv_memcpy_h2d": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "ckv_memcpy_d2h": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "ckv_memset": (C.c_int, [vp, vp, C.c_int, C.c_size_t]),
    "ckv_f32_to_bf16": (C.c_int, [vp, vp, vp, C.c_size_t, C.POINTER(C.c_int)]),
    "ckv_kmeans_init_rows": (C.c_int, [u32, u32, u64, vp]),
    "ckv_mix_seed": (u64, [u64, u64, u64]),
    "ckv_kmeans": (C.c_int, [vp, C.POINTER(KMeansDesc), vp, vp, vp, vp, vp, vp, vp]),
    "ckv_prefill_cluster_count": (u32, [u32, u32, u32, u32]),
    "ckv_cluster_prefill": (C.c_int, [vp, C.POINTER(PrefillDesc), vp, vp, vp, vp, vp, vp, vp, vp]),
    "ckv_cluster_decode_batch": (C.c_int, [vp, C.POINTER(DecodeClusterDesc), vp, vp, vp, vp, vp,
                                           vp]),
    "ckv_kmshard_create": (C.c_int, [vp, C.POINTER(KmShardDesc), vp, C.POINTER(KmShardBufs),
                                     C.POINTER(vp)]),
    "ckv_kmshard_destroy": (C.c_int, [vp]),
    "ckv_kmshard_validate": (C.c_int, [vp]),
    "ckv_kmshard_init": (C.c_int, [vp, vp, u64]),
    "ckv_kmshard_set_active": (C.c_int, [vp, vp]),
    "ckv_kmshard_update": (C.c_int, [vp, C.c_int]),
    "ckv_kmshard_assign": (C.c_int, [vp, u32]),
    "ckv_kmshard_empty": (C.c_int, [vp, vp]),
    "ckv_kmshard_farthest": (C.c_int, [vp, u32, u32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_int64)]),
    "ckv_kmshard_move": (C.c_int, [vp, u32, u32, u32]),
    "ckv_kmshard_finish": (C.c_int, [vp, u32, C.c_int]),
    "ckv_kmshard_partial_sums": (C.c_int, [vp]),
    "ckv_kmshard_result": (C.c_int, [vp, vp, vp, vp]),
    "ckv_comm_nccl_id": (C.c_int, [vp]),
    "ckv_comm_create_nccl": (C.c_int, [vp, C.c_int, C.c_int, vp, C.POINTER(vp)]),
    "ckv_local_group_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "ckv_local_group_destroy": (C.c_int, [vp]),
    "ckv_comm_create_local": (C.c_int, [vp, vp, C.c_int, C.POINTER(vp)]),
    "ckv_comm_destroy": (C.c_int, [vp]),
    "ckv_comm_world": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ckv_comm_allreduce": (C.c_int, [vp, vp, C.c_size_t, C.c_int, C.c_int]),
    "ckv_comm_allgather": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "ckv_kmeans_sharded": (C.c_int, [vp, C.POINTER(KmShardDesc), vp, u64, u64, vp, vp, u32, vp,
                                     vp, vp]),
    "ckv_relayout_kv": (C.c_int, [vp, u32, u32, vp, vp, vp, vp, vp, u32, u32, u32]),
    "ckv_score_range": (C.c_int, [vp, u32, u32, vp, vp, u32, u32, u32, u32, vp]),
    "ckv_select_scored": (C.c_int, [vp, C.POINTER(ShardSelectDesc), vp, vp, vp, vp, vp, vp,
                                    C.POINTER(Runs), vp, vp, vp, vp, vp]),
    "ckv_score_range_approx": (C.c_int, [vp, u32, u32, vp, vp, u32, u32, u32, u32, vp]),
    "ckv_select_approx": (C.c_int, [vp, C.POINTER(ShardSelectDesc), vp, vp, vp, vp, vp, vp, vp,
                                    vp, C.POINTER(Runs), vp, vp, vp, vp, vp]),
    "ckv_attend_partial": (C.c_int, [vp, C.POINTER(AttendDesc), vp, vp, vp, C.POINTER(Runs), vp,
                                     vp, vp, vp]),
    "ckv_attend_merge": (C.c_int, [vp, u32, u32, u32, vp, vp, vp, vp, vp, u32]),
    "ckv_page_reps": (C.c_int, [vp, u32, u32, u32, u32, u32, vp, vp, vp]),
    "ckv_page_select": (C.c_int, [vp, C.POINTER(PageDesc), vp, vp, vp, C.POINTER(Runs), vp, vp]),
    "ckv_exact_topb": (C.c_int, [vp, u32, u32, u32, u32, vp, vp, u32, vp, u32]),
    "ckv_recall": (C.c_int, [vp, u32, vp, u32, vp, vp, u32, u32, vp]),
    "ckv_output_error": (C.c_int, [vp, u32, vp, vp, vp, vp]),
    "ckv_full_runs": (C.c_int, [vp, u32, u32, C.POINTER(Runs), vp]),
    "ckv_build_index": (C.c_int, [vp, u32, u32, u32, u32, vp, vp, vp, vp, vp]),
    "ckv_select": (C.c_int, [vp, C.POINTER(SelectDesc), vp, vp, vp, vp, vp, vp, vp, vp,
                             C.POINTER(Runs), vp, vp, vp, vp, vp, vp]),
    "ckv_cache_create": (C.c_int, [vp, u32, u32, u32, u32, C.POINTER(vp)]),
    "ckv_cache_destroy": (C.c_int, [vp]),
    "ckv_cache_counters": (C.c_int, [vp, vp]),
    "ckv_cache_lookup": (C.c_int, [vp, vp, u32, vp, u32, vp, vp, vp, vp]),
    "ckv_cache_invalidate": (C.c_int, [vp, vp, u32, vp, u32]),
    "ckv_attend": (C.c_int, [vp, C.POINTER(AttendDesc), vp, vp, vp, vp, C.POINTER(Runs), vp, vp,
                             vp]),
    "ckv_session_create": (C.c_int, [vp, C.POINTER(SessionDesc), C.POINTER(vp)]),
    "ckv_session_destroy": (C.c_int, [vp]),
    "ckv_session_kv": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(u32)]),
    "ckv_session_load_prompt": (C.c_int, [vp, vp, vp]),
    "ckv_session_prefill": (C.c_int, [vp, vp]),
    "ckv_session_step": (C.c_int, [vp, vp, vp, vp, vp, C.c_int]),
    "ckv_session_attend_only": (C.c_int, [vp, vp, vp]),
    "ckv_session_set_layer_units": (C.c_int, [vp, u32]),
    "ckv_session_batch_iterations": (C.c_int, [vp, vp]),
    "ckv_session_tier_stats": (C.c_int, [vp, vp]),
    "ckv_session_stats_get": (C.c_int, [vp, C.POINTER(SessionStats)]),
    "ckv_session_state": (C.c_int, [vp] + [C.POINTER(vp)] * 8 + [C.POINTER(u32)] * 2),
    "ckv_session_cache": (vp, [vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libckv_b200.so (raises if it is absent: no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is not built; run `python -m paper_2412_03213_b200.build` "
                "(the ClusterKV hot path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class CkvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[ckv {code}] {msg}")
        self.code = code


class ValidationError(CkvError, ValueError):
    """Raised under the predicates that make the reference throw
    ckv::ValidationError (common.hpp:27-30)."""


def check(rc: int) -> None:
    if rc != CKV_OK:
        msg = lib().ckv_last_error().decode()
        if rc == CKV_EINVAL:
            raise ValidationError(rc, msg)
        raise CkvError(rc, msg)
