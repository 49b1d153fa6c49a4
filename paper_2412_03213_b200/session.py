"""Batched, device-resident decode session (ckv_session_* in the C-ABI).

Mirrors the ClusterKV branch of simulate_head (harness.hpp:155-346) for many
(batch, layer, kv-head) units at once: prefill clustering + index, then per
decode step select (+cache) -> sparse attention -> append -> decode-batch
clustering every m steps.  The metric oracles of the harness are not part of
the serving path and are not run.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from ._native import check, lib
from .api import ClusterConfig, Context

D = 128


class _CAI:
    """__cuda_array_interface__ shim so torch can view ckv-owned memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}


def device_view(ptr: int, shape, dtype: torch.dtype, device) -> torch.Tensor:
    ts = {torch.int16: "<i2", torch.int32: "<i4", torch.float32: "<f4"}[dtype]
    return torch.as_tensor(_CAI(ptr, shape, ts), device=device)


class Session:
    def __init__(self, n_units: int, group: int, prompt_len: int, max_decode: int,
                 budget: int, retention: int = 1, cfg: ClusterConfig | None = None,
                 kv_heads: int = 8, flags: int = 0, ctx: Context | None = None,
                 async_delay: int = 0):
        cfg = cfg or ClusterConfig()
        cfg.validate()
        if cfg.metric != 0:
            raise N.ValidationError(1, "Session: cosine assignment only (DESIGN.md §1)")
        self.ctx = ctx or Context.default()
        self.cfg = cfg
        self.n_units, self.group = n_units, group
        self.n_q = n_units * group
        desc = N.SessionDesc(n_units, group, prompt_len, max_decode, budget, retention,
                             cfg.c0_divisor, cfg.c_plus, cfg.decode_batch, cfg.sink_tokens,
                             cfg.max_iters, cfg.seed, kv_heads, flags, async_delay,
                             cfg.c0_override)
        h = C.c_void_p()
        check(lib().ckv_session_create(self.ctx.h, C.byref(desc), C.byref(h)))
        self.h = h
        self._refresh_kv()
        self.prompt_len = prompt_len

    def _refresh_kv(self):
        """(Re)bind torch views of the KV store; prefill relays it
        cluster-major into new buffers."""
        Kp, Vp, pc = C.c_void_p(), C.c_void_p(), C.c_uint32()
        check(lib().ckv_session_kv(self.h, C.byref(Kp), C.byref(Vp), C.byref(pc)))
        self.p_cap = pc.value
        dev = self.ctx.device
        self.K = device_view(Kp.value, (self.n_units, self.p_cap, D), torch.int16, dev)
        self.V = device_view(Vp.value, (self.n_units, self.p_cap, D), torch.int16, dev)

    def __del__(self):
        try:
            lib().ckv_session_destroy(self.h)
        except Exception:
            pass

    # ---- state -----------------------------------------------------------
    def load_prompt_host(self, K_bf16: np.ndarray, V_bf16: np.ndarray) -> None:
        """K/V: host uint16/int16 bf16 bit patterns [n_units, L, 128]."""
        K_bf16 = np.ascontiguousarray(K_bf16).view(np.int16)
        V_bf16 = np.ascontiguousarray(V_bf16).view(np.int16)
        check(lib().ckv_session_load_prompt(self.h, K_bf16.ctypes.data, V_bf16.ctypes.data))

    def prefill(self):
        info = (N.KMeansInfo * self.n_units)()
        check(lib().ckv_session_prefill(self.h, info))
        self._refresh_kv()
        return [(i.iterations_used, bool(i.converged)) for i in info]

    def step(self, q, k_new, v_new, out=None, on_device: bool = True):
        if on_device:
            if out is None:
                out = torch.empty((self.n_q, D), dtype=torch.float32, device=self.ctx.device)
            check(lib().ckv_session_step(self.h, q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                                         out.data_ptr(), 1))
            return out
        q = np.ascontiguousarray(q, np.float32)
        k_new = np.ascontiguousarray(k_new).view(np.int16)
        v_new = np.ascontiguousarray(v_new).view(np.int16)
        if out is None:
            out = np.empty((self.n_q, D), np.float32)
        check(lib().ckv_session_step(self.h, q.ctypes.data, k_new.ctypes.data, v_new.ctypes.data,
                                     out.ctypes.data, 0))
        return out

    def attend_only(self, q: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        check(lib().ckv_session_attend_only(self.h, q.data_ptr(), out.data_ptr()))
        return out

    def set_layer_units(self, layer_units: int) -> None:
        """Layer mode (ckv_session_set_layer_units): one select + attend per
        slice of layer_units units, in order; 0 = all units at once."""
        check(lib().ckv_session_set_layer_units(self.h, layer_units))

    def batch_iterations(self) -> np.ndarray:
        """k-means iterations of each unit's most recent decode batch."""
        out = np.zeros(self.n_units, np.uint32)
        check(lib().ckv_session_batch_iterations(self.h, out.ctypes.data))
        return out

    def tier_stats(self) -> dict:
        """Physical two-tier cache counters (tiered sessions)."""
        out = np.zeros(5, np.uint64)
        check(lib().ckv_session_tier_stats(self.h, out.ctypes.data))
        return dict(rows_fetched=int(out[0]), clusters_fetched=int(out[1]),
                    clusters_selected=int(out[2]), evictions=int(out[3]),
                    pool_rows_per_unit=int(out[4]),
                    bytes_fetched=int(out[0]) * D * 2 * 2)

    def stats(self) -> N.SessionStats:
        st = N.SessionStats()
        check(lib().ckv_session_stats_get(self.h, C.byref(st)))
        return st

    def state(self) -> dict:
        """Device views of the model / index / last selection."""
        ptrs = [C.c_void_p() for _ in range(8)]
        c_cap, sel_cap = C.c_uint32(), C.c_uint32()
        check(lib().ckv_session_state(self.h, *[C.byref(p) for p in ptrs], C.byref(c_cap),
                                      C.byref(sel_cap)))
        U, dev, P, Cc, S = self.n_units, self.ctx.device, self.p_cap, c_cap.value, sel_cap.value
        return dict(
            centroids=device_view(ptrs[0].value, (U, Cc, D), torch.float32, dev),
            labels=device_view(ptrs[1].value, (U, P), torch.int32, dev),
            n_clusters=device_view(ptrs[2].value, (U,), torch.int32, dev),
            sizes=device_view(ptrs[3].value, (U, Cc), torch.int32, dev),
            starts=device_view(ptrs[4].value, (U, Cc + 1), torch.int32, dev),
            sorted_ids=device_view(ptrs[5].value, (U, P), torch.int32, dev),
            token_ids=device_view(ptrs[6].value, (self.n_q, S), torch.int32, dev),
            n_tokens=device_view(ptrs[7].value, (self.n_q,), torch.int32, dev),
            c_cap=Cc, sel_cap=S)

    def cache_counters(self) -> np.ndarray:
        c = lib().ckv_session_cache(self.h)
        out = np.zeros((self.n_q, 4), np.uint64)
        if c:
            check(lib().ckv_cache_counters(c, out.ctypes.data))
        return out
