"""Quality metrics of the reference harness on the GPU (
harness.hpp:228-310): the exact top-B ground truth, recall, full attention and
the output error, through the C-ABI kernels of ckv_metrics.cu.

Reference-named single-query functions (exact_topb, recall_rate,
full_attention, output_error) mirror selection.hpp / attention.hpp for the
parity tests; `StepQuality` evaluates a whole decode step's selection (every
q head at once) against the exact top-B and full attention, as
simulate_head does per row, for quality sweeps at GPU speed.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._native import ValidationError, check, lib
from .api import AttentionOutput, Context, _check_d, _to_bf16_device

D = 128


def exact_topb(q: np.ndarray, keys: np.ndarray, budget: int,
               ctx: Context | None = None) -> np.ndarray:
    """selection.hpp:115-132: the min(B, n) largest dot_f64(q, k_i), ties to
    the lowest index, ascending."""
    ctx = ctx or Context.default()
    keys = np.ascontiguousarray(keys, np.float32)
    _check_d(keys, "exact_topb")
    n = keys.shape[0]
    bn = min(budget, n)
    if bn == 0:
        return np.zeros(0, np.uint32)
    kb = _to_bf16_device(ctx, keys, "exact_topb keys")
    qd = torch.from_numpy(np.ascontiguousarray(q, np.float32).reshape(1, D)).to(ctx.device)
    ids = torch.zeros((1, bn), dtype=torch.int32, device=ctx.device)
    check(lib().ckv_exact_topb(ctx.h, 1, 1, n, n, qd.data_ptr(), kb.data_ptr(), budget,
                               ids.data_ptr(), bn))
    return ids[0].cpu().numpy().view(np.uint32).copy()


def recall_rate(selected, truth) -> float:
    """attention.hpp:70-93 (host; the batched form is StepQuality)."""
    truth = np.asarray(truth)
    if len(truth) == 0:
        raise ValidationError(1, "recall_rate: truth set must be non-empty")
    a, b = np.sort(np.asarray(selected)), np.sort(truth)
    hits, i, j = 0, 0, 0
    while i < len(a) and j < len(b):
        if a[i] < b[j]:
            i += 1
        elif b[j] < a[i]:
            j += 1
        else:
            hits, i, j = hits + 1, i + 1, j + 1
    return hits / len(b)


def full_attention(q: np.ndarray, keys: np.ndarray, values: np.ndarray,
                   ctx: Context | None = None) -> AttentionOutput:
    """attention.hpp:53-60: approx_attention over every row."""
    from .api import approx_attention
    if keys.shape[0] < 1:
        raise ValidationError(1, "full_attention: need at least one token")
    return approx_attention(q, keys, values, np.arange(keys.shape[0], dtype=np.uint32), ctx)


@dataclass
class OutputError:
    l2_rel: float
    cos_sim: float


def output_error(approx: np.ndarray, exact: np.ndarray) -> OutputError:
    """attention.hpp:101-131 (host, for single outputs)."""
    a = np.asarray(approx, np.float64)
    e = np.asarray(exact, np.float64)
    if a.shape != e.shape:
        raise ValidationError(1, "output_error: dimension mismatch")
    diff2, e2, a2, dot = 0.0, 0.0, 0.0, 0.0
    for x, y in zip(a.tolist(), e.tolist()):
        diff2 += (x - y) * (x - y)
        e2 += y * y
        a2 += x * x
        dot += x * y
    en, an = np.sqrt(e2), np.sqrt(a2)
    l2 = np.sqrt(diff2) if en < 1e-12 else np.sqrt(diff2) / en
    if an < 1e-12 and en < 1e-12:
        cs = 1.0
    elif an < 1e-12 or en < 1e-12:
        cs = 0.0
    else:
        cs = dot / (an * en)
    return OutputError(float(l2), float(cs))


class StepQuality:
    """One decode step's quality for every q head, on the device: recall of
    the selected positions against exact_topb, and the output error of the
    sparse attention against full attention (simulate_head's recall /
    l2_rel / cos_sim, harness.hpp:228-310).

    K, V: a position-ordered store, device bf16 bits [units][p_cap][128];
    n: context length; q head h reads unit h // group."""

    def __init__(self, K: torch.Tensor, V: torch.Tensor, n: int, group: int, budget: int,
                 ctx: Context | None = None):
        self.ctx = ctx or Context.default()
        self.K, self.V, self.n, self.G, self.B = K, V, n, group, budget
        self.p_cap = int(K.shape[1])
        self.n_q = int(K.shape[0]) * group
        dev = K.device
        self.bn = min(budget, n)
        self.truth = torch.zeros((self.n_q, self.bn), dtype=torch.int32, device=dev)
        self.rr = torch.zeros((self.n_q, 1), dtype=torch.int32, device=dev)
        self.ro = torch.zeros((self.n_q, 2), dtype=torch.int32, device=dev)
        self.rc = torch.zeros(self.n_q, dtype=torch.int32, device=dev)
        self.runs = N.Runs(self.rr.data_ptr(), self.ro.data_ptr(), self.rc.data_ptr(), 1)
        self.nt = torch.zeros(self.n_q, dtype=torch.int32, device=dev)
        self.exact = torch.zeros((self.n_q, D), dtype=torch.float32, device=dev)
        self.recall = torch.zeros(self.n_q, dtype=torch.float64, device=dev)
        self.l2 = torch.zeros(self.n_q, dtype=torch.float64, device=dev)
        self.cos = torch.zeros(self.n_q, dtype=torch.float64, device=dev)

    def __call__(self, q: torch.Tensor, sel: torch.Tensor, n_sel: torch.Tensor,
                 approx_out: torch.Tensor) -> dict:
        """q f32 [n_q][128]; sel int32 [n_q][cap] selected positions (n_sel
        each); approx_out f32 [n_q][128] the sparse attention output."""
        L, h = lib(), self.ctx.h
        q = q.contiguous()
        check(L.ckv_exact_topb(h, self.n_q, self.G, self.n, self.p_cap, q.data_ptr(),
                               self.K.data_ptr(), self.B, self.truth.data_ptr(), self.bn))
        check(L.ckv_recall(h, self.n_q, sel.data_ptr(), sel.shape[1], n_sel.data_ptr(),
                           self.truth.data_ptr(), self.bn, self.bn, self.recall.data_ptr()))
        check(L.ckv_full_runs(h, self.n_q, self.n, C.byref(self.runs), self.nt.data_ptr()))
        ad = N.AttendDesc(self.n_q, self.G, self.p_cap, self.n, self.n)
        check(L.ckv_attend(h, C.byref(ad), q.data_ptr(), self.K.data_ptr(), self.V.data_ptr(),
                           None, C.byref(self.runs), self.nt.data_ptr(), self.exact.data_ptr(),
                           None))
        check(L.ckv_output_error(h, self.n_q, approx_out.contiguous().data_ptr(),
                                 self.exact.data_ptr(), self.l2.data_ptr(), self.cos.data_ptr()))
        return dict(recall=self.recall, l2_rel=self.l2, cos_sim=self.cos, truth=self.truth,
                    exact_out=self.exact)
