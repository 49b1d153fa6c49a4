"""ckv_select_scored (the global budgeted top-k of the sharded decode step)
on adversarial scores: many exact ties, zero-size clusters, NaN scores,
budgets below / at / above the total — against select_tokens' ranking and
cut (selection.hpp:74-106) restated over the same scores."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _reference(scores, sizes, B):
    """selection.hpp:80-106 over given scores: std::sort by (score desc, id
    asc) with NaN last (the kernels' convention), then the cum < B walk."""
    C_ = len(scores)
    key = [(1, 0.0, c) if np.isnan(scores[c]) else (0, -scores[c], c) for c in range(C_)]
    ranked = [k[2] for k in sorted(key)]
    cum, taken, trimmed, allow = 0, 0, 0, []
    for c in ranked:
        if cum >= B:
            break
        rem = B - cum
        if sizes[c] <= rem:
            allow.append(int(sizes[c]))
            cum += int(sizes[c])
        else:
            allow.append(rem)
            trimmed = int(sizes[c]) - rem
            cum = B
        taken += 1
    return ranked, taken, trimmed, allow


@pytest.mark.parametrize("C_,B,seed", [(1638, 2048, 0), (1638, 100, 1), (300, 5000, 2),
                                       (4096, 3000, 3), (50, 0, 4), (777, 1, 5)])
def test_select_scored_ties_and_zero_sizes(gpu_ctx, C_, B, seed):
    import torch
    from paper_2412_03213_b200 import _native as N
    rng = np.random.default_rng(seed)
    n_q = 6
    scores = rng.integers(0, 40, (n_q, C_)).astype(np.float64) * 0.25  # many exact ties
    scores[0, :5] = np.nan
    scores[1] = 1.5  # all tied
    sizes = rng.integers(0, 9, C_).astype(np.int32)
    sizes[::7] = 0
    dev = gpu_ctx.device
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)
    gs = t(sizes[None], torch.int32)
    starts = t(np.concatenate([[0], np.cumsum(sizes)])[None], torch.int32)
    pre = torch.zeros_like(gs)
    sc = t(scores, torch.float64)
    run_cap = C_ + 2
    rr = torch.zeros((n_q, run_cap), dtype=torch.int32, device=dev)
    ro = torch.zeros((n_q, run_cap + 1), dtype=torch.int32, device=dev)
    rc = torch.zeros(n_q, dtype=torch.int32, device=dev)
    runs = N.Runs(rr.data_ptr(), ro.data_ptr(), rc.data_ptr(), run_cap)
    nt, nk, tr = [torch.zeros(n_q, dtype=torch.int32, device=dev) for _ in range(3)]
    rk = torch.zeros((n_q, C_), dtype=torch.int32, device=dev)
    d = N.ShardSelectDesc(n_q, n_q, B, C_, C_, C_, 1, int(sizes.sum()) + 1, B + 1, 0, 0, 0, 0, 0,
                          0, 0)
    N.check(N.lib().ckv_select_scored(gpu_ctx.h, C.byref(d), sc.data_ptr(), gs.data_ptr(),
                                      gs.data_ptr(), starts.data_ptr(), pre.data_ptr(), None,
                                      C.byref(runs), None, nt.data_ptr(), nk.data_ptr(),
                                      tr.data_ptr(), rk.data_ptr()))
    rk, nk, tr, ro, nt = (x.cpu().numpy() for x in (rk, nk, tr, ro, nt))
    for h in range(n_q):
        ranked, taken, trimmed, allow = _reference(scores[h], sizes, B)
        assert nk[h] == taken and tr[h] == trimmed
        assert list(rk[h][:taken]) == ranked[:taken]
        assert list(np.diff(ro[h][:taken + 1])) == allow
        assert nt[h] == sum(allow)
