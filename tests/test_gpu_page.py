"""Page-select baseline (selection.hpp:136-194) on the B200 kernels: the
selected token ids bit-exact vs the CPU oracle (pinned to the compiled
reference in tests/test_oracle.py), for both representatives, partial last
pages, budgets below one page / above the context, ties; and the runs feed
ckv_attend over a position-ordered store like the reference's
approx_attention over page_select's ids."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import to_bf16_representable
from tests._inputs import head, port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,B,ps,rep", [(1000, 256, 16, 0), (1000, 256, 16, 1), (37, 100, 7, 1),
                                        (4096, 1024, 32, 0), (10, 5, 16, 0), (4000, 10000, 16, 0),
                                        (32752, 1024, 16, 1)])
def test_page_select_matches_oracle(gpu_ctx, n, B, ps, rep):
    from paper_2412_03213_b200 import api
    h = head(3, 0, 1, max(n, 64), T=8)
    K = h["K"][:n]
    for t in range(3):
        q = h["Q"][t]
        got = api.page_select(q, K, B, ps, rep)
        exp = port().page_select(q, K, B, ps, bool(rep))
        assert np.array_equal(got, exp), (n, B, ps, rep, t)


def test_page_select_ties(gpu_ctx):
    from paper_2412_03213_b200 import api
    rng = np.random.default_rng(2)
    K = np.repeat(to_bf16_representable(rng.standard_normal((8, 128)).astype(np.float32)), 64, 0)
    q = to_bf16_representable(rng.standard_normal(128).astype(np.float32))
    for B in (64, 128, 200):
        assert np.array_equal(api.page_select(q, K, B, 16), port().page_select(q, K, B, 16))


def test_page_select_validation(gpu_ctx):
    from paper_2412_03213_b200 import api
    from paper_2412_03213_b200._native import ValidationError
    K = head(1, 0, 0, 64)["K"]
    with pytest.raises(ValidationError, match="page_size"):
        api.page_select(K[0], K, 32, 0)


def test_page_runs_feed_attention(gpu_ctx):
    """Batched: many q heads over a position-ordered store, runs -> ckv_attend."""
    import torch

    from paper_2412_03213_b200 import _native as N
    U, G, L, B, ps = 3, 2, 2048, 256, 16
    hs = [head(8, 0, u, L, T=16) for u in range(U)]
    bits = lambda x: (np.ascontiguousarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)
    dev = gpu_ctx.device
    Kd = torch.from_numpy(bits(np.stack([x["K"] for x in hs])).view(np.int16)).to(dev)
    Vd = torch.from_numpy(bits(np.stack([x["V"] for x in hs])).view(np.int16)).to(dev)
    Q = np.stack([hs[u]["Q"][3 + 5 * g] for u in range(U) for g in range(G)])
    n_pages = L // ps
    rmax = torch.empty((U, n_pages, 128), dtype=torch.float32, device=dev)
    N.check(N.lib().ckv_page_reps(gpu_ctx.h, U, L, L, ps, n_pages, Kd.data_ptr(), rmax.data_ptr(),
                                  None))
    n_q, n_sel = U * G, B // ps
    rr = torch.zeros((n_q, n_sel + 1), dtype=torch.int32, device=dev)
    ro = torch.zeros((n_q, n_sel + 2), dtype=torch.int32, device=dev)
    rc = torch.zeros(n_q, dtype=torch.int32, device=dev)
    runs = N.Runs(rr.data_ptr(), ro.data_ptr(), rc.data_ptr(), n_sel + 1)
    ids = torch.zeros((n_q, B), dtype=torch.int32, device=dev)
    nt = torch.zeros(n_q, dtype=torch.int32, device=dev)
    qd = torch.from_numpy(Q).to(dev)
    d = N.PageDesc(n_q, G, L, ps, B, n_pages, B, 0)
    N.check(N.lib().ckv_page_select(gpu_ctx.h, C.byref(d), qd.data_ptr(), rmax.data_ptr(), None,
                                    C.byref(runs), ids.data_ptr(), nt.data_ptr()))
    out = torch.zeros((n_q, 128), dtype=torch.float32, device=dev)
    w = torch.zeros((n_q, B), dtype=torch.float32, device=dev)
    ad = N.AttendDesc(n_q, G, L, B, B)
    N.check(N.lib().ckv_attend(gpu_ctx.h, C.byref(ad), qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(),
                               None, C.byref(runs), nt.data_ptr(), out.data_ptr(), w.data_ptr()))
    for u in range(U):
        for g in range(G):
            h = u * G + g
            exp = port().page_select(Q[h], hs[u]["K"], B, ps)
            k = int(nt[h].item())
            assert np.array_equal(ids[h, :k].cpu().numpy().view(np.uint32), exp)
            oo, ow = port().approx_attention(Q[h], hs[u]["K"], hs[u]["V"], exp)
            assert np.abs(out[h].cpu().numpy() - oo).max() <= 2e-5 * np.abs(hs[u]["V"]).max()
            assert np.abs(w[h, :k].cpu().numpy() - ow).max() <= 1e-6 + 2e-5 * ow.max()
