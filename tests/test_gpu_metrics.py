"""Quality metrics on the GPU (ckv_metrics.cu) against the
CPU oracle: exact_topb bit-exact (ties included), recall and output error of
a whole step's selections matching the host restatements of
attention.hpp:70-131 on the same inputs."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import to_bf16_representable
from tests._inputs import head, port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,B", [(1000, 256), (4096, 1024), (300, 1000), (32768, 1024),
                                 (5000, 1), (601, 96), (33, 7), (4097, 1024)])
def test_exact_topb_matches_oracle(gpu_ctx, n, B):
    from paper_2412_03213_b200 import metrics
    h = head(4, 0, 2, max(n, 64), T=8)
    K = h["K"][:n]
    for t in range(3):
        assert np.array_equal(metrics.exact_topb(h["Q"][t], K, B), port().exact_topb(h["Q"][t], K, B))


def test_exact_topb_ties(gpu_ctx):
    from paper_2412_03213_b200 import metrics
    rng = np.random.default_rng(5)
    K = np.repeat(to_bf16_representable(rng.standard_normal((10, 128)).astype(np.float32)), 50, 0)
    q = to_bf16_representable(rng.standard_normal(128).astype(np.float32))
    for B in (1, 30, 77, 500):
        assert np.array_equal(metrics.exact_topb(q, K, B), port().exact_topb(q, K, B))


def test_step_quality_matches_host(gpu_ctx):
    """StepQuality on page-select selections: recall and output error per q
    head equal the host restatements on the oracle's truth / attention."""
    import torch

    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200 import api, metrics
    U, G, L, B, ps = 2, 2, 2048, 256, 16
    hs = [head(12, 0, u, L, T=16) for u in range(U)]
    bits = lambda x: (np.ascontiguousarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)
    dev = gpu_ctx.device
    Kd = torch.from_numpy(bits(np.stack([x["K"] for x in hs])).view(np.int16)).to(dev)
    Vd = torch.from_numpy(bits(np.stack([x["V"] for x in hs])).view(np.int16)).to(dev)
    Q = np.stack([hs[u]["Q"][2 + 6 * g] for u in range(U) for g in range(G)])
    n_q = U * G
    sel = np.zeros((n_q, B), np.int32)
    nsel = np.zeros(n_q, np.int32)
    outs = np.zeros((n_q, 128), np.float32)
    for hh in range(n_q):
        ids = api.page_select(Q[hh], hs[hh // G]["K"], B, ps)
        sel[hh, :len(ids)] = ids
        nsel[hh] = len(ids)
        outs[hh] = api.approx_attention(Q[hh], hs[hh // G]["K"], hs[hh // G]["V"], ids).out
    sq = metrics.StepQuality(Kd, Vd, L, G, B, gpu_ctx)
    t = lambda a: torch.from_numpy(a).to(dev)
    r = sq(t(Q), t(sel), t(nsel), t(outs))
    for hh in range(n_q):
        truth = port().exact_topb(Q[hh], hs[hh // G]["K"], B)
        assert np.array_equal(r["truth"][hh].cpu().numpy().view(np.uint32), truth)
        assert r["recall"][hh].item() == metrics.recall_rate(sel[hh, :nsel[hh]], truth)
        eo, _ = port().approx_attention(Q[hh], hs[hh // G]["K"], hs[hh // G]["V"],
                                        np.arange(L, dtype=np.uint32))
        assert np.abs(r["exact_out"][hh].cpu().numpy() - eo).max() <= 2e-5 * np.abs(hs[hh // G]["V"]).max()
        e = metrics.output_error(outs[hh], r["exact_out"][hh].cpu().numpy())
        assert abs(r["l2_rel"][hh].item() - e.l2_rel) <= 1e-12 * max(1.0, e.l2_rel)
        assert abs(r["cos_sim"][hh].item() - e.cos_sim) <= 1e-12
