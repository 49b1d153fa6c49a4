"""K7 sparse attention vs the f64 oracle (attention.hpp:20-50).

Tolerance: the GPU computes logits / softmax / weighted sum in
f32 from bf16 K/V; the reference in f64.  Bars: max|dout| <= 2e-5 * max|v|,
rel-L2(out) <= 1e-5, max|dweight| <= 1e-6 + 2e-5 * weight.
"""
import numpy as np
import pytest

from tests._inputs import head, port

pytestmark = pytest.mark.gpu


def _check(go, gw, oo, ow, V):
    vmax = np.abs(V).max()
    assert np.abs(go - oo).max() <= 2e-5 * vmax
    assert np.linalg.norm(go - oo) <= 1e-5 * max(np.linalg.norm(oo), 1e-30) + 1e-6
    assert np.all(np.abs(gw - ow) <= 1e-6 + 2e-5 * np.abs(ow))
    assert abs(gw.sum() - 1.0) < 1e-5


@pytest.mark.parametrize("n_sel", [1, 17, 128, 129, 1040, 2064, 4000])
def test_attend_vs_oracle(gpu_ctx, n_sel):
    from paper_2412_03213_b200 import api
    h = head(7, 0, 0, 4096)
    rng = np.random.default_rng(n_sel)
    sel = rng.choice(4096, n_sel, replace=False).astype(np.uint32)
    q = h["Q"][3]
    g = api.approx_attention(q, h["K"], h["V"], sel)
    oo, ow = port().approx_attention(q, h["K"], h["V"], sel)
    _check(g.out, g.weights, oo, ow, h["V"])


def test_attend_duplicate_rows_and_order(gpu_ctx):
    """I_T order and duplicates are honoured (weights are per entry)."""
    from paper_2412_03213_b200 import api
    h = head(8, 0, 0, 300)
    sel = np.array([5, 5, 299, 0, 17, 5], np.uint32)
    q = h["Q"][0]
    g = api.approx_attention(q, h["K"], h["V"], sel)
    oo, ow = port().approx_attention(q, h["K"], h["V"], sel)
    _check(g.out, g.weights, oo, ow, h["V"])


def test_attend_empty_selection_raises(gpu_ctx):
    from paper_2412_03213_b200 import api
    h = head(8, 0, 0, 64)
    with pytest.raises(ValueError, match="empty selection"):
        api.approx_attention(h["Q"][0], h["K"], h["V"], [])


def test_attend_full_budget_identity(gpu_ctx):
    """B >= L selects everything; approx == full attention."""
    from paper_2412_03213_b200 import api
    h = head(9, 0, 0, 2048)
    sel = np.arange(2048, dtype=np.uint32)
    g = api.approx_attention(h["Q"][1], h["K"], h["V"], sel)
    oo, ow = port().approx_attention(h["Q"][1], h["K"], h["V"], sel)
    _check(g.out, g.weights, oo, ow, h["V"])
