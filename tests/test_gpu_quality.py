"""GPU decode-loop quality driver (quality.run_simulation)
against the reference harness's own run_simulation (harness.hpp:362-410,
compiled unmodified into oracle/_ref; outputs committed as
tests/golden/harness_small.npz by tests/golden/make_harness_golden.py) on the
same bf16-rounded synthetic bundle (regenerated here by the oracle port,
whose generator is pinned to the reference in tests/test_oracle.py).

Per row: recall and the cluster-cache deltas (hits, requests, tokens)
bit-exact; l2_rel / cos_sim within the attention tolerance (f32 on the GPU
vs f64).  Summary: means, hit rate, transferred tokens / bytes, the k-means
iteration histogram.  Runs: a budget sweep, retention 2, async clustering.
"""
import os

import numpy as np
import pytest

from oracle.oracle import to_bf16_representable
from tests._inputs import port

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "harness_small.npz")


def _bundle(g):
    from paper_2412_03213_b200.trace import HeadTrace, TraceBundle
    spec = {k[5:]: int(g[k]) for k in g.files if k.startswith("spec_")}
    tr = port().generate_synthetic(spec["seed"], spec["n_layers"], spec["n_heads"], spec["L"],
                                   spec["T"])
    r = lambda a: to_bf16_representable(a)
    heads = [HeadTrace(r(tr.prompt_keys[u]), r(tr.prompt_values[u]), r(tr.decode_queries[u]),
                       r(tr.decode_keys[u]), r(tr.decode_values[u]))
             for u in range(spec["n_layers"] * spec["n_heads"])]
    return TraceBundle(spec["n_layers"], spec["n_heads"], heads), spec


@pytest.mark.parametrize("run", ["b48", "b96", "b200", "b96_r2", "b96_async3"])
def test_quality_run_matches_reference_harness(gpu_ctx, run):
    from paper_2412_03213_b200 import quality as Q
    from paper_2412_03213_b200.api import ClusterConfig
    g = np.load(GOLD)
    bundle, spec = _bundle(g)
    cfg = Q.PolicyConfig(budget=int(g[f"{run}__cfg_budget"]),
                         cluster=ClusterConfig(decode_batch=int(g["common_decode_batch"]),
                                               c0_divisor=int(g["common_c0_divisor"])))
    if f"{run}__cfg_retention" in g.files:
        cfg.retention = int(g[f"{run}__cfg_retention"])
    if f"{run}__cfg_async_clustering" in g.files:
        cfg.async_clustering = bool(g[f"{run}__cfg_async_clustering"])
        cfg.async_delay = int(g[f"{run}__cfg_async_delay"])
    rep = Q.run_simulation(bundle, cfg)
    rf, ru = g[f"{run}__rows_f"], g[f"{run}__rows_u"]
    assert len(rep.rows) == len(rf)
    got_u = np.array([[r.step, r.layer, r.head, r.clusters_hit, r.clusters_requested,
                       r.tokens_transferred] for r in rep.rows], np.uint64)
    assert np.array_equal(got_u, ru)
    got_f = np.array([[r.recall, r.l2_rel, r.cos_sim] for r in rep.rows])
    assert np.array_equal(got_f[:, 0], rf[:, 0]), "recall differs"
    np.testing.assert_allclose(got_f[:, 1], rf[:, 1], rtol=2e-3, atol=2e-4)
    np.testing.assert_allclose(got_f[:, 2], rf[:, 2], rtol=0, atol=2e-4)
    s, sf, su = rep.summary, g[f"{run}__summ_f"], g[f"{run}__summ_u"]
    assert abs(s.mean_recall - sf[0]) <= 1e-12
    assert abs(s.mean_l2_rel - sf[1]) <= 2e-3 * abs(sf[1]) + 2e-4
    assert abs(s.mean_cos_sim - sf[2]) <= 2e-4
    assert s.hit_rate == pytest.approx(sf[3], abs=1e-15)
    assert (s.tokens_transferred, s.bytes_transferred) == (int(su[0]), int(su[1]))
    hist = {i: int(n) for i, n in enumerate(g[f"{run}__hist"]) if n}
    assert s.iteration_histogram == hist


def test_quality_sweep_budget_monotone_recall(gpu_ctx):
    """sweep (harness.hpp:449-475) over the budget axis: one run per value,
    recall non-decreasing in the budget on this bundle."""
    from paper_2412_03213_b200 import quality as Q
    from paper_2412_03213_b200.api import ClusterConfig
    bundle, _ = _bundle(np.load(GOLD))
    base = Q.PolicyConfig(cluster=ClusterConfig(decode_batch=16, c0_divisor=40))
    reps = Q.sweep(bundle, base, "budget", [32, 96, 400])
    rec = [r.summary.mean_recall for r in reps]
    assert rec == sorted(rec) and [r.summary.budget for r in reps] == [32, 96, 400]
    with pytest.raises(ValueError):
        Q.sweep(bundle, base, "distance", ["l2"])
