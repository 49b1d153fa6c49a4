"""SPEC.md's acceptance properties (SURVEY §4 "golden vectors and properties")
on the GPU path, on the reference generator's heads (tests/_inputs.py):

- oracle equivalence: singleton clusters => select_tokens == exact_topb
  (SPEC.md:263, 515);
- k-means invariants: complete labels, no empty cluster, fixed point,
  monotone objective when no repair ran;
- full-budget identity: recall 1.0;
- recall ordering: cluster selection > page(16) > random on the default
  trace shape (8 centres, d = 128, seed 7).
"""
import numpy as np
import pytest

from oracle.oracle import to_bf16_representable
from tests._inputs import head, port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_singleton_clusters_equal_exact_topb(gpu_ctx, seed):
    """Every position its own cluster, centroid = the key: the budgeted
    cluster selection is the exact top-B (as a set)."""
    from paper_2412_03213_b200 import api, metrics
    h = head(seed, 0, 0, 256, T=8)
    K = h["K"]
    m = api.ClusterModel(K.shape[0], K.copy(), np.arange(K.shape[0], dtype=np.int32), 0)
    ix = api.build_index(m)
    for t in range(8):
        q = h["Q"][t]
        for B in (1, 17, 64, 255, 256, 300):
            r = api.select_tokens(q, m, ix, B)
            truth = metrics.exact_topb(q, K, B)
            assert np.array_equal(np.sort(r.token_ids), truth), (t, B)


def test_kmeans_invariants(gpu_ctx):
    from paper_2412_03213_b200 import api
    h = head(11, 0, 0, 4096)
    m = api.cluster_prefill(h["K"], api.ClusterConfig())
    lab = m.labels[m.sink_count:]
    C = m.n_clusters
    assert lab.min() >= 0 and lab.max() < C                    # label completeness
    assert np.all(np.bincount(lab, minlength=C) > 0)            # no empty cluster
    if m.converged:                                             # fixed point
        again = port().assign(h["K"][m.sink_count:], m.centroids)
        assert np.array_equal(again, lab)
    if not m.repair_iterations:                                 # monotone objective
        obj = np.asarray(m.objective_history)
        assert np.all(np.diff(obj) <= 1e-12 * np.abs(obj[:-1]) + 1e-15)


def test_full_budget_recall_one(gpu_ctx):
    """B >= L: every position is selected."""
    from paper_2412_03213_b200 import api, metrics
    h = head(12, 0, 0, 1024, T=4)
    m = api.cluster_prefill(h["K"], api.ClusterConfig())
    ix = api.build_index(m)
    for t in range(4):
        r = api.select_tokens(h["Q"][t], m, ix, 1024)
        truth = metrics.exact_topb(h["Q"][t], h["K"], 1024)
        assert metrics.recall_rate(r.token_ids, truth) == 1.0


def test_recall_ordering_cluster_page_random(gpu_ctx):
    """SPEC.md:517-519 on the default trace shape (L = 4096, B = 256): the
    mean recall of the exact top-B is cluster > page(16) > random (= B / L)."""
    from paper_2412_03213_b200 import api, metrics
    L, B = 4096, 256
    rc, rp = [], []
    for kv in range(2):
        tr = port().generate_head(port().mix_seed(7, 0, kv), L, 32)
        K = to_bf16_representable(tr.prompt_keys)
        Q = to_bf16_representable(tr.decode_queries)
        m = api.cluster_prefill(K, api.ClusterConfig())
        ix = api.build_index(m)
        for t in range(0, 32, 4):
            truth = metrics.exact_topb(Q[t], K, B)
            rc.append(metrics.recall_rate(api.select_tokens(Q[t], m, ix, B).token_ids, truth))
            rp.append(metrics.recall_rate(api.page_select(Q[t], K, B, 16), truth))
    rand = B / L
    assert np.mean(rc) > np.mean(rp) + 0.1, (np.mean(rc), np.mean(rp))
    assert np.mean(rp) > 1.2 * rand, (np.mean(rp), rand)
