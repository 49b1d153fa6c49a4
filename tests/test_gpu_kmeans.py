"""K1-K4 parity: GPU k-means vs the CPU oracle — labels, centroids,
iteration counts, convergence and repairs bit-exact; objective within 1e-9
relative (a diagnostic sum whose order differs, clustering.hpp:118-124)."""
import numpy as np
import pytest

from oracle.oracle import ClusterConfig as OCfg
from tests._inputs import head, port

pytestmark = pytest.mark.gpu


def _cmp_model(g, o, obj=True):
    assert g.iterations_used == o.iterations_used
    assert g.converged == o.converged
    assert np.array_equal(g.labels, o.labels)
    assert np.array_equal(g.centroids.view(np.uint32), o.centroids.view(np.uint32))
    assert list(g.repair_iterations) == list(o.repair_iterations)
    if obj:
        assert len(g.objective_history) == len(o.objective_history)
        np.testing.assert_allclose(g.objective_history, o.objective_history, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("layer,kvh", [(0, 0), (0, 3), (1, 5)])
def test_cluster_prefill_config_a_head(gpu_ctx, layer, kvh):
    from paper_2412_03213_b200 import api
    h = head(7, layer, kvh, 4096)
    seed = port().mix_seed(0, layer, kvh)
    o = port().cluster_prefill(h["K"], OCfg(seed=seed))
    g = api.cluster_prefill(h["K"], api.ClusterConfig(seed=seed))
    assert g.n_clusters == 51 and g.sink_count == 16
    _cmp_model(g, o)


def test_kmeans_init_rows_and_small_max_iters(gpu_ctx):
    from paper_2412_03213_b200 import api
    h = head(3, 0, 0, 1200)
    K = h["K"][16:]
    rows = np.arange(0, 60, 3, dtype=np.uint32)
    o = port().kmeans(K, 20, 0, 3, init_rows=rows)
    g = api.kmeans_cosine(K, 20, 0, 3, init_rows=rows)
    assert not g.converged and g.iterations_used == 3
    _cmp_model(g, o)


def test_kmeans_repair_path(gpu_ctx):
    """Exact duplicate keys make seeded init pick identical centroids; ties go
    to the lowest id, the twins come out empty and are repaired
    (clustering.hpp:128-153), with all-equal distances exercising the
    first-victim tie-break."""
    from paper_2412_03213_b200 import api
    from oracle.oracle import to_bf16_representable
    rng = np.random.default_rng(5)
    base = rng.standard_normal((6, 128)).astype(np.float32)
    K = to_bf16_representable(base[rng.integers(0, 6, 64)])
    n_rep = 0
    for C in (4, 8, 12):
        for seed in range(4):
            o = port().kmeans(K, C, seed, 50)
            g = api.kmeans_cosine(K, C, seed, 50)
            _cmp_model(g, o)
            n_rep += len(o.repair_iterations)
    assert n_rep > 10, "fixture should exercise repairs"


def test_kmeans_singletons_fixed_point(gpu_ctx):
    """N = C: each key its own centroid, converges in 1 iteration."""
    from paper_2412_03213_b200 import api
    h = head(11, 0, 0, 16 + 48)
    K = h["K"][16:]
    g = api.kmeans_cosine(K, 48, 9)
    o = port().kmeans(K, 48, 9)
    _cmp_model(g, o)
    assert g.converged and g.iterations_used == 1


def test_kmeans_validation_errors(gpu_ctx):
    from paper_2412_03213_b200 import api
    K = head(1, 0, 0, 64)["K"]
    with pytest.raises(ValueError, match="1 <= C <= N"):
        api.kmeans_cosine(K, 65, 0)
    with pytest.raises(ValueError, match="1 <= C <= N"):
        api.kmeans_cosine(K, 0, 0)
    bad = K.copy()
    bad[3, 7] = np.inf
    with pytest.raises(ValueError, match="finite"):
        api.kmeans_cosine(bad, 4, 0)
    with pytest.raises(ValueError, match="zero-norm"):
        api.kmeans_cosine(np.zeros((32, 128), np.float32), 4, 0)
    with pytest.raises(ValueError, match="init_rows"):
        api.kmeans_cosine(K, 4, 0, init_rows=[1, 2])


def test_prefill_cluster_count_kats():
    """SPEC.md:137-139 (no GPU needed: host arithmetic of the C-ABI)."""
    from paper_2412_03213_b200 import api
    cfg = api.ClusterConfig()
    assert api.prefill_cluster_count(32016, cfg) == 400
    assert api.prefill_cluster_count(96, cfg) == 1
    assert api.prefill_cluster_count(16, cfg) == 0
    assert api.prefill_cluster_count(4096, cfg) == 51
    assert api.prefill_cluster_count(32768, cfg) == 409
    assert api.prefill_cluster_count(131072, cfg) == 1638


def test_cluster_prefill_all_sinks(gpu_ctx):
    from paper_2412_03213_b200 import api
    K = head(1, 0, 0, 16)["K"]
    m = api.cluster_prefill(K, api.ClusterConfig())
    assert m.n_clusters == 0 and m.sink_count == 16 and m.converged
    assert np.all(m.labels == -1)


def test_decode_batch_kats(gpu_ctx):
    """320 keys -> +4 clusters; 2 keys -> +2; ids disjoint."""
    from paper_2412_03213_b200 import api
    h = head(7, 0, 1, 1024, T=400)
    seed = port().mix_seed(0, 0, 1)
    cfg = api.ClusterConfig(seed=seed)
    g = api.cluster_prefill(h["K"], cfg)
    o = port().cluster_prefill(h["K"], OCfg(seed=seed))
    api.cluster_decode_batch(g, h["dK"][:320], cfg)
    oc, ol, oit = port().cluster_decode_batch(o.centroids, o.labels, h["dK"][:320], OCfg(seed=seed))
    assert g.n_clusters == o.n_clusters + 4
    assert np.array_equal(g.labels, ol)
    assert np.array_equal(g.centroids.view(np.uint32), oc.view(np.uint32))
    assert g.invocation_iterations[-1] == oit
    api.cluster_decode_batch(g, h["dK"][320:322], cfg)
    oc, ol, _ = port().cluster_decode_batch(oc, ol, h["dK"][320:322], OCfg(seed=seed))
    assert g.n_clusters == o.n_clusters + 6
    assert np.array_equal(g.labels, ol)
    assert set(g.labels[-2:]) == {o.n_clusters + 4, o.n_clusters + 5}
