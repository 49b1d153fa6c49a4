"""Generates tests/golden/golden_v1.npz from the COMPILED REFERENCE
(oracle/_ref/libckv_ref.so, built from /root/reference/proj/include by
oracle/Makefile).  Run here (the reference is not on the GPU box):

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import ClusterConfig, Oracle, build, to_bf16_representable  # noqa: E402


def main():
    build(ref=True)
    R = Oracle("reference")
    out = {}
    seed, L, T = R.mix_seed(7, 0, 0), 96, 8
    tr = R.generate_head(seed, L, T)
    out.update(gen_seed=seed, gen_L=L, gen_T=T, gen_prompt_keys=tr.prompt_keys,
               gen_decode_queries=tr.decode_queries)
    tr = R.generate_head(R.mix_seed(7, 0, 1), 1200, 16)
    K = to_bf16_representable(tr.prompt_keys)
    V = to_bf16_representable(tr.prompt_values)
    km_seed = R.mix_seed(0, 0, 1)
    m = R.cluster_prefill(K, ClusterConfig(seed=km_seed))
    out.update(km_keys=K, km_seed=km_seed, km_iters=m.iterations_used, km_converged=m.converged,
               km_labels=m.labels, km_centroids=m.centroids, km_objective=m.objective_history)
    q = to_bf16_representable(tr.decode_queries[5])
    rec = np.arange(1200, 1207, dtype=np.uint32)
    s = R.select_tokens(q, m.centroids, m.labels, m.sink_count, 200, rec)
    out.update(sel_q=q, sel_budget=200, sel_recency=rec, sel_ranked=s.ranked_clusters,
               sel_token_ids=s.token_ids, sel_taken=s.n_clusters_taken,
               sel_trimmed=s.trimmed_from_last)
    rows = s.token_ids[s.token_ids < 1200]
    o, w = R.approx_attention(q, K, V, rows)
    out.update(att_values=V, att_rows=rows, att_out=o, att_weights=w)
    rng = np.random.default_rng(3)
    sizes = rng.integers(1, 60, 64).astype(np.uint32)
    sel = np.full((25, 12), -1, np.int64)
    c = R.cache(2)
    for i in range(25):
        k = int(rng.integers(0, 12))
        ids = np.sort(rng.choice(64, k, replace=False)).astype(np.uint32)
        sel[i, :k] = ids
        c.lookup_and_update(ids, sizes)
    out.update(cache_sel=sel, cache_sizes=sizes, cache_counters=c.counters())
    dk = to_bf16_representable(tr.decode_keys[:16])
    cc, ll, _ = R.cluster_decode_batch(m.centroids, m.labels, dk, ClusterConfig(seed=km_seed))
    out.update(dec_keys=dk, dec_centroids=cc, dec_labels=ll)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
