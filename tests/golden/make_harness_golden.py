"""Writes tests/golden/harness_small.npz: the reference harness's own
run_simulation (harness.hpp:362-410, ClusterKV policy; compiled unmodified
from /root/reference into oracle/_ref) on a small bf16-rounded synthetic
bundle, for a budget sweep, a retention and an async-clustering variant —
the golden for the GPU decode-loop quality driver
(paper_2412_03213_b200/quality.py, tests/test_gpu_quality.py).  The bundle
itself is regenerated bit-exactly by the oracle port (generator pinned to the
reference in tests/test_oracle.py), so only the outputs are committed.

    python tests/golden/make_harness_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle  # noqa: E402

SPEC = dict(n_centers=8, seed=7, L=600, T=50, n_layers=2, n_heads=2)
COMMON = dict(decode_batch=16, c0_divisor=40)
RUNS = {
    "b48": dict(budget=48),
    "b96": dict(budget=96),
    "b200": dict(budget=200),
    "b96_r2": dict(budget=96, retention=2),
    "b96_async3": dict(budget=96, async_clustering=True, async_delay=3),
}


def main():
    R = Oracle("reference")
    out = {f"spec_{k}": np.array(v) for k, v in SPEC.items()}
    for k, v in COMMON.items():
        out[f"common_{k}"] = np.array(v)
    for name, kw in RUNS.items():
        r = R.run_simulation_synth(SPEC, **COMMON, **kw)
        for k, v in r.items():
            out[f"{name}__{k}"] = v
        for k, v in kw.items():
            out[f"{name}__cfg_{k}"] = np.array(v)
        print(name, r["summ_f"], r["summ_u"])
    np.savez_compressed(os.path.join(HERE, "harness_small.npz"), **out)


if __name__ == "__main__":
    main()
