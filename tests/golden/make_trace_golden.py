"""Writes tests/golden/synthetic_small.ckvt with the compiled reference's own
generate_synthetic + write_trace (trace.hpp:200-225, 268-303) — the CKVT
golden fixture for tests/test_trace.py.  Needs oracle/_ref (built from
/root/reference); the committed file is what the GPU box and CI use.

    python tests/golden/make_trace_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle  # noqa: E402

SPEC = dict(n_centers=8, seed=7, L=48, T=6, d=128, n_layers=2, n_heads=2)


def main():
    R = Oracle("reference")
    path = os.path.join(HERE, "synthetic_small.ckvt")
    rc = R.lib.ref_write_synthetic_trace(path.encode(), SPEC["n_centers"], SPEC["seed"],
                                         SPEC["L"], SPEC["T"], SPEC["d"], SPEC["n_layers"],
                                         SPEC["n_heads"])
    assert rc == 0, R.lib.ref_last_error()
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
