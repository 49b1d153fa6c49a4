"""The reference-signature C++ drop-in (include/clusterkv_b200/clusterkv.hpp)
runs end to end on the B200 kernels and matches the CPU oracle: k-means,
index, selection, scores, attention, decode-batch clustering, cache and the
ValidationError predicates (tests/cpp/shim_parity.cpp)."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_dropin_parity(gpu_ctx):
    from tests.cpp.build import build
    exe = build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim parity OK" in r.stdout
