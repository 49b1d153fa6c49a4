"""The moved-cluster reduced assignment (opt-in CKV_MCR=1, ckv_assign_tc.cu)
must give the same k-means as the CPU oracle bit for bit.  Run in a
subprocess because the switch is read once per process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, sys
sys.path.insert(0, %r)
from tests._inputs import head, port
from tests.test_gpu_kmeans_tc import _batched_kmeans
for Cn, n, U in ((409, 8192, 3), (700, 6000, 2), (51, 4080, 2)):
    keys = np.stack([head(31, 0, u, n + 16)["K"][16:] for u in range(U)])
    seeds = [port().mix_seed(0, 5, u) for u in range(U)]
    c, l, info = _batched_kmeans(keys, Cn, seeds, 50, 0)
    for u in range(U):
        o = port().kmeans(keys[u], Cn, seeds[u], 50)
        assert info[u] == (o.iterations_used, o.converged), (Cn, u, info[u])
        assert np.array_equal(l[u], o.labels), (Cn, u)
        assert np.array_equal(c[u].view(np.uint32), o.centroids.view(np.uint32)), (Cn, u)
print("mcr ok")
""" % ROOT


def test_mcr_matches_oracle(gpu_ctx):
    env = dict(os.environ, CKV_MCR="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "mcr ok" in r.stdout, r.stdout + r.stderr
