"""bench.py's multi-rank plumbing (independent units,
no data-path collective; the reference's run_simulation fan-out,
harness.hpp:362-378): --gpus N re-execs under torchrun with one rank per
GPU, refuses N above the visible GPUs, and reports the max over ranks of the
per-rank device times.  CPU parts here (gloo, world 2); the shared-GPU run
of the whole bench at world 2 is in tests/test_gpu_bench_world.py."""
import os
import subprocess
import sys

import pytest

from tests._dist import run_world

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _max_rank(rank, world):
    import torch

    import bench
    return bench._max_over_ranks(torch, "cpu", world, [1.0 + rank, 10.0 - rank, 3.0])


def test_max_over_ranks_gloo_world2():
    res = run_world(2, "tests.test_bench_world", "_max_rank")
    assert res[0] == res[1] == [2.0, 10.0, 3.0]


def test_gpus_above_visible_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 64:
        pytest.skip("needs fewer than 64 visible GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.pop("CKV_BENCH_SHARE_GPU", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True,
                       env=env, timeout=300)
    assert r.returncode != 0
    assert "visible GPU" in r.stderr
