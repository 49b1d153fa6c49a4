"""bench.py --gpus 2 end to end: the self-launched torchrun world (two
ranks sharing cuda:0 through CKV_BENCH_SHARE_GPU=1, gloo for the barrier and
the max over ranks, since one GPU is all a test box has), each rank running
its own batch row of units, rank 0 printing one JSON line with n_gpus 2."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_self_launches_two_ranks(gpu_ctx):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CKV_BENCH_SHARE_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "4", "--warmup", "3", "--e2e-steps", "3", "--layers", "2",
                        "--L", "4096", "--no-cpu", "--no-extra"],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 2
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert abs(line["value"] - 2 * 1000.0 / line["ms_per_step"]) < 1e-6 * line["value"]
