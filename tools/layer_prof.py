"""Layer-mode decode step (config B shape) diagnostics: device time per step
(CUDA events), host submission time per step (wall clock of the step calls
with no sync), the layer-batched step beside it.  Run under ncu with
--nvtx-free kernel filters to get the per-launch durations.

    python tools/layer_prof.py [steps] [max_iters]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_03213_b200.api import ClusterConfig, Context  # noqa: E402
from paper_2412_03213_b200.session import Session  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 50
dev = torch.device("cuda", 0)
layers, kvh, G, L, B = 32, 8, 4, 32768, 1024
U = layers * kvh
T = 4 * steps + 20
ctx = Context(0)
sess = Session(U, G, L, T, B, retention=1, cfg=ClusterConfig(max_iters=mi), kv_heads=kvh, ctx=ctx)
g, centers = bench.gen_inputs(torch, dev, U, G, L, T, seed=7)
bench.fill_kv(torch, dev, g, centers, sess.K, sess.V, L)
q_all, kn_all, vn_all = bench.gen_decode(torch, dev, g, centers, G, T)
sess.prefill()
out = torch.empty((U * G, 128), dtype=torch.float32, device=dev)
t = 0


def run(mode, n):
    global t
    sess.set_layer_units(mode)
    for _ in range(3):
        sess.step(q_all[t], kn_all[t], vn_all[t], out); t += 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(n):
        sess.step(q_all[t], kn_all[t], vn_all[t], out); t += 1
    h1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3, (h1 - h0) / n * 1e6


for mode in (0, kvh):
    d_us, h_us = run(mode, steps)
    print(f"layer_units={mode}: device {d_us:.1f} us/step, host submit {h_us:.1f} us/step", flush=True)
