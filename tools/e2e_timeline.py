"""Timeline of the end-to-end (pinned host buffer) session step at config B:
CUPTI activity through torch.profiler, so the host API calls and the
kernels of each ckv_session_step land on one clock.  Prints, per step, the
offset of every runtime call and kernel from the call's start, and the
median host wall time of the call.

    python tools/e2e_timeline.py [steps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_03213_b200 import _native as N  # noqa: E402
from paper_2412_03213_b200.api import ClusterConfig, Context  # noqa: E402
from paper_2412_03213_b200.session import Session  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
dev = torch.device("cuda", 0)
U, G, L, B, D = 256, 4, 32768, 1024, 128
T = 64
ctx = Context(0)
sess = Session(U, G, L, T, B, retention=1, cfg=ClusterConfig(), kv_heads=8,
               flags=N.CKV_SESSION_L2_PERSIST, ctx=ctx)
g, centers = bench.gen_inputs(torch, dev, U, G, L, T)
bench.fill_kv(torch, dev, g, centers, sess.K, sess.V, L)
q_all, kn_all, vn_all = bench.gen_decode(torch, dev, g, centers, G, T)
sess.prefill()
n_q = U * G
qh = torch.empty((n_q, D), dtype=torch.float32).pin_memory()
kh = torch.empty((U, D), dtype=torch.int16).pin_memory()
vh = torch.empty((U, D), dtype=torch.int16).pin_memory()
oh = torch.empty((n_q, D), dtype=torch.float32).pin_memory()
lib = N.lib()
t = 0
walls = []


def one(record=False):
    global t
    qh.copy_(q_all[t].cpu()); kh.copy_(kn_all[t].cpu()); vh.copy_(vn_all[t].cpu())
    torch.cuda.synchronize()
    with torch.profiler.record_function("ckv_step"):
        h0 = time.perf_counter()
        N.check(lib.ckv_session_step(sess.h, qh.data_ptr(), kh.data_ptr(), vh.data_ptr(),
                                     oh.data_ptr(), 0))
        walls.append((time.perf_counter() - h0) * 1e6)
    t += 1


for _ in range(8):
    one()
walls.clear()
for _ in range(20):
    one()
print(f"wall per e2e call (no profiler): median {np.median(walls):.1f} us, min {min(walls):.1f}")
walls.clear()
act = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=act) as prof:
    for _ in range(steps):
        one()
evs = [e for e in prof.events()]
marks = sorted([e for e in evs if e.name == "ckv_step"], key=lambda e: e.time_range.start)
for m in marks[-3:]:
    s0, s1 = m.time_range.start, m.time_range.end
    print(f"--- step: host {s1 - s0:.1f} us")
    rows = []
    for e in evs:
        st = e.time_range.start
        if e is m or e.name == "ckv_step":
            continue
        if s0 - 1 <= st <= s1 + 50:
            rows.append((st - s0, e.time_range.end - st, e.device_type, e.name[:60]))
    for r in sorted(rows):
        print(f"  {r[0]:8.1f} +{r[1]:7.1f}  {str(r[2]).split('.')[-1]:5s} {r[3]}")
