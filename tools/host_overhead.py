"""Host-side cost of one ckv_session_step call (config B shape, short
prompt): wall time of back-to-back calls with device buffers (no sync) and
with pinned host buffers, and the synced per-step e2e time.

    python tools/host_overhead.py [L]
"""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_03213_b200 import _native as N  # noqa: E402
from paper_2412_03213_b200.api import ClusterConfig, Context  # noqa: E402
from paper_2412_03213_b200.session import Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = torch.device("cuda", 0)
U, G, B, D = 256, 4, 1024, 128
T = 400
ctx = Context(0)
flags = 0 if os.environ.get("CKV_NO_L2_PERSIST") else N.CKV_SESSION_L2_PERSIST
sess = Session(U, G, L, T, B, retention=1, cfg=ClusterConfig(max_iters=4), kv_heads=8, flags=flags,
               ctx=ctx)
g, centers = bench.gen_inputs(torch, dev, U, G, L, T, seed=7)
bench.fill_kv(torch, dev, g, centers, sess.K, sess.V, L)
q_all, kn_all, vn_all = bench.gen_decode(torch, dev, g, centers, G, T)
sess.prefill()
out = torch.empty((U * G, D), dtype=torch.float32, device=dev)
t = 0
for _ in range(5):
    sess.step(q_all[t], kn_all[t], vn_all[t], out); t += 1
torch.cuda.synchronize()
n = 100
h0 = time.perf_counter()
for _ in range(n):
    N.check(N.lib().ckv_session_step(sess.h, q_all[t].data_ptr(), kn_all[t].data_ptr(),
                                     vn_all[t].data_ptr(), out.data_ptr(), 1)); t += 1
h1 = time.perf_counter()
torch.cuda.synchronize()
print(f"device buffers: host {1e6 * (h1 - h0) / n:.1f} us per call")
qh = torch.empty((U * G, D), dtype=torch.float32).pin_memory()
kh = torch.empty((U, D), dtype=torch.int16).pin_memory()
vh = torch.empty((U, D), dtype=torch.int16).pin_memory()
oh = torch.empty((U * G, D), dtype=torch.float32).pin_memory()
qh.copy_(q_all[0].cpu()); kh.copy_(kn_all[0].cpu()); vh.copy_(vn_all[0].cpu())
torch.cuda.synchronize()
h0 = time.perf_counter()
for _ in range(n):
    N.check(N.lib().ckv_session_step(sess.h, qh.data_ptr(), kh.data_ptr(), vh.data_ptr(),
                                     oh.data_ptr(), 0)); t += 1
h1 = time.perf_counter()
torch.cuda.synchronize()
print(f"pinned host buffers: host {1e6 * (h1 - h0) / n:.1f} us per call")
es = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    a.record()
    N.check(N.lib().ckv_session_step(sess.h, qh.data_ptr(), kh.data_ptr(), vh.data_ptr(),
                                     oh.data_ptr(), 0)); t += 1
    b.record()
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    es.append((a.elapsed_time(b) * 1e3, (w1 - w0) * 1e6))
es = es[2:]
print(f"e2e per step: event {sum(e for e, _ in es) / len(es):.1f} us, wall {sum(w for _, w in es) / len(es):.1f} us")


def per_step(fn, reps=20):
    es = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        es.append((a.elapsed_time(b) * 1e3, (w1 - w0) * 1e6))
    es = es[2:]
    return sum(e for e, _ in es) / len(es), sum(w for _, w in es) / len(es)


def dev_step():
    global t
    N.check(N.lib().ckv_session_step(sess.h, q_all[t].data_ptr(), kn_all[t].data_ptr(),
                                     vn_all[t].data_ptr(), out.data_ptr(), 1)); t += 1


qp = torch.empty((U * G, D), dtype=torch.float32)
kp = torch.empty((U, D), dtype=torch.int16)
vp = torch.empty((U, D), dtype=torch.int16)
op = torch.empty((U * G, D), dtype=torch.float32)


def pageable_step():
    global t
    N.check(N.lib().ckv_session_step(sess.h, qp.data_ptr(), kp.data_ptr(), vp.data_ptr(),
                                     op.data_ptr(), 0)); t += 1


for name, fn in (("device buffers, synced", dev_step), ("pageable host buffers (staged)", pageable_step)):
    e, w = per_step(fn)
    print(f"{name}: event {e:.1f} us, wall {w:.1f} us")
