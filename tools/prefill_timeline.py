"""Kernel timeline of one config B ckv_cluster_prefill (CUPTI through
torch.profiler): per kernel name the launches and summed device time, the
call's span, and the GPU-busy time (union of kernel intervals), so idle gaps
between kernels show up.  python tools/prefill_timeline.py"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_03213_b200 import _native as N  # noqa: E402
from paper_2412_03213_b200.api import Context  # noqa: E402

dev = torch.device("cuda", 0)
U, L, D = 256, 32768, 128
ctx = Context(0)
K = torch.empty((U, L, D), dtype=torch.int16, device=dev)
V = torch.empty_like(K)
g, centers = bench.gen_inputs(torch, dev, U, 4, L, 0, seed=7)
bench.fill_kv(torch, dev, g, centers, K, V, L)
del V
lib = N.lib()
c_cap = lib.ckv_prefill_cluster_count(L, 80, 16, 0) + 64
cents = torch.empty((U, c_cap, D), dtype=torch.float32, device=dev)
labels = torch.empty((U, L), dtype=torch.int32, device=dev)
ncl = torch.empty((U,), dtype=torch.int32, device=dev)
seeds = (C.c_uint64 * U)(*[lib.ckv_mix_seed(0, u // 8, u % 8) for u in range(U)])
info = (N.KMeansInfo * U)()
desc = N.PrefillDesc(U, L, L, c_cap, 80, 16, 50, 0, 0)


def call():
    N.check(lib.ckv_cluster_prefill(ctx.h, C.byref(desc), K.data_ptr(), C.cast(seeds, C.c_void_p),
                                    cents.data_ptr(), labels.data_ptr(), ncl.data_ptr(),
                                    C.cast(info, C.c_void_p), None, None))
    torch.cuda.synchronize()


for _ in range(2):
    call()
act = [torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=act) as prof:
    call()
ks = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks.sort(key=lambda e: e.time_range.start)
t0, t1 = ks[0].time_range.start, max(e.time_range.end for e in ks)
busy, cur_s, cur_e = 0.0, None, None
for e in ks:
    s, f = e.time_range.start, e.time_range.end
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
agg = {}
for e in ks:
    k = e.name.split("(")[0].replace("void ", "")[:50]
    n, t = agg.get(k, (0, 0.0))
    agg[k] = (n + 1, t + e.time_range.end - e.time_range.start)
print(f"span {(t1 - t0) / 1e3:.2f} ms, GPU busy {busy / 1e3:.2f} ms, kernels {len(ks)}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"  {t / 1e3:8.2f} ms  {n:5d}  {k}")
