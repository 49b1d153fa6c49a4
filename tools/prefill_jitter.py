"""Back-to-back ckv_cluster_prefill calls at config B (256 units x 32k):
per call the CUDA-event time, the host wall time, and (with
CKV_TRACE_HOST=1) the host timestamps of each phase on stderr."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_03213_b200 import _native as N  # noqa: E402
from paper_2412_03213_b200.api import Context  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 12
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
torch.cuda.synchronize()
for i in range(calls):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    N.check(lib.ckv_cluster_prefill(ctx.h, C.byref(desc), K.data_ptr(), C.cast(seeds, C.c_void_p),
                                    cents.data_ptr(), labels.data_ptr(), ncl.data_ptr(),
                                    C.cast(info, C.c_void_p), None, None))
    e1.record()
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    print(f"call {i}: event {e0.elapsed_time(e1):.2f} ms  wall {(w1 - w0) * 1e3:.2f} ms", flush=True)
