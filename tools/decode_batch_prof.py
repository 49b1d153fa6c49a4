"""ckv_cluster_decode_batch at config D's shape (256 units, 320 new keys,
C+ = 4): a few calls, CUDA-event time per call (profile target for
k_kmeans_small under ncu)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_03213_b200 import _native as N  # noqa: E402
from paper_2412_03213_b200.api import Context  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
U, P, D, rows, c_cap = 256, 1024, 128, 320, 64
ctx = Context(0)
K = torch.empty((U, P, D), dtype=torch.int16, device=dev)
V = torch.empty_like(K)
g, centers = bench.gen_inputs(torch, dev, U, 4, P, 0, seed=3)
bench.fill_kv(torch, dev, g, centers, K, V, P)
lib = N.lib()
cents = torch.zeros((U, c_cap, D), dtype=torch.float32, device=dev)
labels = torch.full((U, P), -1, dtype=torch.int32, device=dev)
seeds = (C.c_uint64 * U)(*[lib.ckv_mix_seed(0, u // 8, u % 8) for u in range(U)])
its = (C.c_uint32 * U)()
for i in range(calls):
    ncl = torch.zeros((U,), dtype=torch.int32, device=dev)
    d = N.DecodeClusterDesc(U, 100 + i, rows, P, c_cap, 4, 50)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    N.check(lib.ckv_cluster_decode_batch(ctx.h, C.byref(d), K.data_ptr(), C.cast(seeds, C.c_void_p),
                                         cents.data_ptr(), labels.data_ptr(), ncl.data_ptr(),
                                         C.cast(its, C.c_void_p)))
    e1.record()
    torch.cuda.synchronize()
    print(f"call {i}: {e0.elapsed_time(e1) * 1e3:.1f} us, iterations min/max "
          f"{min(its)}/{max(its)}", flush=True)
