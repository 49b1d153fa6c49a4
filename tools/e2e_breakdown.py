"""Where the end-to-end decode step's time goes (config B session): host
copies, API / launch overhead and the device step.  Run on the GPU box."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2412_03213_b200 import _native as N
from paper_2412_03213_b200.session import Session
from paper_2412_03213_b200.api import ClusterConfig, Context

dev = torch.device("cuda", 0)
ctx = Context.default()
U, G, L, T, B = 256, 4, 32768, 64, 1024
D = 128
sess = Session(U, G, L, T, B, retention=1, cfg=ClusterConfig(), kv_heads=8, ctx=ctx)
g, centers = bench.gen_inputs(torch, dev, U, G, L, T)
bench.fill_kv(torch, dev, g, centers, sess.K, sess.V, L)
q_all, kn_all, vn_all = bench.gen_decode(torch, dev, g, centers, G, T)
sess.prefill()
n_q = U * G
qh = torch.empty((n_q, D), dtype=torch.float32).pin_memory()
kh = torch.empty((U, D), dtype=torch.int16).pin_memory()
vh = torch.empty((U, D), dtype=torch.int16).pin_memory()
oh = torch.empty((n_q, D), dtype=torch.float32).pin_memory()
out = torch.empty((n_q, D), dtype=torch.float32, device=dev)
lib = N.lib()
res = {"host_e2e": [], "dev_sync": [], "copies_only": []}
for t in range(40):
    qh.copy_(q_all[t].cpu()); kh.copy_(kn_all[t].cpu()); vh.copy_(vn_all[t].cpu())
    torch.cuda.synchronize()
    if t % 2 == 0:
        t0 = time.perf_counter()
        N.check(lib.ckv_session_step(sess.h, qh.data_ptr(), kh.data_ptr(), vh.data_ptr(), oh.data_ptr(), 0))
        res["host_e2e"].append((time.perf_counter() - t0) * 1e6)
    else:
        t0 = time.perf_counter()
        N.check(lib.ckv_session_step(sess.h, q_all[t].data_ptr(), kn_all[t].data_ptr(), vn_all[t].data_ptr(), out.data_ptr(), 1))
        torch.cuda.synchronize()
        res["dev_sync"].append((time.perf_counter() - t0) * 1e6)
    s = torch.cuda.current_stream()
    t0 = time.perf_counter()
    q_all[t].copy_(qh.view(n_q, D), non_blocking=True)
    oh.copy_(out, non_blocking=True)
    torch.cuda.synchronize()
    res["copies_only"].append((time.perf_counter() - t0) * 1e6)
print({k: round(float(np.median(v[2:])), 1) for k, v in res.items()})
