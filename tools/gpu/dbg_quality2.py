import faulthandler, sys, time, os
sys.path.insert(0, os.getcwd())
faulthandler.dump_traceback_later(60, exit=True)
import numpy as np, torch, ctypes as C
from tests.test_gpu_quality import _bundle, GOLD
from paper_2412_03213_b200 import quality as Q, _native as N
from paper_2412_03213_b200.api import ClusterConfig, Context
from paper_2412_03213_b200.session import Session
g = np.load(GOLD)
bundle, spec = _bundle(g)
ctx = Context.default(); dev = ctx.device
U, L, T = 4, 600, 50
def bits(name):
    x = torch.from_numpy(np.stack([getattr(tr, name) for tr in bundle.traces])).to(dev)
    return x.to(torch.bfloat16).view(torch.int16).contiguous()
Kp, Vp, dK, dV = bits("prompt_keys"), bits("prompt_values"), bits("decode_keys"), bits("decode_values")
Qd = torch.from_numpy(np.stack([tr.decode_queries for tr in bundle.traces])).to(dev)
sess = Session(U, 1, L, T, 96, retention=1, cfg=ClusterConfig(decode_batch=16, c0_divisor=40), kv_heads=2, flags=N.CKV_SESSION_TOKEN_IDS, ctx=ctx)
sess.K[:, :L].copy_(Kp); sess.V[:, :L].copy_(Vp)
print("prefill", sess.prefill(), flush=True)
out = torch.zeros((U, 128), dtype=torch.float32, device=dev)
for t in range(20):
    sess.step(Qd[:, t].contiguous(), dK[:, t].contiguous(), dV[:, t].contiguous(), out)
    torch.cuda.synchronize()
    print("step", t, flush=True)
    print(sess.cache_counters()[:, :2].tolist(), flush=True)
