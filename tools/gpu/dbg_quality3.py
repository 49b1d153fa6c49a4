import faulthandler, sys, time, os
sys.path.insert(0, os.getcwd())
faulthandler.dump_traceback_later(60, exit=True)
import numpy as np, torch, ctypes as C
from tests.test_gpu_quality import _bundle, GOLD
from paper_2412_03213_b200 import _native as N
from paper_2412_03213_b200.api import ClusterConfig, Context
from paper_2412_03213_b200.session import Session
g = np.load(GOLD)
bundle, spec = _bundle(g)
ctx = Context.default(); dev = ctx.device; h = ctx.h; Lb = N.lib()
U, L, T, B = 4, 600, 50, 96
def bits(name):
    x = torch.from_numpy(np.stack([getattr(tr, name) for tr in bundle.traces])).to(dev)
    return x.to(torch.bfloat16).view(torch.int16).contiguous()
Kp, Vp, dK, dV = bits("prompt_keys"), bits("prompt_values"), bits("decode_keys"), bits("decode_values")
Qd = torch.from_numpy(np.stack([tr.decode_queries for tr in bundle.traces])).to(dev)
sess = Session(U, 1, L, T, B, retention=1, cfg=ClusterConfig(decode_batch=16, c0_divisor=40), kv_heads=2, flags=N.CKV_SESSION_TOKEN_IDS, ctx=ctx)
sess.K[:, :L].copy_(Kp); sess.V[:, :L].copy_(Vp)
sess.prefill()
P = L + T
Kpos = torch.zeros((U, P, 128), dtype=torch.int16, device=dev); Vpos = torch.zeros_like(Kpos)
Kpos[:, :L].copy_(Kp); Vpos[:, :L].copy_(Vp)
truth = torch.zeros((U, B), dtype=torch.int32, device=dev)
rec = torch.zeros(U, dtype=torch.float64, device=dev)
out = torch.zeros((U, 128), dtype=torch.float32, device=dev)
st = sess.state()
def sync(tag):
    torch.cuda.synchronize(); print(tag, flush=True)
q = Qd[:, 0].contiguous()
sess.step(q, dK[:, 0].contiguous(), dV[:, 0].contiguous(), out); sync("step")
N.check(Lb.ckv_exact_topb(h, U, 1, L, P, q.data_ptr(), Kpos.data_ptr(), B, truth.data_ptr(), B)); sync("topb")
N.check(Lb.ckv_recall(h, U, st["token_ids"].data_ptr(), st["sel_cap"], st["n_tokens"].data_ptr(), truth.data_ptr(), B, B, rec.data_ptr())); sync("recall")
print(rec.cpu().numpy())
rr = torch.zeros((U, 1), dtype=torch.int32, device=dev); ro = torch.zeros((U, 2), dtype=torch.int32, device=dev); rc = torch.zeros(U, dtype=torch.int32, device=dev)
runs = N.Runs(rr.data_ptr(), ro.data_ptr(), rc.data_ptr(), 1); fnt = torch.zeros(U, dtype=torch.int32, device=dev)
N.check(Lb.ckv_full_runs(h, U, L, C.byref(runs), fnt.data_ptr())); sync("full_runs")
print(rr.tolist(), ro.tolist(), rc.tolist(), fnt.tolist())
exact = torch.zeros((U, 128), dtype=torch.float32, device=dev)
ad = N.AttendDesc(U, 1, P, L, L)
N.check(Lb.ckv_attend(h, C.byref(ad), q.data_ptr(), Kpos.data_ptr(), Vpos.data_ptr(), None, C.byref(runs), fnt.data_ptr(), exact.data_ptr(), None)); sync("attend")
