"""How much of a unit's selected KV the G q heads share at config B: per
unit, |union of the heads' token sets| / sum of their sizes, over a few
decode steps (the bytes a GQA-union attention would read vs per-head).

    python tools/gqa_overlap.py [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_03213_b200 import _native as N  # noqa: E402
from paper_2412_03213_b200.api import ClusterConfig, Context  # noqa: E402
from paper_2412_03213_b200.session import Session  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device("cuda", 0)
layers, kvh, G, L, B = 32, 8, 4, 32768, 1024
U = layers * kvh
T = steps + 8
ctx = Context(0)
sess = Session(U, G, L, T, B, retention=1, cfg=ClusterConfig(max_iters=8), kv_heads=kvh,
               flags=N.CKV_SESSION_TOKEN_IDS, ctx=ctx)
g, centers = bench.gen_inputs(torch, dev, U, G, L, T, seed=7)
bench.fill_kv(torch, dev, g, centers, sess.K, sess.V, L)
q_all, kn_all, vn_all = bench.gen_decode(torch, dev, g, centers, G, T)
sess.prefill()
out = torch.empty((U * G, 128), dtype=torch.float32, device=dev)
tot_sum = tot_union = 0
for t in range(steps):
    sess.step(q_all[t], kn_all[t], vn_all[t], out)
    torch.cuda.synchronize()
    st = sess.state()
    ids, nt = st["token_ids"].cpu(), st["n_tokens"].cpu()
    s_sum = s_union = 0
    for u in range(U):
        sets = [set(ids[u * G + h, : int(nt[u * G + h])].tolist()) for h in range(G)]
        s_sum += sum(len(x) for x in sets)
        s_union += len(set().union(*sets))
    tot_sum += s_sum
    tot_union += s_union
    print(f"step {t}: per-head rows {s_sum}, union rows {s_union}, ratio {s_union / s_sum:.3f}")
print(f"overall union / sum = {tot_union / tot_sum:.3f}")
