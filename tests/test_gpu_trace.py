"""A CKVT trace (paper_2412_03213_b200/trace.py) through the device session:
write a synthetic trace, read it memory-mapped, upload it (bf16), prefill and
one decode step; the selection and attention must match the CPU oracle run on
the same (bf16-rounded) trace data."""
import numpy as np
import pytest

from oracle.oracle import ClusterConfig as OCfg
from oracle.oracle import to_bf16_representable
from tests._inputs import port

pytestmark = pytest.mark.gpu


def test_trace_roundtrip_through_session(gpu_ctx, tmp_path):
    import torch

    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200 import trace as T
    from paper_2412_03213_b200.api import ClusterConfig
    from paper_2412_03213_b200.session import Session
    L, Tn, heads = 1040, 16, 2
    trs = [port().generate_head(port().mix_seed(7, 0, h), L, Tn) for h in range(heads)]
    b = T.TraceBundle(1, heads, [T.HeadTrace(t.prompt_keys, t.prompt_values, t.decode_queries,
                                             t.decode_keys, t.decode_values) for t in trs],
                      {"generator": "test"})
    path = str(tmp_path / "t.ckvt")
    T.write_trace(b, path)
    rb = T.read_trace(path)
    K, V, Q = T.to_device(rb, gpu_ctx.device)
    sess = Session(heads, 1, L, 4, 256, retention=1, cfg=ClusterConfig(), kv_heads=heads,
                   flags=N.CKV_SESSION_TOKEN_IDS, ctx=gpu_ctx)
    sess.K[:, :L].copy_(K)
    sess.V[:, :L].copy_(V)
    sess.prefill()
    q = Q[:, 0].contiguous()
    out = torch.empty((heads, 128), dtype=torch.float32, device=gpu_ctx.device)
    kn = K[:, 0].contiguous()
    sess.step(q, kn, V[:, 0].contiguous(), out)
    st = sess.state()
    for h in range(heads):
        Kh = to_bf16_representable(trs[h].prompt_keys)
        Vh = to_bf16_representable(trs[h].prompt_values)
        qh = to_bf16_representable(trs[h].decode_queries[0])
        o = port().cluster_prefill(Kh, OCfg(seed=port().mix_seed(0, 0, h)))
        sel = port().select_tokens(qh, o.centroids, o.labels, 16, 256)
        nt = int(st["n_tokens"][h].item())
        assert np.array_equal(st["token_ids"][h, :nt].cpu().numpy(), sel.token_ids)
        oo, _ = port().approx_attention(qh, Kh, Vh, sel.token_ids)
        assert np.abs(out[h].cpu().numpy() - oo).max() <= 2e-5 * np.abs(Vh).max()
