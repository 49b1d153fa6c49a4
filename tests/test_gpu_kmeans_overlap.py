"""kmeans_run's two-stream split (CKV_KM_OVERLAP: a call of >= 16 units runs
its halves on two contexts / streams from two host threads) and the lagged
active-count read-back: a 19-unit batched ckv_kmeans must give, unit by unit,
the bits a one-unit call gives (which the oracle tests pin), including the
iteration counts, objective and repair logs."""
import ctypes as C

import numpy as np
import pytest

from tests._inputs import head

pytestmark = pytest.mark.gpu

D = 128


def _run(ctx, keys_u, C_, seeds, max_iters):
    import torch
    from paper_2412_03213_b200 import _native as N
    from paper_2412_03213_b200.api import _to_bf16_device
    lib = N.lib()
    U, n = keys_u.shape[0], keys_u.shape[1]
    kb = _to_bf16_device(ctx, keys_u.reshape(U * n, D), "kmeans")
    rows = np.zeros((U, C_), np.uint32)
    for u in range(U):
        lib.ckv_kmeans_init_rows(n, C_, int(seeds[u]), rows[u].ctypes.data)
    d_rows = torch.from_numpy(rows.view(np.int32).reshape(-1)).to(ctx.device)
    cents = torch.empty((U, C_, D), dtype=torch.float32, device=ctx.device)
    labels = torch.empty((U, n), dtype=torch.int32, device=ctx.device)
    desc = N.KMeansDesc(U, n, C_, max_iters, n * D, C_, n, N.CKV_KM_OBJECTIVE)
    info = (N.KMeansInfo * U)()
    obj = np.zeros(U * (max_iters + 1), np.float64)
    rep = np.zeros(U * (max_iters + 1), np.uint32)
    N.check(lib.ckv_kmeans(ctx.h, C.byref(desc), kb.data_ptr(), d_rows.data_ptr(),
                           cents.data_ptr(), labels.data_ptr(), C.cast(info, C.c_void_p),
                           obj.ctypes.data, rep.ctypes.data))
    its = [(int(i.iterations_used), bool(i.converged)) for i in info]
    return (cents.cpu().numpy(), labels.cpu().numpy(), its,
            obj.reshape(U, -1), rep.reshape(U, -1))


def test_kmeans_two_stream_split_matches_single_unit_calls(gpu_ctx):
    from oracle.oracle import to_bf16_representable
    U, n, C_, MI = 19, 4096, 51, 50
    keys = np.stack([to_bf16_representable(head(11, u // 8, u % 8, n + 16)["K"][16:])
                     for u in range(U)])
    seeds = np.arange(100, 100 + U)
    cb, lb, ib, ob, rb = _run(gpu_ctx, keys, C_, seeds, MI)
    for u in range(U):
        c1, l1, i1, o1, r1 = _run(gpu_ctx, keys[u:u + 1], C_, seeds[u:u + 1], MI)
        assert ib[u] == i1[0], u
        assert np.array_equal(lb[u], l1[0]), u
        assert np.array_equal(cb[u].view(np.uint32), c1[0].view(np.uint32)), u
        assert np.array_equal(rb[u], r1[0]), u
        np.testing.assert_allclose(ob[u], o1[0], rtol=1e-9, atol=1e-9)
