"""Per-rank bodies of the sharded-path tests (run under tests/_dist.py)."""
from __future__ import annotations

import numpy as np


def kmeans_rank(rank, world, keys, C_, seeds, max_iters, init_rows, device):
    """One rank of the sequence-sharded k-means on its contiguous shard of
    keys [U][N][128]; device = None -> the CPU checker, else a CUDA index
    (the CUDA kernels, collectives staged through gloo)."""
    import torch

    from paper_2412_03213_b200.sharded import Comm, kmeans_cosine_sharded, shard_range
    U, n_total, _ = keys.shape
    lo, hi = shard_range(n_total, world, rank)
    if device is None:
        from tests._shard_cpu import CpuShard
        shard = CpuShard(keys[:, lo:hi], C_)
    else:
        from paper_2412_03213_b200.api import Context
        from paper_2412_03213_b200.sharded import DeviceShard
        from tests._inputs import bf16_bits
        torch.cuda.set_device(device)
        kb = torch.from_numpy(bf16_bits(keys[:, lo:hi]).view(np.int16)).cuda(device)
        shard = DeviceShard(kb, C_, ctx=Context(device))
    r = kmeans_cosine_sharded(shard, n_total, lo, seeds=seeds, max_iters=max_iters,
                              init_rows=init_rows, comm=Comm(), want_objective=True)
    return dict(lo=lo, labels=r.labels.cpu().numpy(), centroids=r.centroids.cpu().numpy(),
                iters=r.iterations_used, converged=r.converged, reps=r.repair_iterations,
                obj=r.objective_history)


def decode_rank(rank, world, K, V, Q, Kr, Vr, C_, seeds, G, budget, device, full_rank=True,
                exact_scores=False):
    """Sharded prefill k-means + one sharded decode step (select + attend)
    on rank `rank`; K, V [U][L][128] prompt, Kr, Vr [U][n_rec][128] the
    recency rows (positions L..), Q [U*G][128].  Returns this rank's share."""
    import torch

    from paper_2412_03213_b200.api import Context
    from paper_2412_03213_b200.sharded import (Comm, DeviceShard, ShardedDecoder,
                                               kmeans_cosine_sharded, shard_range)
    from tests._inputs import bf16_bits
    torch.cuda.set_device(device)
    ctx = Context(device)
    comm = Comm()
    U, L, _ = K.shape
    n = L - 16
    lo, hi = shard_range(n, world, rank)
    dev = torch.device("cuda", device)
    t = lambda x: torch.from_numpy(bf16_bits(x).view(np.int16)).to(dev)
    # the rank's KV store in position order: sinks (rank 0), shard, recency
    # (last rank); the k-means reads its shard rows in place
    sink_rows = 16 if rank == 0 else 0
    n_rec = Kr.shape[1] if rank == world - 1 else 0
    Ks = np.concatenate([K[:, :sink_rows], K[:, 16 + lo:16 + hi], Kr[:, :n_rec]], 1)
    Vs = np.concatenate([V[:, :sink_rows], V[:, 16 + lo:16 + hi], Vr[:, :n_rec]], 1)
    Kst, Vst = t(Ks).contiguous(), t(Vs).contiguous()
    shard = DeviceShard(Kst[:, sink_rows:sink_rows + hi - lo], C_, ctx=ctx)
    km = kmeans_cosine_sharded(shard, n, lo, seeds=seeds, comm=comm)
    del shard
    dec = ShardedDecoder(km, Kst, Vst, G, budget, comm, sink_rows=sink_rows, n_rec=n_rec,
                         rec_pos=L, ctx=ctx)
    r = dec.step(torch.from_numpy(Q).to(dev), want_ids=True, want_weights=True, full_rank=full_rank,
                 exact_scores=exact_scores)
    ctx.sync()
    g = lambda x: x.cpu().numpy()
    return dict(out=g(r["out"]), ids=g(r["token_ids"]), w=g(r["weights"]),
                n_tokens=g(r["n_tokens"]), n_taken=g(r["n_taken"]), trimmed=g(r["trimmed"]),
                ranked=g(r["ranked"]), off=g(r["run_off"]), iters=km.iterations_used)


def sizes_rank(rank, world, labels_all, C_):
    """global_sizes / score_slice on CPU: each rank counts its shard's labels."""
    import torch

    from paper_2412_03213_b200.sharded import Comm, global_sizes, score_slice, shard_range
    U, n = labels_all.shape
    lo, hi = shard_range(n, world, rank)
    lsize = torch.from_numpy(np.stack([np.bincount(labels_all[u, lo:hi], minlength=C_)
                                       for u in range(U)]).astype(np.int32))
    g, p = global_sizes(Comm(), lsize)
    return dict(g=g.numpy(), p=p.numpy(), lsize=lsize.numpy(), slice=score_slice(C_, world, rank))
