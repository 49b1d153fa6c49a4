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
