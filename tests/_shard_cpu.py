"""CPU checker for the sequence-sharded k-means protocol (test-only).

`CpuShard` implements paper_2412_03213_b200.sharded.ShardSteps with the
oracle's restatement of the reference (oracle/ckv_oracle.c: AssignScorer,
cosine_distance) and exact f64 member sums, so the protocol in sharded.py
(collectives, repair, convergence) can run under gloo at world_size 2 on a
machine without a GPU.  It is test infrastructure: the product path binds
DeviceShard (the CUDA kernels) instead.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.oracle import Oracle

D = 128


class CpuShard:
    def __init__(self, keys: np.ndarray, C_: int):
        self.P = Oracle("port")
        self.keys = np.ascontiguousarray(keys, np.float32)  # [U][n_local][128]
        U, n, _ = self.keys.shape
        self.n_units, self.n_local, self.C = U, n, C_
        self.sums = torch.zeros((U, C_, D), dtype=torch.float64)
        self.counts = torch.zeros((U, C_), dtype=torch.int32)
        self.stat = torch.zeros((U, 4), dtype=torch.int32)
        self.objective = torch.zeros((U,), dtype=torch.float64)
        self.cents = np.zeros((U, C_, D), np.float32)
        self.lab = [np.zeros((U, n), np.int32), np.zeros((U, n), np.int32)]
        self.cur = 0
        self.active = np.ones(U, np.int32)

    def validate(self):
        for u in range(self.n_units):
            k = self.keys[u].astype(np.float64)
            self.stat[u, 1] = int(not np.isfinite(k).all())
            self.stat[u, 2] = int((np.sqrt((k * k).sum(1)) >= 1e-12).any())

    def init(self, rows, row_lo):
        s = self.sums.numpy()
        s[:] = 0.0
        for u in range(self.n_units):
            for c, r in enumerate(rows[u]):
                if row_lo <= r < row_lo + self.n_local:
                    s[u, c] = self.keys[u, r - row_lo]

    def set_active(self, active):
        self.active = np.array(active, np.int32)

    def update(self, from_init):
        s = self.sums.numpy()
        cnt = self.counts.numpy().astype(np.float64)
        for u in np.nonzero(self.active)[0]:
            den = 1.0 if from_init else cnt[u][:, None]
            with np.errstate(invalid="ignore", divide="ignore"):
                self.cents[u] = (s[u] / den).astype(np.float32)

    def assign(self, pass_):
        self.cur = pass_ & 1
        for u in range(self.n_units):
            if self.active[u]:
                self.lab[self.cur][u] = self.P.assign(self.keys[u], self.cents[u])
                self.counts[u] = torch.from_numpy(
                    np.bincount(self.lab[self.cur][u], minlength=self.C).astype(np.int32))
            else:
                self.counts[u] = 0

    def empty(self):
        c = self.counts.numpy()
        return np.array([int(self.active[u] and (c[u] == 0).any())
                         for u in range(self.n_units)], np.int32)

    def farthest(self, unit, cluster):
        best, row = -1.0, -1
        lab = self.lab[self.cur][unit]
        for i in range(self.n_local):
            if lab[i] != cluster:
                continue
            d = self.P.cosine_distance(self.keys[unit, i], self.cents[unit, cluster])
            if d > best:
                best, row = d, i
        return best, row

    def move(self, unit, local_row, cluster):
        self.lab[self.cur][unit, local_row] = cluster

    def finish(self, pass_, want_objective):
        for u in range(self.n_units):
            ch = 0
            if pass_ > 0 and self.active[u]:
                ch = int((self.lab[self.cur][u] != self.lab[self.cur ^ 1][u]).any())
            self.stat[u, 0] = ch
            if want_objective and self.active[u]:
                lab = self.lab[self.cur][u]
                self.objective[u] = sum(self.P.cosine_distance(self.keys[u, i],
                                                               self.cents[u, lab[i]])
                                        for i in range(self.n_local))

    def partial_sums(self):
        s = self.sums.numpy()
        for u in np.nonzero(self.active)[0]:
            s[u] = 0.0
            np.add.at(s[u], self.lab[self.cur][u], self.keys[u].astype(np.float64))

    def result(self, iters):
        labels = np.stack([self.lab[int(iters[u]) & 1][u] for u in range(self.n_units)])
        return torch.from_numpy(self.cents.copy()), torch.from_numpy(labels)
