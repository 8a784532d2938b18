"""CPU stand-in for a sharded device handle (test infrastructure only).

Implements the HodlrOperator shard interface (exchange_count, shard_begin,
shard_local, shard_end, row0, n_local) in numpy binary64 with exactly the
exchange layout the C ABI uses (include/hodlr_b200.h, dist.exchange_layout):
send[(slot_k + c) * s + q] = V'_{k,j}[own rows, c]^T x_own[:, q], j = rank's
level-k ancestor; shard_end sums the sibling subtree's ranks in rank order.
The GPU tests check the device send buffers against this emulator, so the
gloo tests of dist.py exercise the same protocol the NCCL path runs.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle.matvec import dense_of
from paper_2407_21637_b200.dist import exchange_layout, shard_geometry


def _node_factors(H, k, j):
    """(U_{k,j}, V'_{k,j}): U of the block whose rows are node j, V of the block
    whose columns are node j (plan.h re-keying)."""
    up, lo = H.blocks[k - 1][j // 2]
    return (up.U, lo.V) if j % 2 == 0 else (lo.U, up.V)


class EmulatedShard:
    def __init__(self, H, rank, nranks):
        self.H, self.rank, self.nranks = H, rank, nranks
        self.L, self.row0, self.n_local = shard_geometry(H, rank, nranks)
        self.slots, self.count = exchange_layout(H, nranks)
        own = slice(self.row0, self.row0 + self.n_local)
        # the subtree + leaves part: external blocks never meet (own, own)
        self.local_dense = dense_of(H)[own, own]

    def exchange_count(self, s=1):
        return self.count * s

    def _anc(self, k):
        j = self.rank >> (self.L - k)
        a, _ = self.H.tree.ranges[k][j]
        return j, self.row0 - a

    def as_working(self, X):
        if not isinstance(X, torch.Tensor) or X.is_cuda:
            raise TypeError("the CPU emulator takes CPU tensors")
        return X.to(torch.float64)

    def shard_begin(self, X, send):
        x = X.numpy()
        s = x.shape[1]
        out = np.zeros(self.count * s)
        for k in range(1, self.L + 1):
            slot, _ = self.slots[k - 1]
            j, off = self._anc(k)
            _, V = _node_factors(self.H, k, j)
            t = V[off:off + self.n_local].T @ x  # (r, s)
            out[slot * s:slot * s + t.size] = t.reshape(-1)
        send.copy_(torch.from_numpy(out))

    def shard_local(self, X, B):
        B.copy_(torch.from_numpy(self.local_dense @ X.numpy()))

    def shard_end(self, X, recv, B):
        s = X.shape[1]
        rv = recv.numpy().reshape(self.nranks, self.count * s)
        b = B.numpy().copy()
        for k in range(1, self.L + 1):
            slot, _ = self.slots[k - 1]
            j, off = self._anc(k)
            U, _ = _node_factors(self.H, k, j)
            r = U.shape[1]
            sib = j ^ 1
            g0, g1 = sib << (self.L - k), (sib + 1) << (self.L - k)
            t = rv[g0, slot * s:(slot + r) * s].copy()
            for g in range(g0 + 1, g1):
                t += rv[g, slot * s:(slot + r) * s]
            b += U[off:off + self.n_local] @ t.reshape(r, s)
        B.copy_(torch.from_numpy(b))
