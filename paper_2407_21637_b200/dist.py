"""Multi-GPU HODLR matvec: the cluster tree sharded at level L = log2(P)
(north_star "tree sharded at level log2(P)").

One process per GPU.  Rank g owns level-L node g: its rows, its whole subtree
(levels L+1..l and its leaves) and the row slices of the level-1..L factors
that touch its rows.  Per matvec (Alg. 3, split by rows):

  1. ``shard_begin``: send = [V'_k[own rows]^T x_own for k = 1..L] (Σ_k rmax_k·s
     values, a few KB);
  2. ``all_gather_into_tensor(recv, send)`` over NCCL/NVLink, asynchronous, while
     ``shard_local`` computes b_own = D x + Σ_{k>L} U_k t_k (the single-vector
     fused kernel) on the compute stream;
  3. ``shard_end``: t_k = Σ over the sibling subtree's ranks of recv (rank order),
     b_own += U_k[own rows] t_k.

Coefficients, not x, cross NVLink: an x all-gather would move (P-1)/P·n·s·8 B.
The host logic here (row ranges, exchange layout, the protocol) is backend-
agnostic: ``ShardedOperator`` drives any object with the HodlrOperator shard
interface, so the gloo CPU tests run it with an emulated local operator.
"""

from __future__ import annotations

import numpy as np

__all__ = ["levels_of", "shard_geometry", "exchange_layout", "ShardedOperator"]


def levels_of(nranks: int) -> int:
    """L = log2(nranks), the tree level the shards are cut at."""
    if nranks < 1 or nranks & (nranks - 1):
        raise ValueError(f"nranks must be a power of two (got {nranks})")
    return nranks.bit_length() - 1


def shard_geometry(H, rank: int, nranks: int):
    """(L, row0, n_local) of rank's shard: level-L node ``rank`` of the tree
    (mirrors hodlr_create_sharded's row range; equal to hodlr_info)."""
    L = levels_of(nranks)
    if L > H.depth:
        raise ValueError("more ranks than level-depth nodes (nranks > 2^depth)")
    if not 0 <= rank < nranks:
        raise ValueError("rank out of range")
    a, b = H.tree.ranges[L][rank]
    return L, int(a), int(b - a)


def exchange_layout(H, nranks: int):
    """Per external level k = 1..L: (slot, rmax_k); total count per unit s.

    The send buffer of every rank is [level 1 | level 2 | ... | level L], each
    level rmax_k = max rank over that level's blocks columns wide (slots past a
    node's own rank hold 0), times s right-hand sides, column-major in s:
    send[(slot_k + c) * s + q]."""
    L = levels_of(nranks)
    slots, off = [], 0
    for k in range(1, L + 1):
        rmax = max(max(up.rank, lo.rank) for up, lo in _level_pairs(H, k))
        slots.append((off, rmax))
        off += rmax
    return slots, off


def _level_pairs(H, k):
    if hasattr(H, "blocks"):
        return H.blocks[k - 1]
    return [(up, lo) for kk, _i, _r1, _r2, up, lo in H.offdiag_blocks() if kk == k]


class ShardedOperator:
    """b_own = (H x)[own rows] across ``nranks`` processes.

    ``backend_op`` defaults to the device operator
    (``linops.HodlrOperator(H, device, rank, nranks)``, the C ABI's sharded
    handle); any object with ``exchange_count/shard_begin/shard_local/shard_end``
    and ``row0/n_local`` works (the CPU tests pass an emulator)."""

    def __init__(self, H, rank=None, nranks=None, device=None, group=None, backend_op=None, use_graph=None):
        import os

        import torch.distributed as tdist

        # use_graph: replay the whole step (phase A, all-gather, phase B: 4-6 launches
        # of 5-70 us each at P = 8) as ONE captured CUDA graph per (x, out) buffer
        # pair; any capture failure falls back to eager launches for that pair
        self.use_graph = (os.environ.get("HODLR_B200_SHARD_GRAPH", "0") == "1") if use_graph is None else bool(use_graph)
        self._graphs = {}
        self.graph_replays = 0

        self.group = group
        self.rank = tdist.get_rank(group) if rank is None else int(rank)
        self.nranks = tdist.get_world_size(group) if nranks is None else int(nranks)
        self.L, self.row0, self.n_local = shard_geometry(H, self.rank, self.nranks)
        if backend_op is None:
            from .linops import HodlrOperator

            backend_op = HodlrOperator(H, device, self.rank, self.nranks)
        self.op = backend_op
        if (self.op.row0, self.op.n_local) != (self.row0, self.n_local):
            raise RuntimeError("backend shard geometry disagrees with the tree")
        self.working_format = H.working_format
        self._bufs = {}

    def _buffers(self, s, like):
        import torch

        key = (s, like.dtype, like.device)
        if key not in self._bufs:
            count = self.op.exchange_count(s)
            send = torch.zeros(count, dtype=like.dtype, device=like.device)
            recv = torch.zeros(count * self.nranks, dtype=like.dtype, device=like.device)
            self._bufs[key] = (send, recv)
        return self._bufs[key]

    def exchange_bytes(self, s=1, itemsize=8):
        return self.op.exchange_count(s) * itemsize

    def matvec(self, x_local, out=None):
        """x_local: (n_local,) or (n_local, s) tensor on this rank's device, in
        the working dtype; returns b_own in the same shape."""
        import torch
        import torch.distributed as tdist

        if not isinstance(x_local, torch.Tensor):
            raise TypeError("ShardedOperator.matvec expects a torch tensor on this rank's device")
        vec = x_local.dim() == 1
        X = x_local.reshape(-1, 1) if vec else x_local
        if X.dim() != 2 or X.shape[0] != self.n_local:
            raise ValueError(f"length mismatch: x_local has {X.shape[0]} rows, shard has {self.n_local}")
        X = self.op.as_working(X)  # device check + single RNE rounding to the working dtype
        if X.stride(1) != 1:
            X = X.contiguous()
        B = out if out is not None else torch.empty_like(X)
        if out is not None and (B.dtype != X.dtype or B.device != X.device or tuple(B.shape) != tuple(X.shape)
                                or B.stride(1) != 1):
            raise ValueError("out has the wrong shape / dtype / device / layout")
        send, recv = self._buffers(X.shape[1], X)
        if not (self.use_graph and X.is_cuda and self._replay(X, B, send, recv)):
            self._step(X, B, send, recv)
        return B[:, 0] if (vec and out is None) else B

    def _step(self, X, B, send, recv):
        import torch.distributed as tdist

        self.op.shard_begin(X, send)
        work = None
        if send.numel():
            work = tdist.all_gather_into_tensor(recv, send, group=self.group, async_op=True)
        self.op.shard_local(X, B)  # overlaps the exchange
        if work is not None:
            work.wait()
        self.op.shard_end(X, recv, B)

    def _replay(self, X, B, send, recv) -> bool:
        """Replay (capturing on first use) the step for this buffer pair; False -> run eagerly."""
        import torch

        key = (X.data_ptr(), B.data_ptr(), tuple(X.shape), X.stride(0), B.stride(0), X.dtype)
        g = self._graphs.get(key)
        if g is None:
            try:
                cur = torch.cuda.current_stream(X.device)
                side = torch.cuda.Stream(X.device)
                side.wait_stream(cur)
                with torch.cuda.stream(side):
                    for _ in range(2):  # warm up on the capture stream: its workspace, NCCL channels
                        self._step(X, B, send, recv)
                side.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    self._step(X, B, send, recv)
                cur.wait_stream(side)
            except Exception:  # capture not possible here: eager launches from now on
                g = False
            self._graphs[key] = g
        if g is False:
            return False
        g.replay()
        self.graph_replays += 1
        return True
