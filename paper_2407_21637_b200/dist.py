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

import json
import os
import time

import numpy as np

__all__ = ["shard_geometry", "exchange_layout", "ShardedOperator", "bench_sharded"]


def _levels(nranks: int) -> int:
    if nranks < 1 or nranks & (nranks - 1):
        raise ValueError(f"nranks must be a power of two (got {nranks})")
    return nranks.bit_length() - 1


def shard_geometry(H, rank: int, nranks: int):
    """(L, row0, n_local) of rank's shard: level-L node ``rank`` of the tree
    (mirrors hodlr_create_sharded's row range; equal to hodlr_info)."""
    L = _levels(nranks)
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
    L = _levels(nranks)
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

    def __init__(self, H, rank=None, nranks=None, device=None, group=None, backend_op=None):
        import torch.distributed as tdist

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

        vec = x_local.dim() == 1
        X = x_local.reshape(-1, 1) if vec else x_local
        if X.shape[0] != self.n_local:
            raise ValueError(f"length mismatch: x_local has {X.shape[0]} rows, shard has {self.n_local}")
        if X.stride(1) != 1:
            X = X.contiguous()
        B = out if out is not None else torch.empty_like(X)
        send, recv = self._buffers(X.shape[1], X)
        self.op.shard_begin(X, send)
        work = None
        if send.numel():
            work = tdist.all_gather_into_tensor(recv, send, group=self.group, async_op=True)
        self.op.shard_local(X, B)  # overlaps the exchange
        if work is not None:
            work.wait()
        self.op.shard_end(X, recv, B)
        return B[:, 0] if (vec and out is None) else B


# ------------------------------------------------------------------ benchmark
def _weak_workload(world, cfg):
    """Per-GPU work fixed at one cfg2-sized shard: n = 65536·P, depth 8 + log2 P,
    the cfg2 kernel A_ij = 1/(1+|i-j|), eps 1e-6, fp64 working."""
    from . import problems
    from .formats import FP64

    L = _levels(world)
    n, depth = 65536 * world, 8 + L
    H, x, src = problems.toeplitz_config(n, depth, 1e-6, FP64, 2)
    desc = (f"cfg2 weak-scaled: n=65536*{world}={n} depth={depth} leaf=256, A_ij=1/(1+|i-j|), eps=1e-6, "
            f"adaptive, fp64 working, 1 rhs; tree sharded at level {L}")
    return H, x, desc, (lambda v: problems.toeplitz_times(v)), src.frob2_all() ** 0.5


def bench_sharded(args, build_workload, alg_bytes, peaks, ClockSampler):
    """bench.py's N-GPU arm (torchrun, one rank per GPU, NCCL)."""
    import torch
    import torch.distributed as tdist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    opts = None
    try:
        opts = tdist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True  # the all-gather's CTAs go first next to the persistent kernel
    except Exception:
        opts = None
    kw = {"backend": "nccl", "device_id": dev}
    if opts is not None:
        kw["pg_options"] = opts
    tdist.init_process_group(**kw)
    try:
        return _bench_sharded(args, build_workload, alg_bytes, peaks, ClockSampler, rank, world, local, dev)
    finally:
        tdist.destroy_process_group()


def _bench_sharded(args, build_workload, alg_bytes, peaks, ClockSampler, rank, world, local, dev):
    import torch
    import torch.distributed as tdist

    weak = args.config == "2"
    t_build = time.perf_counter()
    if weak:
        H, x, desc, Kx, normA = _weak_workload(world, args.config)
    else:
        H, x, desc, Kx, normA = build_workload(args.config)
        desc += f"; tree sharded at level {_levels(world)} (strong scaling)"
    t_build = time.perf_counter() - t_build
    x = np.asarray(x).reshape(H.n, -1)
    s = x.shape[1]
    wb = 8 if H.working_format.name == "fp64" else 4
    dt = torch.float64 if wb == 8 else torch.float32
    sop = ShardedOperator(H, rank, world, device=local)
    op = sop.op
    r0, nl = sop.row0, sop.n_local
    xd = torch.from_numpy(np.ascontiguousarray(x[r0:r0 + nl])).to(dev).to(dt)
    bd = torch.empty_like(xd)
    flush = torch.ones((256 << 20) // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        sop.matvec(xd, out=bd)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # parity: gather b on every rank, rank 0 checks against the oracle and K x
    parts = [torch.empty_like(bd) for _ in range(world)]
    tdist.all_gather(parts, bd)
    parity = None
    if rank == 0:
        from oracle.matvec import matvec_oracle

        from .metrics import matvec_backward_error, matvec_bound

        b = torch.cat(parts).double().cpu().numpy()
        xw = x.astype(np.float32).astype(np.float64) if wb == 4 else x
        b_or = matvec_oracle(H, xw, "fp64")
        kx = np.asarray(Kx(xw if s > 1 else xw[:, 0])).reshape(H.n, s)
        beta = matvec_backward_error(kx, xw, b, normA)
        bound = matvec_bound(H.depth, H.eps)
        parity = {"rel_err_vs_oracle": float(np.linalg.norm(b - b_or) / np.linalg.norm(b_or)),
                  "backward_error": beta, "bound_thm35": bound, "within_10x_bound": beta <= 10 * bound}

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ClockSampler(local) as clocks:
        tdist.barrier()
        torch.cuda.synchronize()
        for i in range(K):
            flush.sum()  # read-only L2 flush, untimed
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        tdist.barrier()
        # e2e: pinned host x_own in, b_own out, every step
        Ke = max(10, K // 4)
        xh = torch.from_numpy(np.ascontiguousarray(x[r0:r0 + nl])).pin_memory()
        bh = torch.empty_like(xh).pin_memory()
        xe = torch.empty((nl, s), dtype=torch.float64, device=dev)

        def e2e_step():
            xe.copy_(xh, non_blocking=True)
            step_in = xe if dt == torch.float64 else xe.to(dt)
            sop.matvec(step_in, out=bd)
            bh.copy_(bd.double() if dt != torch.float64 else bd, non_blocking=True)

        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize()
        tdist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(Ke):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms_local = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    ms_e2e_local = e0.elapsed_time(e1) / Ke
    t = torch.tensor([ms_local, ms_e2e_local], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms, ms_e2e = float(t[0]), float(t[1])
    B_all = alg_bytes(H, s, wb)
    mb = torch.tensor([op.matrix_bytes + 2 * nl * s * wb], dtype=torch.float64, device=dev)
    tdist.all_reduce(mb, op=tdist.ReduceOp.MAX)
    if rank != 0:
        return 0
    peak, peak_src = peaks()
    per_gpu = float(mb[0])  # largest shard's algorithmic bytes (matrix rows + x + b)
    achieved = per_gpu / (ms * 1e-3) / 1e9
    units = world if weak else 1  # weak: one 65536-row (cfg2-sized) shard matvec per GPU per step
    value = units * 1000.0 / ms
    line = {
        "metric": "HODLR matvecs/sec", "value": value,
        "unit": _unit(weak),
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64" if wb == 8 else "f32",
        "data": "synthetic (seeded, BASELINE shapes)",
        "config": {
            "workload": desc, "n": H.n, "depth": H.depth, "s": s, "eps": H.eps,
            "level_formats": [f.name for f in H.plan.chosen],
            "global_matvecs_per_s": 1000.0 / ms, "alg_bytes_per_matvec": int(B_all),
            "alg_bytes_largest_shard": int(per_gpu), "effective_GBps_total": B_all / (ms * 1e-3) / 1e9,
            "exchange_bytes_per_rank": sop.exchange_bytes(s, wb),
            "l2": "flushed before every timed step (256 MiB read, untimed)",
            "build_seconds": t_build, "parallelism": f"tree sharded at level {_levels(world)} over {world} GPUs, "
                                                     "NCCL all-gather of V^T x coefficients",
        },
        "parity": parity,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_src,
                     "kernel": "whole sharded step per GPU (k_ext_v + k_stream subtree + k_ext_u, "
                               "all-gather overlapped)"},
        "e2e": {"value": units * 1000.0 / ms_e2e, "unit": _unit(weak), "h2d_bytes_per_step": int(H.n * s * 8),
                "d2h_bytes_per_step": int(H.n * s * 8), "ms_per_step": ms_e2e},
        "gpu_launches": K * (op.path(s)[1] + 3 * (world > 1)) * world,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def _unit(weak):
    return "matvec/s (cfg2-sized 65536-row shards)" if weak else "matvec/s"
