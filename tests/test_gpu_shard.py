"""GPU parity of the sharded matvec on one device: P sharded
handles side by side, the all-gather emulated by concatenating the send
buffers (no kernel waits on another rank's kernel).  Checks
  * C row ranges == dist.shard_geometry;
  * every rank's device send buffer == the CPU emulator's (same layout the
    gloo tests drive through dist.ShardedOperator), <= 1e-13 relative;
  * the assembled b == oracle (fp64: 1e-12, fp32: 1e-5), fused-subtree and
    generic local paths, s = 1 and s > 1;
  * ShardedOperator over a real NCCL process group of one rank.
"""

import os
import socket

import numpy as np
import pytest

from conftest import load_case, random_hodlr
from oracle.matvec import matvec_oracle

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def run_emulated(torch, H, X, nranks, check_send=True):
    from paper_2407_21637_b200 import linops
    from paper_2407_21637_b200.dist import shard_geometry
    from shard_emulator import EmulatedShard

    wdt = torch.float64 if H.working_format.name == "fp64" else torch.float32
    ops = [linops.HodlrOperator(H, rank=g, nranks=nranks) for g in range(nranks)]
    s = X.shape[1]
    count = ops[0].exchange_count(s)
    sends, xs = [], []
    for g, op in enumerate(ops):
        L, r0, nl = shard_geometry(H, g, nranks)
        assert (op.row0, op.n_local) == (r0, nl)
        xl = torch.from_numpy(np.ascontiguousarray(X[r0:r0 + nl])).cuda().to(wdt)
        send = torch.full((count,), float("nan"), dtype=wdt, device="cuda")
        op.shard_begin(xl, send)
        if check_send and count:
            emu = EmulatedShard(H, g, nranks)
            ref = torch.zeros(count, dtype=torch.float64)
            emu.shard_begin(torch.from_numpy(xl.double().cpu().numpy()), ref)
            got = send.double().cpu().numpy()
            assert np.isfinite(got).all(), "send slots left unwritten"
            # fp32: 1e-6 for the SIMT external-level kernels; the tensor-core
            # phase A (3xTF32, fragment slabs) sums hi/lo products: 1e-5
            slab = op.path(s)[0] in ("mrhs_slab", "mrhs_tc")
            assert rel(got, ref.numpy()) <= (1e-13 if wdt == torch.float64 else (1e-5 if slab else 1e-6))
        sends.append(send)
        xs.append(xl)
    recv = torch.cat(sends)
    out = np.zeros(X.shape)
    for op, xl in zip(ops, xs):
        bl = torch.empty_like(xl)
        op.shard_local(xl, bl)
        op.shard_end(xl, recv, bl)
        out[op.row0:op.row0 + op.n_local] = bl.double().cpu().numpy()
    return out, ops


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
@pytest.mark.parametrize("case", ["toep1024_e4_fp64", "g2000_fp32", "toep1024_e2_fp32"])
def test_sharded_golden_generic(cuda, nranks, case):
    H, vec, _ = load_case(case)
    X = vec["x"]
    out, _ = run_emulated(cuda, H, X, nranks)
    if H.working_format.name == "fp64":
        assert rel(out, matvec_oracle(H, X)) <= 1e-12
    else:
        assert rel(out, vec["b_alg3"]) <= 1e-5


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("working", ["fp64", "fp32"])
def test_sharded_fused_subtree(cuda, nranks, working):
    """Uniform per-level ranks/formats and 256-row leaves: each rank's subtree
    runs in the fused single-vector kernel (launch count says so)."""
    H = random_hodlr(8192, 5, ["fp64", "fp32", "bf16", "fp16", "q52"], [12, 10, 9, 7, 6], working=working, seed=4)
    X = np.random.default_rng(9).standard_normal((H.n, 1))
    out, ops = run_emulated(cuda, H, X, nranks)
    assert all(op.launches_per_matvec == 1 + 3 for op in ops), [op.launches_per_matvec for op in ops]
    ref = matvec_oracle(H, X.astype(np.float32).astype(np.float64) if working == "fp32" else X)
    assert rel(out, ref) <= (1e-12 if working == "fp64" else 1e-5)
    # multi-RHS through the same handles: generic local path
    X3 = np.random.default_rng(10).standard_normal((H.n, 3))
    out3, _ = run_emulated(cuda, H, X3, nranks, check_send=False)
    ref3 = matvec_oracle(H, X3.astype(np.float32).astype(np.float64) if working == "fp32" else X3)
    assert rel(out3, ref3) <= (1e-12 if working == "fp64" else 1e-5)


def test_sharded_repeat_deterministic(cuda):
    H = random_hodlr(8192, 5, ["fp64", "fp32", "bf16", "fp16", "q52"], [12, 10, 9, 7, 6], seed=4)
    X = np.random.default_rng(9).standard_normal((H.n, 1))
    a, _ = run_emulated(cuda, H, X, 4, check_send=False)
    b, _ = run_emulated(cuda, H, X, 4, check_send=False)
    assert np.array_equal(a, b)


def test_sharded_operator_nccl_world1(cuda):
    torch = cuda
    import torch.distributed as tdist

    from paper_2407_21637_b200.dist import ShardedOperator

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                             device_id=torch.device("cuda", 0))
    try:
        H, vec, _ = load_case("toep1024_e4_fp64")
        X = vec["x"]
        sop = ShardedOperator(H, device=0)
        b = sop.matvec(torch.from_numpy(np.ascontiguousarray(X)).cuda())
        assert rel(b.cpu().numpy(), matvec_oracle(H, X)) <= 1e-12
    finally:
        tdist.destroy_process_group()


def test_sharded_operator_graph_replay(cuda):
    """use_graph: the whole step replayed as one captured CUDA graph equals the
    eager launches bit for bit, on repeated calls and on the slab (s = 16) and
    fused (s = 1) paths."""
    torch = cuda
    from paper_2407_21637_b200.dist import ShardedOperator

    H = random_hodlr(8192, 5, ["fp32"] * 5, [7, 6, 5, 4, 3], "fp64", seed=21)
    for s in (16, 1):
        X = torch.from_numpy(np.random.default_rng(s).standard_normal((H.n, s))).cuda()
        eager = ShardedOperator(H, rank=0, nranks=1, device=0, use_graph=False)
        graph = ShardedOperator(H, rank=0, nranks=1, device=0, use_graph=True)
        want = eager.matvec(X).clone()
        out = torch.empty_like(X)
        for _ in range(3):
            out.zero_()
            graph.matvec(X, out=out)
            assert torch.equal(out, want)
        assert graph.graph_replays == 3
        X2 = X * 2.0  # another buffer pair: its own graph
        assert torch.equal(graph.matvec(X2), eager.matvec(X2))
        assert rel(want.cpu().numpy(), matvec_oracle(H, X.cpu().numpy())) <= 1e-12


def _nccl_worker(rank, world, port, path, q):
    import torch
    import torch.distributed as tdist

    from paper_2407_21637_b200.dist import ShardedOperator
    from paper_2407_21637_b200.model import load_hodlr

    torch.cuda.set_device(rank)
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                             device_id=torch.device("cuda", rank))
    try:
        H = load_hodlr(path)
        X = np.random.default_rng(3).standard_normal((H.n, 4))
        out = []
        for use_graph in (False, True):
            sop = ShardedOperator(H, device=rank, use_graph=use_graph)
            xl = torch.from_numpy(np.ascontiguousarray(X[sop.row0:sop.row0 + sop.n_local])).cuda()
            for _ in range(2):
                b = sop.matvec(xl)
            out.append(b.cpu().numpy())
        q.put((rank, sop.row0, out[0], out[1]))
    finally:
        tdist.destroy_process_group()


def test_sharded_operator_nccl_two_gpus(cuda):
    """Two processes, two GPUs, a real NCCL all-gather over NVLink (skipped on a
    one-GPU box): eager and graph-replayed steps both reproduce the oracle."""
    torch = cuda
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp

    from conftest import GOLDEN

    path = os.path.join(GOLDEN, "hodlr_toep1024_e4_fp64.npz")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(60)
    H, _, _ = load_case("toep1024_e4_fp64")
    X = np.random.default_rng(3).standard_normal((H.n, 4))
    want = matvec_oracle(H, X)
    for k in (2, 3):
        b = np.concatenate([g[k] for g in got])
        assert rel(b, want) <= 1e-12
