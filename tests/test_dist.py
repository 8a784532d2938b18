"""Multi-process tests of the sharded matvec's host side (dist.py) on CPU:
world_size 2 and 4 over gloo, the local compute emulated (shard_emulator.py),
the protocol, row ranges and exchange layout exactly as the NCCL path runs
them.  The device side of the same protocol is checked in
test_gpu_matvec.py::test_sharded_* against the same emulator."""

import json
import os
import socket

import numpy as np
import pytest

from conftest import random_hodlr

torch = pytest.importorskip("torch")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {
    # name: (n, depth, formats per level, ranks per level, s)
    "uniform": (1024, 4, ["fp64", "fp32", "bf16", "q52"], [6, 5, 4, 3], 1),
    "ragged_ranks": (1000, 3, ["fp32", "fp16", "fp64"], [(1, 7), (0, 5), (2, 4)], 3),
}


def _worker(rank, world, port, case, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as tdist

    from oracle.matvec import matvec_oracle
    from paper_2407_21637_b200.dist import ShardedOperator
    from shard_emulator import EmulatedShard

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        n, depth, fmts, ranks, s = CASES[case]
        H = random_hodlr(n, depth, fmts, ranks, seed=11)
        X = np.random.default_rng(5).standard_normal((n, s))
        sop = ShardedOperator(H, backend_op=EmulatedShard(H, tdist.get_rank(), tdist.get_world_size()))
        xl = torch.from_numpy(np.ascontiguousarray(X[sop.row0:sop.row0 + sop.n_local]))
        b1 = sop.matvec(xl)
        b2 = sop.matvec(xl)  # buffers reused across calls
        sizes = [None] * world
        tdist.all_gather_object(sizes, (sop.row0, sop.n_local))
        parts = [None] * world
        tdist.all_gather_object(parts, b1.numpy())
        if rank == 0:
            assert [r for r, _ in sizes] == sorted(r for r, _ in sizes)
            assert sum(m for _, m in sizes) == n
            b = np.concatenate(parts, axis=0)
            ref = matvec_oracle(H, X)
            res = {"rel": float(np.linalg.norm(b - ref) / np.linalg.norm(ref)),
                   "repeat_equal": bool(np.array_equal(b1.numpy(), b2.numpy())),
                   "exchange": sop.exchange_bytes(s)}
            with open(os.path.join(outdir, "result.json"), "w") as f:
                json.dump(res, f)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", sorted(CASES))
def test_sharded_protocol_gloo(tmp_path, world, case):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _port(), case, str(tmp_path)), nprocs=world, join=True)
    res = json.load(open(tmp_path / "result.json"))
    assert res["rel"] <= 1e-12, res
    assert res["repeat_equal"]
    assert res["exchange"] > 0


def test_shard_geometry_and_layout():
    from paper_2407_21637_b200.dist import exchange_layout, shard_geometry

    H = random_hodlr(1000, 3, ["fp32", "fp16", "fp64"], [(1, 7), (0, 5), (2, 4)], seed=3)
    rows = [shard_geometry(H, g, 4) for g in range(4)]
    assert all(L == 2 for L, _, _ in rows)
    assert [r0 for _, r0, _ in rows] == [a for a, _ in H.tree.ranges[2]]
    assert sum(m for _, _, m in rows) == 1000
    slots, count = exchange_layout(H, 4)
    r1 = max(max(u.rank, l.rank) for u, l in H.blocks[0])
    r2 = max(max(u.rank, l.rank) for u, l in H.blocks[1])
    assert slots == [(0, r1), (r1, r2)] and count == r1 + r2
    assert exchange_layout(H, 1) == ([], 0)
    with pytest.raises(ValueError):
        shard_geometry(H, 0, 3)
    with pytest.raises(ValueError):
        shard_geometry(H, 0, 16)  # more ranks than level-depth nodes
