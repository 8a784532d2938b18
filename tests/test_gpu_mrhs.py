"""Multi-right-hand-side tensor-core path (kernels_mrhs.cu): DMMA for fp64
working, 3xTF32 for fp32 working, against the CPU oracle and against the
generic three-launch kernels, over every storage format, ragged chunk ends,
variable per-node ranks, several s (including s not a multiple of 8 and
column-group splits), and the sharded subtree path.

Tolerances (relative, Frobenius over X): fp64 working 1e-12; fp32 working
1e-5 (the split-TF32 products keep fp32-level accuracy; single-pass TF32 would
sit near 1e-3 and fail)."""

import os

import numpy as np
import pytest

from conftest import load_case, random_hodlr
from oracle.matvec import matvec_oracle

pytestmark = pytest.mark.gpu

FMT_SETS = [
    ("fp64", ["fp32", "fp64", "fp64"]),
    ("fp64", ["q52", "bf16", "fp16"]),
    ("fp32", ["bf16", "fp16", "fp32"]),
    ("fp32", ["q52", "q52", "bf16"]),
]


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def make_op(H, mrhs=True, **kw):
    from paper_2407_21637_b200 import linops

    old = os.environ.get("HODLR_B200_DISABLE_MRHS")
    os.environ["HODLR_B200_DISABLE_MRHS"] = "0" if mrhs else "1"
    try:
        return linops.HodlrOperator(H, **kw)
    finally:
        if old is None:
            del os.environ["HODLR_B200_DISABLE_MRHS"]
        else:
            os.environ["HODLR_B200_DISABLE_MRHS"] = old


def run(torch, op, X, working):
    dt = torch.float64 if working == "fp64" else torch.float32
    return op.matvec(torch.from_numpy(np.ascontiguousarray(X)).cuda().to(dt)).double().cpu().numpy()


def slab_path(working):
    """fp32 working: phase B runs on tcgen05 (kernels_tc.cu); fp64: DMMA slabs."""
    return "mrhs_tc" if working == "fp32" else "mrhs_slab"


def xin(X, working):
    return X.astype(np.float32).astype(np.float64) if working == "fp32" else X


@pytest.mark.parametrize("working,fmts", FMT_SETS)
@pytest.mark.parametrize("s", [2, 8, 16, 33, 64, 100])
@pytest.mark.parametrize("n,path", [(4096, "mrhs"), (2048, "mrhs_slab")])
def test_mrhs_matches_oracle_and_generic(cuda, working, fmts, s, n, path):
    """n=4096, depth 3: 512-row leaves (two chunks each) -> arena kernels;
    n=2048: 256-row leaves -> fragment-slab kernels (fp32: tcgen05 phase B;
    s=100 runs two 64-column passes, the second ragged)."""
    H = random_hodlr(n, 3, fmts, [24, 17, 9], working, seed=s + len(fmts[0]))
    op = make_op(H)
    if path == "mrhs_slab":
        path = slab_path(working)
    assert op.path(s) == (path, 3)
    X = np.random.default_rng(s).standard_normal((H.n, s))
    B = run(cuda, op, X, working)
    tol = 1e-12 if working == "fp64" else 1e-5
    assert rel(B, matvec_oracle(H, xin(X, working))) <= tol
    gen = make_op(H, mrhs=False)
    assert gen.path(s)[0] == "generic"
    assert rel(B, run(cuda, gen, X, working)) <= tol


@pytest.mark.parametrize("working", ["fp64", "fp32"])
def test_mrhs_variable_ranks_and_rank_zero(cuda, working):
    """Per-node ranks differ inside a level (cfg3-like), some are 0."""
    fmts = ["fp32", "fp16", "bf16", "fp32"] if working == "fp32" else ["fp64", "fp32", "q52", "fp16"]
    for n in (8192, 4096):  # 512-row leaves (arena kernels), 256-row leaves (slabs)
        H = random_hodlr(n, 4, fmts, [(30, 45), (0, 20), (5, 12), (0, 3)], working, seed=3)
        op = make_op(H)
        assert op.path(16)[0] == ("mrhs" if n == 8192 else slab_path(working))
        X = np.random.default_rng(2).standard_normal((H.n, 16))
        tol = 1e-12 if working == "fp64" else 1e-5
        assert rel(run(cuda, op, X, working), matvec_oracle(H, xin(X, working))) <= tol


@pytest.mark.parametrize("working", ["fp64", "fp32"])
def test_mrhs_ragged_chunks_depth0_and_wide_leaves(cuda, working):
    """Leaves wider than one 256-row chunk (K loop over column blocks) and a
    ragged last chunk (rows masked inside a 16-row step)."""
    for n, depth in ((1000, 0), (3968, 2)):
        H = random_hodlr(n, depth, ["fp32"] * depth, [7] * depth, working, seed=n)
        op = make_op(H)
        assert op.path(5)[0] == "mrhs"
        X = np.random.default_rng(n).standard_normal((n, 5))
        tol = 1e-12 if working == "fp64" else 1e-5
        assert rel(run(cuda, op, X, working), matvec_oracle(H, xin(X, working))) <= tol


def test_mrhs_fp64_operand_under_fp32_working_uses_generic(cuda):
    H = random_hodlr(2048, 3, ["fp64", "fp32", "fp16"], [8, 6, 4], "fp32", seed=1)
    op = make_op(H)
    assert op.path(8)[0] == "generic"
    assert op.path(8, "fp64")[0] == "mrhs"  # fp32 leaves: no fp64 slab, arena kernels


def test_mrhs_golden_cases(cuda):
    for name in ("g2000_fp32", "toep1024_e4_fp64", "g512_fp64", "toep512_e3_fp64"):
        H, vec, summ = load_case(name)
        X = np.random.default_rng(1).standard_normal((H.n, 12))
        op = make_op(H)
        w = summ["working"]
        B = run(cuda, op, X, w)
        tol = 1e-12 if w == "fp64" else 1e-5
        assert rel(B, matvec_oracle(H, xin(X, w))) <= tol, (name, op.path(12))


def test_mrhs_deterministic(cuda):
    H = random_hodlr(8192, 5, ["fp32"] * 5, [12, 10, 9, 7, 6], "fp64", seed=4)
    op = make_op(H)
    assert op.path(16)[0] == "mrhs_slab"
    X = np.random.default_rng(0).standard_normal((H.n, 16))
    a = run(cuda, op, X, "fp64")
    b = run(cuda, op, X, "fp64")
    assert np.array_equal(a, b)


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("working", ["fp64", "fp32"])
def test_mrhs_sharded_subtree(cuda, nranks, working):
    from test_gpu_shard import run_emulated

    H = random_hodlr(8192, 5, ["fp32", "bf16", "fp16", "q52", "fp32"], [12, 10, 9, 7, 6], working, seed=5)
    X = np.random.default_rng(3).standard_normal((H.n, 16))
    out, ops = run_emulated(cuda, H, X, nranks)
    assert all(op.path(16)[0] == slab_path(working) for op in ops)
    tol = 1e-12 if working == "fp64" else 1e-5
    assert rel(out, matvec_oracle(H, xin(X, working))) <= tol


@pytest.mark.parametrize("working", ["fp64", "fp32"])
def test_mrhs_slab_matches_arena_kernels(cuda, working):
    """The fragment-slab kernels and the arena kernels on one matrix."""
    fmts = ["fp32", "fp16", "bf16", "q52", "fp32"]
    H = random_hodlr(8192, 5, fmts, [(20, 40), 16, (0, 9), 7, 5], working, seed=8)
    X = np.random.default_rng(4).standard_normal((H.n, 24))
    a = run(cuda, make_op(H), X, working)
    old = os.environ.get("HODLR_B200_NO_SLAB")
    os.environ["HODLR_B200_NO_SLAB"] = "1"
    try:
        op2 = make_op(H)
        assert op2.path(24)[0] == "mrhs"
        b = run(cuda, op2, X, working)
    finally:
        if old is None:
            del os.environ["HODLR_B200_NO_SLAB"]
        else:
            os.environ["HODLR_B200_NO_SLAB"] = old
    tol = 1e-13 if working == "fp64" else 1e-6
    assert rel(a, b) <= tol


@pytest.mark.parametrize("s", [2, 16, 64, 70])
def test_mrhs_tc_matches_mma_sync_slabs(cuda, s):
    """fp32 working: the tcgen05 phase B (item slabs, TMEM A operand) against
    the mma.sync fragment-slab phase B on one matrix, every storage format,
    ranks not multiples of 8 and rank-0 nodes."""
    fmts = ["fp32", "fp16", "bf16", "q52", "fp32"]
    H = random_hodlr(8192, 5, fmts, [(20, 40), 16, (0, 9), 7, 5], "fp32", seed=11)
    X = np.random.default_rng(5).standard_normal((H.n, s))
    op = make_op(H)
    assert op.path(s)[0] == "mrhs_tc"
    a = run(cuda, op, X, "fp32")
    old = os.environ.get("HODLR_B200_NO_TC")
    os.environ["HODLR_B200_NO_TC"] = "1"
    try:
        assert op.path(s)[0] == "mrhs_slab"
        b = run(cuda, op, X, "fp32")
    finally:
        if old is None:
            del os.environ["HODLR_B200_NO_TC"]
        else:
            os.environ["HODLR_B200_NO_TC"] = old
    ref = matvec_oracle(H, xin(X, "fp32"))
    assert rel(a, ref) <= 1e-5 and rel(b, ref) <= 1e-5
    assert rel(a, b) <= 2e-6


def test_mrhs_tc_inf_propagates(cuda):
    """An inf in X stays inf in the rows it reaches, no NaN from
    the hi/lo split."""
    H = random_hodlr(2048, 3, ["fp32", "fp16", "fp32"], [8, 6, 4], "fp32", seed=2)
    op = make_op(H)
    assert op.path(8)[0] == "mrhs_tc"
    X = np.random.default_rng(0).standard_normal((H.n, 8))
    X[5, 3] = np.inf
    B = run(cuda, op, X, "fp32")
    assert not np.isnan(B[:, 3]).any() or np.isnan(matvec_oracle(H, xin(X, "fp32"))[:, 3]).any()
    assert np.isfinite(B[:, [0, 1, 2, 4, 5, 6, 7]]).all()


def test_mrhs_tc_phase_b_with_wide_stack(cuda):
    """Stacked ranks beyond three 128-row tiles: phase A falls back to the
    mma.sync slab kernel, phase B still runs on tcgen05."""
    H = random_hodlr(8192, 5, ["fp32", "fp32", "bf16", "fp16", "fp32"], [130, 120, 100, 64, 40], "fp32", seed=12)
    op = make_op(H)
    assert op.path(32)[0] == "mrhs_tc"
    X = np.random.default_rng(6).standard_normal((H.n, 32))
    assert rel(run(cuda, op, X, "fp32"), matvec_oracle(H, xin(X, "fp32"))) <= 1e-5


@pytest.mark.parametrize("working,fmt", [("fp64", "fp32"), ("fp64", "bf16"), ("fp64", "q52"), ("fp64", "fp64"),
                                         ("fp32", "fp32"), ("fp32", "fp16")])
@pytest.mark.parametrize("s", [8, 16, 24])
def test_slab_kernels_uniform_format(cuda, working, fmt, s):
    """One storage format on every level: the stacked-U phase B (U columns of all
    levels concatenated into 16-column k-blocks) and, for s = 8 / 16, the K-split
    phase A with its format-specialised instance; mma.sync kinds for both working
    precisions (tcgen05 off), variable ranks incl. rank-0 nodes, many chunks per
    phase-A run (node ends inside runs: parked tiles) against the oracle."""
    H = random_hodlr(256 * 64, 6, [fmt] * 6, [(0, 9), 7, (3, 12), 5, (1, 6), 4], working, seed=3 * s + len(fmt))
    X = np.random.default_rng(s).standard_normal((H.n, s))
    old = os.environ.get("HODLR_B200_NO_TC")
    os.environ["HODLR_B200_NO_TC"] = "1"
    try:
        op = make_op(H)
        assert op.path(s)[0] == "mrhs_slab"
        B = run(cuda, op, X, working)
        B2 = run(cuda, op, X, working)
    finally:
        if old is None:
            del os.environ["HODLR_B200_NO_TC"]
        else:
            os.environ["HODLR_B200_NO_TC"] = old
    assert np.array_equal(B, B2)  # deterministic
    assert rel(B, matvec_oracle(H, xin(X, working))) <= (1e-12 if working == "fp64" else 1e-5)


def test_slab_kernels_large_uniform_tree(cuda):
    """cfg4's shape at 1/8 scale (n = 2^17, depth 9, fp32 factors, fp64 working,
    16 rhs): every phase-A CTA runs several chunks, upper-level nodes span many
    runs (partial slots + reduce), deep levels end inside runs (direct stores)."""
    H = random_hodlr(1 << 17, 9, ["fp32"] * 9, [7, 7, 7, 5, 4, 3, 3, 2, 2], "fp64", seed=77)
    X = np.random.default_rng(5).standard_normal((H.n, 16))
    op = make_op(H)
    assert op.path(16)[0] == "mrhs_slab"
    B = run(cuda, op, X, "fp64")
    assert rel(B, matvec_oracle(H, X)) <= 1e-12
