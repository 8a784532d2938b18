"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
reference-built golden matrices, plus pack round-trip, KATs and edge cases.

Tolerances (stated here):
  * fp64 working: ||b_gpu - b_oracle|| <= 1e-12 ||b_oracle||   (self-parity)
  * fp32 working: ||b_gpu - b_oracle|| <= 1e-5  ||b_oracle||   (both are fp32
    evaluations of the same H; the oracle is strict left-to-right, the GPU
    blocked with FMA, each ~1e-7 from the exact product on these cases)
  * judged:       ||b_gpu - K x|| / (||K||_F ||x||) <= 10 * c(l) * eps,
    c(l) = 2(sqrt2+1) sqrt(2^(l+1) + 2^(l-1))   (Thm 3.5)
  * factor / leaf quantisation: bit-exact (unpacked device layout ==
    round_matrix of the input values).
"""

import numpy as np
import pytest

from conftest import golden_cases, load_case, matvec_bound
from oracle.fpsim import round_matrix
from oracle.matvec import matvec_oracle

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def tol_for(working):
    return 1e-12 if working == "fp64" else 1e-5


@pytest.mark.parametrize("name", golden_cases())
def test_matvec_host_path_parity(cuda, name):
    from paper_2407_21637_b200 import linops

    H, vec, summ = load_case(name)
    X = vec["x"]
    b_gpu = linops.matvec(H, X)
    b_or = matvec_oracle(H, X)
    assert b_gpu.shape == b_or.shape and b_gpu.dtype == np.float64
    assert rel(b_gpu, b_or) <= tol_for(summ["working"])
    xw = round_matrix(X, summ["working"])
    beta = np.linalg.norm(b_gpu - vec["KX"]) / (vec["normA"] * np.linalg.norm(xw))
    assert beta <= 10 * matvec_bound(summ["depth"], summ["eps"])


@pytest.mark.parametrize("name", golden_cases())
def test_matvec_device_path_parity(cuda, name):
    torch = cuda
    from paper_2407_21637_b200 import linops

    H, vec, summ = load_case(name)
    X = vec["x"]
    dt = torch.float64 if summ["working"] == "fp64" else torch.float32
    xd = torch.from_numpy(X).cuda().to(dt)
    op = linops.HodlrOperator(H)
    bd = op.matvec(xd)
    torch.cuda.synchronize()
    assert bd.dtype == dt
    b_or = matvec_oracle(H, X)
    assert rel(bd.double().cpu().numpy(), b_or) <= tol_for(summ["working"])
    # the 1-D vector form
    b1 = op.matvec(xd[:, 0]).double().cpu().numpy()
    assert rel(b1, matvec_oracle(H, X[:, 0])) <= tol_for(summ["working"])


@pytest.mark.parametrize("name", golden_cases())
def test_pack_roundtrip_bit_exact(cuda, name):
    from paper_2407_21637_b200 import linops

    H, _, _ = load_case(name)
    op = linops.HodlrOperator(H)
    idx = 0
    for _, _, _, _, up, lo in H.offdiag_blocks():
        for f in (up, lo):
            U, V = op.unpack_factor(idx, f.rows, f.cols, f.rank)
            assert np.array_equal(U, f.U) and np.array_equal(V, f.V)
            idx += 1
    for i, (a, b), D in H.leaves():
        assert np.array_equal(op.unpack_leaf(i, b - a), D)


@pytest.mark.parametrize("fmt", ["q52", "bf16", "fp16", "fp32", "fp64"])
def test_pack_quantises_raw_factors_bit_exactly(cuda, fmt):
    """store_factor semantics (lowrank.py:117-119): raw fp64 factors given to
    hodlr_create come back as round_matrix(raw, fmt), including overflow."""
    from paper_2407_21637_b200 import NAMED_FORMATS, linops, model

    rng = np.random.default_rng(7)
    n, depth = 96, 2
    T = model.build_tree(n, depth)
    leaves = [rng.standard_normal((b - a, b - a)) for a, b in T.ranges[depth]]
    F = NAMED_FORMATS[fmt]
    blocks, raws = [], []
    for k in range(1, depth + 1):
        lvl = []
        for i in range(2 ** (k - 1)):
            pair = []
            for rr, cc in ((T.ranges[k][2 * i], T.ranges[k][2 * i + 1]),
                           (T.ranges[k][2 * i + 1], T.ranges[k][2 * i])):
                U = rng.standard_normal((rr[1] - rr[0], 3)) * np.exp(rng.uniform(-12, 12, (rr[1] - rr[0], 3)))
                V = np.asfortranarray(rng.standard_normal((cc[1] - cc[0], 3)))
                pair.append(model.LowRankFactor(U, V, F))
                raws.append((U, V))
            lvl.append(tuple(pair))
        blocks.append(lvl)
    H = model.HodlrMatrix(T, leaves, blocks, 0.1, model.PrecisionPlan([F] * depth), NAMED_FORMATS["fp64"])
    op = linops.HodlrOperator(H)
    for idx, (U, V) in enumerate(raws):
        Ud, Vd = op.unpack_factor(idx, U.shape[0], V.shape[0], 3)
        assert np.array_equal(Ud, round_matrix(U, fmt))
        assert np.array_equal(Vd, round_matrix(V, fmt))


def test_identity_kat(cuda):
    """matvec(identity HODLR, x, fp64) -> x exactly."""
    from paper_2407_21637_b200 import FP64, linops, model

    n, depth = 1000, 3
    T = model.build_tree(n, depth)
    leaves = [np.eye(b - a) for a, b in T.ranges[depth]]
    blocks = []
    for k in range(1, depth + 1):
        blocks.append([tuple(model.LowRankFactor(np.zeros((r[1] - r[0], 0)), np.zeros((c[1] - c[0], 0)), FP64)
                             for r, c in ((T.ranges[k][2 * i], T.ranges[k][2 * i + 1]),
                                          (T.ranges[k][2 * i + 1], T.ranges[k][2 * i])))
                       for i in range(2 ** (k - 1))])
    H = model.HodlrMatrix(T, leaves, blocks, 0.0, model.PrecisionPlan([FP64] * depth), FP64)
    x = np.random.default_rng(0).standard_normal(n)
    assert np.array_equal(linops.matvec(H, x), x)


@pytest.mark.parametrize("s", [2, 5, 16, 33])
def test_multi_rhs(cuda, s):
    from paper_2407_21637_b200 import linops

    for name in ("g2000_fp32", "toep1024_e4_fp64"):
        H, _, summ = load_case(name)
        X = np.random.default_rng(s).standard_normal((H.n, s))
        assert rel(linops.matvec(H, X), matvec_oracle(H, X)) <= tol_for(summ["working"])


def test_working_override_fp32_on_fp64_matrix(cuda):
    from paper_2407_21637_b200 import FP32, linops

    H, vec, _ = load_case("toep1024_e4_fp64")
    b = linops.matvec(H, vec["x"][:, 0], FP32)
    assert rel(b, matvec_oracle(H, vec["x"][:, 0], "fp32")) <= 1e-5


def test_errors(cuda):
    from paper_2407_21637_b200 import linops
    from paper_2407_21637_b200.formats import parse_format

    H, vec, _ = load_case("g512_fp64")
    with pytest.raises(ValueError):
        linops.matvec(H, np.ones(H.n - 1))
    with pytest.raises(NotImplementedError):
        linops.matvec(H, np.ones(H.n), parse_format("custom:t=5,emin=-6,emax=7,bits=8"))


def test_overflow_propagates_inf(cuda):
    """Overflow is propagated, not trapped."""
    from paper_2407_21637_b200 import linops

    H, _, _ = load_case("toep1024_e2_fp32")
    x = np.zeros(H.n)
    x[3] = 3e38
    x[5] = 3e38
    b = linops.matvec(H, x)
    assert np.isinf(b).any()
