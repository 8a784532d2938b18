"""The Fig. 4 harness (SPEC.md:600-607 cmd_matvec) and the
strict-order kernels behind its bf16 column.

CPU part: the problem generators against the SPEC's worked examples and the
oracle's narrow-working C loop against reference-generated goldens
(tests/golden/make_golden_r2.py).  GPU part: the strict-order kernels are
bit-identical to the reference's Arithmetic(working) outputs, and the sweep
satisfies Theorem 3.5 wherever its hypothesis holds (acceptance 5).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_case
from oracle.matvec import matvec_oracle

NARROW = ("bf16", "fp16", "q52")
NARROW_CASES = ["g512_fp64", "toep1024_e4_fp64", "rand96_fp32", "toep512_e3_fp64", "depth0_fp32", "g600_bf16"]


def same_bits(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture(scope="module")
def narrow():
    with np.load(os.path.join(GOLDEN, "narrow_golden.npz")) as z:
        return {k: z[k] for k in z.files}


def golden_path(name):
    return os.path.join(GOLDEN, ("nwhodlr_" if name == "g600_bf16" else "hodlr_") + name + ".npz")


def load_h(name):
    from paper_2407_21637_b200.model import load_hodlr

    return load_hodlr(golden_path(name))


# ---------------------------------------------------------------- CPU
def test_problem_generators_match_spec_examples():
    from paper_2407_21637_b200 import experiments as ex

    assert np.array_equal(ex.grid_1d(3)[:, 0], [0.0, 0.5, 1.0])
    g = ex.grid_1d(2000)[:, 0]
    assert g[0] == 0.0 and g[-1] == 1.0 and abs((g[1] - g[0]) - 1 / 1999) < 1e-15
    assert np.array_equal(ex.grid_2d(4), [[-1, -1], [-1, 1], [1, -1], [1, 1]])
    assert np.array_equal(ex.grid_2d(1), [[-1, -1]])
    P = ex.grid_2d(2000)
    assert P.shape == (2000, 2) and np.unique(P[:, 0]).size == 45  # m = 45 grid, first 2000 points
    # kernel (i) on {0, 0.5}: [[1, -2], [2, 1]]
    assert np.array_equal(ex.kernel_matrix("i", np.array([[0.0], [0.5]])), [[1.0, -2.0], [2.0, 1.0]])
    K1 = ex.paper_matrix("mat-1", 64)
    off = ~np.eye(64, dtype=bool)
    assert np.array_equal(K1[off], -K1.T[off])                    # antisymmetric off the diagonal
    K2 = ex.kernel_matrix("ii", np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 0.0]]))
    assert K2[0, 1] == 0.0 and K2[0, 2] == 0.0 and K2[0, 0] == 0.0  # coincident points -> 0; log 1 = 0
    K3 = ex.paper_matrix("mat-3", 50)
    assert np.all(np.diag(K3) == 1.0) and np.array_equal(K3, K3.T)
    with pytest.raises(ValueError):
        ex.kernel_matrix("i", ex.grid_2d(4))
    assert ex.main(["matvec", "--trials", "0"]) == 1               # usage error exit code


def test_trial_vectors_reproducible():
    from paper_2407_21637_b200.experiments import trial_vectors

    a, b = trial_vectors(100, 3, 7), trial_vectors(100, 3, 7)
    assert np.array_equal(a, b) and np.all(np.abs(a) < 1.0) and not np.array_equal(a, trial_vectors(100, 3, 8))


@pytest.mark.parametrize("name", NARROW_CASES)
@pytest.mark.parametrize("w", NARROW)
def test_oracle_narrow_working_matches_reference(narrow, name, w):
    """The oracle's strict-sequential C loop == the reference's Arithmetic(w)."""
    H = load_h(name)
    got = matvec_oracle(H, narrow[f"{name}__x"], w)
    assert same_bits(got, narrow[f"{name}__{w}"])


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", NARROW_CASES)
@pytest.mark.parametrize("w", NARROW)
def test_gpu_narrow_working_bit_identical_to_reference(cuda, narrow, name, w):
    """linops.matvec in a simulated low working precision reproduces the
    reference arithmetic bit for bit (host and device entry points)."""
    from paper_2407_21637_b200 import NAMED_FORMATS, linops

    H = load_h(name)
    X = narrow[f"{name}__x"]
    want = narrow[f"{name}__{w}"]
    op = linops.HodlrOperator(H, device=0)
    assert op.path(X.shape[1], NAMED_FORMATS[w])[0] == "strict"
    got = op.matvec(cuda.from_numpy(X).cuda(), working=NAMED_FORMATS[w])
    assert got.dtype == cuda.float64 and same_bits(got.cpu().numpy(), want)
    assert same_bits(op.matvec_host(X, working=NAMED_FORMATS[w]), want)
    assert same_bits(linops.matvec(H, X[:, 0], NAMED_FORMATS[w]), want[:, 0])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g2000_fp32", "toep1024_e2_fp32", "rand96_fp32", "g512_e9_fp32"])
def test_gpu_strict_fp32_bit_identical_to_reference(cuda, name):
    """hodlr_matvec_strict in fp32 == the reference's Arithmetic(FP32) output
    recorded in the round-1 goldens (b_alg3), bit for bit."""
    from paper_2407_21637_b200 import FP32, linops

    H, vec, _ = load_case(name)
    op = linops.HodlrOperator(H, device=0)
    got = op.matvec_strict(cuda.from_numpy(vec["x"]).cuda(), working=FP32).cpu().numpy()
    assert same_bits(got.reshape(vec["b_alg3"].shape), vec["b_alg3"])


@pytest.mark.gpu
def test_gpu_strict_workspace_and_errors(cuda):
    import ctypes

    from paper_2407_21637_b200 import BF16, _lib, linops

    H = load_h("g600_bf16")
    op = linops.HodlrOperator(H, device=0)
    need = _lib.c_sz()
    _lib.check(_lib.lib().hodlr_workspace_size_for(op._h, 1, 0, 2, ctypes.byref(need)))
    assert need.value >= 600 * 2 * 8
    x = cuda.zeros((600, 2), dtype=cuda.float64, device="cuda")
    b = cuda.empty_like(x)
    ws = cuda.zeros(16, dtype=cuda.uint8, device="cuda")
    st = _lib.lib().hodlr_matvec(op._h, 1, x.data_ptr(), 2, b.data_ptr(), 2, 2, ws.data_ptr(), 16, None)
    assert st == _lib.HODLR_ERR_INVALID  # caller workspace too small
    with pytest.raises(ValueError):
        op.matvec(cuda.zeros(599, dtype=cuda.float64, device="cuda"), working=BF16)
    # a fast call and a strict call share the stream's workspace without disturbing each other
    xs = cuda.from_numpy(np.random.default_rng(0).uniform(-1, 1, 600)).cuda()
    b1 = op.matvec(xs, working=BF16).clone()
    op.matvec(xs.float(), working=linops.FP32)
    assert cuda.equal(op.matvec(xs, working=BF16), b1)


@pytest.mark.gpu
def test_fig4_sweep_bound_and_plateau(cuda):
    """A reduced Fig. 4 sweep: every cell whose hypothesis u <= eps/n holds
    satisfies Thm 3.5 (acceptance 5); the bf16 column plateaus near
    bf16's unit roundoff for small eps while fp64 tracks eps."""
    from paper_2407_21637_b200 import BF16, FP32, FP64
    from paper_2407_21637_b200.experiments import sweep_matvec

    rows = sweep_matvec(("mat-1", "mat-3"), n=2000, depth=8, eps_grid=(1e-2, 1e-7, 1e-10),
                        workings=(FP64, FP32, BF16), trials=3)
    assert len(rows) == 18
    cell = {(r["matrix"], r["eps"], r["working"]): r for r in rows}
    for r in rows:
        assert r["status"] != "VIOLATED", r
        if r["hypothesis_met"]:
            assert r["backward_error"] <= r["bound"]
        assert (r["kernel_path"] == "strict") == (r["working"] == "bf16")
    for m in ("mat-1", "mat-3"):
        e7, e10 = cell[(m, 1e-7, "bf16")]["backward_error"], cell[(m, 1e-10, "bf16")]["backward_error"]
        assert 0.1 <= e7 / e10 <= 10.0                              # plateau (acceptance 5)
        assert e10 > 1e-5                                           # ... near bf16's u, far above eps
        assert cell[(m, 1e-10, "fp64")]["backward_error"] < 1e-9    # fp64 tracks eps
        assert cell[(m, 1e-10, "fp64")]["backward_error"] < cell[(m, 1e-2, "fp64")]["backward_error"]
    assert not cell[("mat-1", 1e-7, "bf16")]["hypothesis_met"]
    assert cell[("mat-1", 1e-2, "fp64")]["hypothesis_met"]
