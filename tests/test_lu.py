"""HODLR LU and triangular solves (Alg. 4, acceptance
7 and 9 at SPEC.md:655-657).  The reference ships no LU, so the oracle is the
dense unpivoted LU / dense triangular solve of the same matrices (the SPEC's own
"[DERIVED: dense oracle]" examples).  The recursion is exercised on the host
(device="cpu") in the CPU suite and on the GPU in the gpu suite.
"""

import numpy as np
import pytest

from conftest import load_case, random_hodlr


def dd_matrix(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    return A + np.diag(np.abs(A).sum(axis=1) + 1.0)


def build(A, depth, eps, working="fp64"):
    from paper_2407_21637_b200 import NAMED_FORMATS, build_tree
    from paper_2407_21637_b200.construct import DenseSource, build_adaptive

    W = NAMED_FORMATS[working]
    return build_adaptive(DenseSource(A), build_tree(A.shape[0], depth), eps, working=W,
                          available=tuple(NAMED_FORMATS[f] for f in ("q52", "bf16", "fp16", "fp32", "fp64")))


def dense_lu_nopivot(A):
    A = A.copy()
    n = A.shape[0]
    for j in range(n - 1):
        A[j + 1:, j] /= A[j, j]
        A[j + 1:, j + 1:] -= np.outer(A[j + 1:, j], A[j, j + 1:])
    return np.tril(A, -1) + np.eye(n), np.triu(A)


def check_suite(device):
    import torch

    from paper_2407_21637_b200 import lu as hl
    from paper_2407_21637_b200.formats import FP32, FP64
    from oracle.matvec import dense_of

    # identity -> L = U = I
    H = build(np.eye(64), 2, 1e-8)
    F = hl.lu(H, device=device)
    Ld, Ud = hl.reconstruct_lu(F)
    assert np.array_equal(Ld, np.eye(64)) and np.array_equal(Ud, np.eye(64))
    assert hl.lu_backward_error(np.eye(64), F) == 0.0

    # diagonally dominant 16 x 16, depth 1, eps 1e-12 -> 1e-10
    A = dd_matrix(16, 1)
    F = hl.lu(build(A, 1, 1e-12), device=device)
    assert hl.lu_backward_error(A, F) <= 1e-10
    Ld, Ud = hl.reconstruct_lu(F)
    assert np.array_equal(Ld, np.tril(Ld)) and np.all(np.diag(Ld) == 1.0) and np.array_equal(Ud, np.triu(Ud))
    L0, U0 = dense_lu_nopivot(A)
    assert np.allclose(Ld, L0, atol=1e-10) and np.allclose(Ud, U0, atol=1e-10)

    # depth 0: dense LU of the rounded matrix
    F = hl.lu(build(A, 0, 1e-3, "fp32"), device=device)
    A32 = A.astype(np.float32).astype(np.float64)
    assert hl.lu_backward_error(A32, F) <= 1e-5

    # Cor. 3.8 on diagonally dominant randoms, depths {2, 8} where the hypothesis holds
    for n, depth, eps, w in ((256, 2, 1e-6, FP64), (256, 8, 1e-8, FP64), (512, 2, 1e-10, FP64), (256, 2, 1e-2, FP32)):
        A = dd_matrix(n, n + depth)
        H = build(A, depth, eps, w.name)
        F = hl.lu(H, device=device)
        Ah = dense_of(H)
        Ld, Ud = hl.reconstruct_lu(F)
        err = hl.lu_backward_error(Ah, F)
        bound = hl.lu_bound(depth, eps, np.linalg.norm(Ah), np.linalg.norm(Ld), np.linalg.norm(Ud))
        assert hl.hypothesis_holds(w, eps, n)
        assert err <= bound, (n, depth, eps, w.name, err, bound)
        # solve through the factors
        x0 = np.random.default_rng(n).standard_normal((n, 3))
        x = hl.lu_solve(F, Ah @ x0)
        assert np.linalg.norm(x - x0) <= (1e3 * eps + (1e-4 if w is FP32 else 1e-10)) * np.linalg.norm(x0)

    # triangular solves: rank preservation, dense oracle, shape errors
    A = dd_matrix(128, 7)
    H = build(A, 2, 1e-12)
    F = hl.lu(H, device=device)
    Ld, Ud = hl.reconstruct_lu(F)
    rng = np.random.default_rng(2)
    tt = lambda a: torch.as_tensor(a, dtype=torch.float64, device=device)
    for r in (0, 2, 3):
        Ub, Vb = rng.standard_normal((128, r)), rng.standard_normal((128, r))
        W, V2 = hl.solve_lower(F.L, (tt(Ub), tt(Vb)))
        assert W.shape == (128, r) and V2.shape == (128, r)
        assert np.allclose(Ld @ W.cpu().numpy(), Ub, atol=1e-10)
        U2, W2 = hl.solve_upper_right((tt(Ub), tt(Vb)), F.U)
        assert W2.shape == (128, r) and np.allclose(U2.cpu().numpy() @ W2.cpu().numpy().T @ Ud, Ub @ Vb.T, atol=1e-9)
    Bd = rng.standard_normal((128, 5))
    assert np.allclose(Ld @ hl.solve_lower(F.L, tt(Bd)).cpu().numpy(), Bd, atol=1e-10)
    assert np.allclose(hl.solve_upper_right(tt(Bd.T.copy()), F.U).cpu().numpy() @ Ud, Bd.T, atol=1e-9)
    with pytest.raises(ValueError):
        hl.solve_lower(F.L, tt(np.zeros((127, 2))))
    with pytest.raises(ValueError):
        hl.solve_upper_right(tt(np.zeros((2, 127))), F.U)

    # schur_update: rank-0 update leaves H22 unchanged; exact cancellation collapses the ranks
    root = hl.to_nodes(H, device=device)
    z = tt(np.zeros((64, 0)))
    assert hl.schur_update(root.c2, (z, z), (z, z), 1e-12) is root.c2
    D22 = A[64:, 64:]
    Lz, Uz = tt(rng.standard_normal((64, 2))), tt(rng.standard_normal((64, 2)))
    core = tt(np.eye(2))
    S = hl.schur_update(root.c2, (Lz, core), (core, Uz), 1e-12)
    want = D22 - Lz.cpu().numpy() @ Uz.cpu().numpy().T
    assert np.linalg.norm(hl._dense(S).cpu().numpy() - want) <= 1e-10 * np.linalg.norm(want)
    Zn = hl.to_nodes(build(Lz.cpu().numpy() @ Uz.cpu().numpy().T, 1, 1e-13), device=device)
    C = hl.schur_update(Zn, (Lz, core), (core, Uz), 1e-8)
    assert C.upper[0].shape[1] == 0 and C.lower[0].shape[1] == 0
    assert float(C.c1.dense.abs().max()) <= 1e-12 and float(C.c2.dense.abs().max()) <= 1e-12

    # singular pivot -> error naming the leaf
    Z = np.eye(32)
    Z[20, 20] = 0.0
    with pytest.raises(hl.SingularPivotError, match="leaf 2"):
        hl.lu(build(Z, 2, 1e-8), device=device)
    with pytest.raises(NotImplementedError):
        from paper_2407_21637_b200 import BF16

        hl.lu(H, working=BF16, device=device)


def test_lu_recursion_on_host():
    pytest.importorskip("torch")
    check_suite("cpu")


def test_lu_needs_a_gpu_by_default():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2407_21637_b200 import lu as hl

    with pytest.raises(RuntimeError, match="GPU"):
        hl.lu(build(np.eye(8), 1, 1e-8))


@pytest.mark.gpu
def test_lu_on_gpu(cuda):
    check_suite("cuda")


@pytest.mark.gpu
def test_lu_of_reference_built_matrix_and_solve(cuda):
    """LU of a reference-built kernel matrix (golden container), then H x = b
    solved through the factors and checked with the GPU matvec."""
    from paper_2407_21637_b200 import linops
    from paper_2407_21637_b200 import lu as hl
    from oracle.matvec import dense_of

    H, vec, _ = load_case("g512_fp64")  # Gaussian kernel + nugget, depth 2, eps 1e-8
    F = hl.lu(H)
    Ah = dense_of(H)
    Ld, Ud = hl.reconstruct_lu(F)
    err = hl.lu_backward_error(Ah, F)
    assert err <= hl.lu_bound(H.depth, H.eps, np.linalg.norm(Ah), np.linalg.norm(Ld), np.linalg.norm(Ud))
    x0 = vec["x"][:, 0]
    b = linops.matvec(H, x0)
    x = hl.lu_solve(F, b)
    assert np.linalg.norm(linops.matvec(H, x) - b) <= 1e-6 * np.linalg.norm(b)
