"""BASELINE configs 3 and 4 (point-kernel sources, multi-RHS) through the
matrix-free device builder and the CUDA matvec.

Same-distribution analogs at sizes the CPU oracle finishes in seconds, plus
(``-m "gpu and slow"``) the full BASELINE sizes.  Tolerances:
  * vs the oracle (the same H evaluated by the CPU restatement of Alg. 3):
    fp64 working 1e-12, fp32 working 1e-5 (relative, Frobenius over X);
  * judged: ||B - K X||_F / (||K||_F ||X||_F) <= 10 c(l) eps (Thm 3.5).
"""

import numpy as np
import pytest

from conftest import matvec_bound
from oracle.matvec import matvec_oracle

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def check(H, X, src, tol_oracle):
    import torch

    from paper_2407_21637_b200 import linops, problems

    op = linops.HodlrOperator(H)
    dt = torch.float64 if H.working_format.name == "fp64" else torch.float32
    B = op.matvec(torch.from_numpy(X).cuda().to(dt)).double().cpu().numpy()
    ref = matvec_oracle(H, X, "fp64")  # H in binary64: both working precisions approximate it
    assert rel(B, ref) <= tol_oracle
    KX = problems.kernel_times(src, X)
    beta = np.linalg.norm(B - KX) / (np.sqrt(src.frob2_all()) * np.linalg.norm(X))
    assert beta <= 10 * matvec_bound(H.depth, H.eps), beta
    return beta


def test_cfg4_analog(cuda):
    from paper_2407_21637_b200 import problems

    H, X, src = problems.cfg4(n=1 << 15, depth=7, s=16)
    assert H.working_format.name == "fp64"
    assert all(f.name in ("q52", "bf16", "fp16", "fp32", "fp64") for f in H.plan.chosen)
    check(H, X, src, 1e-12)


def test_cfg3_analog(cuda):
    from paper_2407_21637_b200 import problems

    H, X, src = problems.cfg3(n=8192, depth=5, s=8)
    assert H.working_format.name == "fp32"
    check(H, X, src, 1e-5)


def test_point_source_tiles_match_dense(cuda):
    """Tiled products / norms of the matrix-free source == the dense block."""
    import torch

    from paper_2407_21637_b200 import problems

    P = np.random.default_rng(7).random((3000, 2))
    src = problems.PointKernelSource(P[problems.morton_order(P)], lambda r: torch.exp(-r / 0.2))
    src.tile = 700
    A = src.block(0, 3000, 0, 3000).cpu().numpy()
    X = np.random.default_rng(8).standard_normal((3000 - 1200, 3))
    Y = src._apply(100, 1400, 1200, 3000, torch.from_numpy(X).cuda()).cpu().numpy()
    assert np.allclose(Y, A[100:1400, 1200:3000] @ X, rtol=1e-12, atol=1e-12)
    assert abs(src.block_frob2(100, 1400, 1200, 3000) - np.sum(A[100:1400, 1200:3000] ** 2)) < 1e-9
    assert abs(src.frob2_all() - np.sum(A * A)) < 1e-8 * np.sum(A * A)


@pytest.mark.slow
def test_cfg4_full(cuda):
    from paper_2407_21637_b200 import problems

    H, X, src = problems.cfg4()
    check(H, X, src, 1e-12)


@pytest.mark.slow
def test_cfg3_full(cuda):
    from paper_2407_21637_b200 import problems

    H, X, src = problems.cfg3()
    check(H, X, src, 1e-5)
