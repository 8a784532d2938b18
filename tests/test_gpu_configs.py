"""BASELINE configs 3 and 4 (point-kernel sources, multi-RHS) through the
matrix-free device builder and the CUDA matvec.

Same-distribution analogs at sizes the CPU oracle finishes in seconds, plus
every BASELINE config at its full size (cfg2, cfg3, cfg4 and the five cfg5
precision-sweep points; builds take 2-40 s each on a B200).  Tolerances:
  * vs the oracle (the same H evaluated by the CPU restatement of Alg. 3):
    fp64 working 1e-12, fp32 working 1e-5 (relative, Frobenius over X);
  * judged: ||B - K X||_F / (||K||_F ||X||_F) <= 10 c(l) eps (Thm 3.5,
    PAPER.md:639-649), with the SPEC hypothesis flag u <= eps/n
     recorded beside it (the bound is only proven when it holds).
Each full-size case appends one JSON record (errors, bound, flag) to
gpurun_out/parity_full.jsonl when that directory exists.
"""

import json
import os

import numpy as np
import pytest

from conftest import matvec_bound
from oracle.matvec import matvec_oracle

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _record(name, H, rec):
    from paper_2407_21637_b200.metrics import hypothesis_holds

    rec = dict(case=name, n=H.n, depth=H.depth, eps=H.eps, working=H.working_format.name,
               level_formats=[f.name for f in H.plan.chosen],
               hypothesis_u_le_eps_over_n=bool(hypothesis_holds(H.working_format, H.eps, H.n)), **rec)
    print(json.dumps(rec))
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "parity_full.jsonl"), "a") as f:
            f.write(json.dumps(rec) + "\n")
    return rec


def check(H, X, src, tol_oracle, name=None, kx=None, normk=None):
    import torch

    from paper_2407_21637_b200 import linops, problems

    op = linops.HodlrOperator(H)
    dt = torch.float64 if H.working_format.name == "fp64" else torch.float32
    X = np.asarray(X, np.float64).reshape(H.n, -1)
    if dt == torch.float32:
        X = X.astype(np.float32).astype(np.float64)  # x pre-rounded to the working format
    B = op.matvec(torch.from_numpy(X).cuda().to(dt)).double().cpu().numpy()
    path = op.path(X.shape[1])[0]
    del op
    ref = matvec_oracle(H, X, "fp64")  # H in binary64: both working precisions approximate it
    e_or = rel(B, ref)
    assert e_or <= tol_oracle, (e_or, tol_oracle)
    KX = (problems.kernel_times(src, X) if kx is None else kx(X)).reshape(B.shape)
    normk = np.sqrt(src.frob2_all()) if normk is None else normk
    beta = float(np.linalg.norm(B - KX) / (normk * np.linalg.norm(X)))
    bound = matvec_bound(H.depth, H.eps)
    if name:
        _record(name, H, dict(kernel_path=path, s=X.shape[1], rel_err_vs_oracle=e_or, tol_oracle=tol_oracle,
                              backward_error=beta, bound_thm35=bound, judged_tol=10 * bound))
    assert beta <= 10 * bound, beta
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


def test_cfg2_full(cuda):
    """BASELINE config 2: n=65536, depth 8, 1/(1+|i-j|), eps 1e-6, fp64 working, one x."""
    from paper_2407_21637_b200 import problems

    H, x, src = problems.cfg2()
    assert H.working_format.name == "fp64"
    check(H, x, src, 1e-12, "cfg2", kx=problems.toeplitz_times)


def test_cfg4_full(cuda):
    """BASELINE config 4 (the largest): n=2^20, depth 12, Gaussian sigma 0.01, eps 1e-6, fp64, 16 rhs."""
    from paper_2407_21637_b200 import problems

    H, X, src = problems.cfg4()
    assert H.working_format.name == "fp64" and X.shape == (1 << 20, 16)
    check(H, X, src, 1e-12, "cfg4")


def test_cfg3_full(cuda):
    """BASELINE config 3: n=2^18, depth 10, 2-D exponential kernel, eps 1e-4, fp32, 64 rhs."""
    from paper_2407_21637_b200 import problems

    H, X, src = problems.cfg3()
    assert H.working_format.name == "fp32" and X.shape == (1 << 18, 64)
    check(H, X, src, 1e-5, "cfg3")


@pytest.fixture(scope="module")
def cfg5_svd_cache():
    return {}


@pytest.mark.parametrize("eps", [1e-2, 1e-4, 1e-6, 1e-8, 1e-10])
def test_cfg5_full(cuda, cfg5_svd_cache, eps):
    """BASELINE config 5 precision sweep at n=2^18: fp32 working for eps >= 1e-4, else fp64."""
    from paper_2407_21637_b200 import problems

    H, x, src = problems.cfg5(eps, svd_cache=cfg5_svd_cache)
    assert H.working_format.name == ("fp32" if eps >= 1e-4 else "fp64")
    check(H, x, src, 1e-5 if eps >= 1e-4 else 1e-12, f"cfg5_eps{eps:g}", kx=problems.toeplitz_times)
