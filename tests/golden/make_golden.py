"""Generate the committed golden fixtures FROM THE REFERENCE PACKAGE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``hodlrmp`` from /root/reference/pkg/src (read-only) and records:

* ``round_golden.npz``: adversarial binary64 inputs (random exponents, exact
  midpoints, +-1 ulp around midpoints, subnormal midpoints, overflow edges,
  signed zeros, infs, nan) and the reference ``round_matrix`` output for each
  named format (fpsim.py:180-185), plus the SPEC KATs.
* ``hodlr_<case>.npz``: matrices built by the reference ``build_adaptive``
  (hodlr.py:227-265) and written by the reference ``save_hodlr`` (container v1,
  hodlr.py:297-324).
* ``vec_<case>.npz``: x (or X), ``reconstruct_dense(H) @ x`` (hodlr.py:268-276),
  and Algorithm 3 evaluated with the reference's own
  ``offdiag_blocks``/``leaves`` traversal and ``Arithmetic`` class
  (arithmetic.py:14-67) in the working format, plus the precision plan,
  per-block ranks and ``storage_bits`` (hodlr.py:279-287).
* ``cfg1_summary.npz``: BASELINE config 1 (n=4096, depth 4, eps=1e-8) built by
  the reference: plan, ranks, storage bits, x, dense product and Alg. 3 output
  (factor payloads omitted; the 10 MB matrix is rebuilt by the harness builder
  and compared against this summary).

The GPU box never sees /root/reference: tests only read these files.
"""

from __future__ import annotations

import json
import math
import os
import sys
import zlib

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from hodlrmp import fpsim, hodlr, tree  # noqa: E402
from hodlrmp.arithmetic import Arithmetic  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ALL = (fpsim.Q52, fpsim.BF16, fpsim.FP16, fpsim.FP32, fpsim.FP64)


# ---------------------------------------------------------------- rounding
def adversarial(fmt, rng, count):
    t, emin, emax = fmt.t, fmt.e_min, fmt.e_max
    parts = []
    # random magnitudes over (and beyond) the exponent range
    e = rng.integers(emin - t - 3, emax + 3, size=count)
    parts.append(np.ldexp(rng.random(count) + 0.5, e) * rng.choice([-1.0, 1.0], count))
    # exact midpoints between adjacent representable values (normal + subnormal)
    e = rng.integers(emin - t + 1, emax + 1, size=count)
    qexp = np.maximum(e - t, emin - t + 1)
    base = np.ldexp(np.floor(np.ldexp(np.ldexp(0.5 + rng.random(count) / 2, e), -qexp)), qexp)
    mid = base + np.ldexp(0.5, qexp)
    parts.append(mid)
    parts.append(np.nextafter(mid, np.inf))
    parts.append(np.nextafter(mid, -np.inf))
    parts.append(-mid)
    # overflow edges
    xm = fmt.x_max
    half = math.ldexp(1.0, fmt.e_max - fmt.t)  # half ulp at the top binade
    edges = np.array([xm, xm + half, np.nextafter(xm + half, 0), np.nextafter(xm + half, np.inf),
                      2 * xm, 1e300, fmt.smallest_subnormal, fmt.smallest_subnormal / 2,
                      np.nextafter(fmt.smallest_subnormal / 2, 1), np.nextafter(fmt.smallest_subnormal / 2, 0),
                      fmt.x_min, 5e-324, 0.0, -0.0, np.inf, -np.inf, 1.0, 1.0 + 2.0 ** -9])
    parts.append(np.concatenate([edges, -edges]))
    return np.concatenate(parts)


def make_round_golden():
    rng = np.random.default_rng(20240731)
    out = {}
    for fmt in ALL[:-1]:
        x = adversarial(fmt, rng, 6000)
        x = np.concatenate([x, [np.nan]])
        out[f"x_{fmt.name}"] = x
        out[f"y_{fmt.name}"] = fpsim.round_matrix(x, fmt)
    kat = {
        "7e4_fp16": fpsim.round_scalar(7.0e4, fpsim.FP16),
        "1p2m9_bf16": fpsim.round_scalar(1 + 2.0 ** -9, fpsim.BF16),
        "u_fp16": fpsim.unit_roundoff(fpsim.FP16),
        "u_fp64": fpsim.unit_roundoff(fpsim.FP64),
        "u_q52": fpsim.unit_roundoff(fpsim.Q52),
    }
    out["kat"] = json.dumps(kat)
    np.savez_compressed(os.path.join(OUT, "round_golden.npz"), **out)


# ---------------------------------------------------------------- matrices
def gaussian_1d(n, sigma, nugget, seed):
    t = np.sort(np.random.default_rng(seed).random(n))
    A = np.exp(-((t[:, None] - t[None, :]) ** 2) / (2 * sigma * sigma))
    return A + nugget * np.eye(n)


def exp_1d(n, ell, seed):
    t = np.sort(np.random.default_rng(seed).random(n))
    return np.exp(-np.abs(t[:, None] - t[None, :]) / ell)


def toeplitz_inv(n):
    i = np.arange(n)
    return 1.0 / (1.0 + np.abs(i[:, None] - i[None, :]))


def alg3_reference(H, X, working):
    """Alg. 3 through the reference's own primitives (arithmetic.py, hodlr.py)."""
    ar = Arithmetic(working, "full-arithmetic")
    X = fpsim.round_matrix(X, working)
    B = np.zeros_like(X)
    for _, _, (a, b), (c, d), up, lo in H.offdiag_blocks():
        B[a:b] = ar.add(B[a:b], ar.matmul(up.U, ar.matmul(up.V.T, X[c:d])))
        B[c:d] = ar.add(B[c:d], ar.matmul(lo.U, ar.matmul(lo.V.T, X[a:b])))
    for _, (a, b), D in H.leaves():
        B[a:b] = ar.add(B[a:b], ar.matmul(D, X[a:b]))
    return B


def summary(H):
    ranks = [[up.rank, lo.rank] for _, _, _, _, up, lo in H.offdiag_blocks()]
    return {
        "formats": [f.name for f in H.plan.chosen],
        "xi": H.plan.xi,
        "thresholds": H.plan.thresholds,
        "fallback": H.plan.fallback,
        "ranks": ranks,
        "storage_bits": int(hodlr.storage_bits(H)),
        "working": H.working_format.name,
        "n": H.n,
        "depth": H.depth,
        "eps": H.eps,
    }


CASES = {
    # name: (A builder, n, depth, eps, working, s)
    "g512_fp64": (lambda: gaussian_1d(512, 0.05, 1e-2, 0), 512, 2, 1e-8, fpsim.FP64, 1),
    "g2000_fp32": (lambda: gaussian_1d(2000, 0.02, 0.0, 3), 2000, 8, 1e-4, fpsim.FP32, 1),
    "g512_e9_fp32": (lambda: gaussian_1d(512, 0.05, 1e-2, 0), 512, 2, 1e-9, fpsim.FP32, 2),
    "toep512_e3_fp64": (lambda: toeplitz_inv(512), 512, 2, 3e-3, fpsim.FP64, 1),
    "toep1024_e2_fp32": (lambda: toeplitz_inv(1024), 1024, 3, 1e-2, fpsim.FP32, 1),
    "toep1024_e4_fp64": (lambda: toeplitz_inv(1024), 1024, 3, 1e-4, fpsim.FP64, 2),
    "blockdiag64_fp64": (lambda: np.diag(np.arange(1.0, 65.0)), 64, 2, 1e-8, fpsim.FP64, 1),
    "depth0_fp32": (lambda: np.random.default_rng(5).standard_normal((16, 16)), 16, 0, 1e-3, fpsim.FP32, 1),
    "rand96_fp32": (lambda: np.random.default_rng(6).standard_normal((96, 96)), 96, 3, 1e-1, fpsim.FP32, 3),
}


def make_case(name, build, n, depth, eps, working, s):
    A = build()
    T = tree.build_tree(n, depth)
    H = hodlr.build_adaptive(A, T, eps, working=working, available=ALL)
    hodlr.save_hodlr(H, os.path.join(OUT, f"hodlr_{name}.npz"))
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    X = rng.standard_normal((n, s))
    Xw = fpsim.round_matrix(X, working)
    dense = hodlr.reconstruct_dense(H)
    b_dense = dense @ Xw
    b_alg3 = alg3_reference(H, X, working)
    b_alg3_fp64 = alg3_reference(H, Xw, fpsim.FP64) if working.name != "fp64" else b_alg3
    KX = A @ Xw
    np.savez_compressed(
        os.path.join(OUT, f"vec_{name}.npz"),
        x=X, b_dense=b_dense, b_alg3=b_alg3, b_alg3_fp64=b_alg3_fp64, KX=KX,
        normA=np.linalg.norm(A), summary=json.dumps(summary(H)),
    )
    print(name, summary(H)["formats"], [r[0] for r in summary(H)["ranks"]][:8], hodlr.storage_bits(H))


def make_cfg1():
    A = gaussian_1d(4096, 0.05, 1e-2, 0)
    T = tree.build_tree(4096, 4)
    H = hodlr.build_adaptive(A, T, 1e-8, working=fpsim.FP64, available=ALL)
    x = np.random.default_rng(1).standard_normal(4096)
    b_dense = hodlr.reconstruct_dense(H) @ x
    b_alg3 = alg3_reference(H, x.reshape(-1, 1), fpsim.FP64)[:, 0]
    np.savez_compressed(
        os.path.join(OUT, "cfg1_summary.npz"),
        x=x, b_dense=b_dense, b_alg3=b_alg3, KX=A @ x, normA=np.linalg.norm(A),
        summary=json.dumps(summary(H)),
    )
    print("cfg1", summary(H)["formats"], summary(H)["storage_bits"])


if __name__ == "__main__":
    make_round_golden()
    for name, args in CASES.items():
        make_case(name, *args)
    make_cfg1()
