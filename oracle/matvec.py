"""Oracle restatement of Algorithm 3, HODLR_MATVEC (TEST INFRASTRUCTURE).

Follows, in order:
  * PAPER.md:512-534 (Alg. 3): b <- 0; for k = 1..l, for each sibling pair i:
    b_{2i-1} += U_{2i-1} (V_{2i}^T x_{2i}); b_{2i} += U_{2i} (V_{2i-1}^T x_{2i-1});
    then for every leaf b_i += H_ii x_i.  Each line "computed in precision u".
  * SPEC.md:334-342 (linops.matvec): two-stage evaluation (V^T x before U .),
    factors upcast to binary64, every operation rounded to ``working``;
    length mismatch -> ValueError; overflow propagates as inf.
  * level-major, sibling-pair accumulation order.
  * hodlr.py:111-135 traversal (``offdiag_blocks`` then ``leaves``).
  * arithmetic.py:14-67 rounding model (exact BLAS for fp64 working; otherwise
    per-operation rounding with left-to-right contraction, here in C:
    oracle/c/seq_arith.c).

Deviation shared with the GPU path and documented in DESIGN.md: ``x`` is
rounded to the working format on entry (so the simulated arithmetic is
realisable on hardware); for fp64 working this is the identity.

``H`` is duck-typed: any object with ``n``, ``offdiag_blocks()`` and
``leaves()`` like the reference ``HodlrMatrix`` (hodlr.py:95-135) works,
including the product package's mirror.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .fpsim import as_oracle_format, round_matrix

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle_seq.so")
        src = os.path.join(_HERE, "c", "seq_arith.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle_seq.so"])
        lib = ctypes.CDLL(path)
        i, i64, dp = ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        lib.oracle_round.argtypes = [i, i, i, i, dp, dp, i64]
        lib.oracle_seq_matmul.argtypes = [i, i, i, i, i64, i64, i64, dp, i64, dp, i64, dp, i64]
        lib.oracle_seq_add.argtypes = [i, i, i, i, dp, dp, i64]
        _LIB = lib
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _fargs(f):
    return (f.t, f.e_min, f.e_max, int(f.subnormals))


def c_round(x, fmt) -> np.ndarray:
    """Elementwise rounding through the C restatement (for self-tests)."""
    f = as_oracle_format(fmt)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    _lib().oracle_round(*_fargs(f), _ptr(x), _ptr(y), x.size)
    return y


def seq_matmul(A, B, fmt) -> np.ndarray:
    """Arithmetic(fmt, 'full-arithmetic').matmul restated (arithmetic.py:51-67)."""
    f = as_oracle_format(fmt)
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
        raise ValueError(f"matmul shape mismatch: {A.shape} x {B.shape}")
    m, q = A.shape
    s = B.shape[1]
    out = np.empty((m, s))
    if m and s:
        _lib().oracle_seq_matmul(*_fargs(f), m, q, s, _ptr(A), max(q, 1), _ptr(B), max(s, 1),
                                 _ptr(out), s)
    return out


def seq_add(b, y, fmt) -> None:
    """In place b <- rnd(b + y) (arithmetic.py:39-40); b must be C-contiguous."""
    f = as_oracle_format(fmt)
    y = np.ascontiguousarray(y, dtype=np.float64)
    assert b.flags.c_contiguous and b.dtype == np.float64 and b.shape == y.shape
    if b.size:
        _lib().oracle_seq_add(*_fargs(f), _ptr(b), _ptr(y), b.size)


def _prep_x(H, x, f):
    x = np.asarray(x, dtype=np.float64)
    vec = x.ndim == 1
    X = x.reshape(-1, 1) if vec else x
    if X.ndim != 2 or X.shape[0] != H.n:
        raise ValueError(f"length mismatch: x has {x.shape[0] if x.ndim else 0} rows, H is {H.n}")
    return vec, round_matrix(X, f)


def matvec_oracle(H, x, working=None) -> np.ndarray:
    """Alg. 3 on the CPU.  fp64 working -> numpy BLAS (as Arithmetic(FP64)
    does, arithmetic.py:59-60); any other working format -> C strict-sequential
    per-op rounding (bit-identical to Arithmetic(working).matmul/add)."""
    f = as_oracle_format(working if working is not None else H.working_format)
    vec, X = _prep_x(H, x, f)
    B = np.zeros_like(X)
    if f.identity:
        for _, _, (a, b), (c, d), upper, lower in H.offdiag_blocks():
            B[a:b] += upper.U @ (upper.V.T @ X[c:d])
            B[c:d] += lower.U @ (lower.V.T @ X[a:b])
        for _, (a, b), D in H.leaves():
            B[a:b] += D @ X[a:b]
    else:
        for _, _, (a, b), (c, d), upper, lower in H.offdiag_blocks():
            y = seq_matmul(upper.U, seq_matmul(upper.V.T, X[c:d], f), f)
            seq_add(B[a:b], y, f)
            y = seq_matmul(lower.U, seq_matmul(lower.V.T, X[a:b], f), f)
            seq_add(B[c:d], y, f)
        for _, (a, b), D in H.leaves():
            seq_add(B[a:b], seq_matmul(D, X[a:b], f), f)
    return B[:, 0] if vec else B


def matvec_arith_py(H, x, working=None) -> np.ndarray:
    """Pure-Python restatement with numpy per-op rounding (small cases only);
    cross-checks the C loop."""
    f = as_oracle_format(working if working is not None else H.working_format)
    vec, X = _prep_x(H, x, f)

    def mm(A, Bm):
        q = A.shape[1]
        if q == 0:
            return np.zeros((A.shape[0], Bm.shape[1]))
        acc = round_matrix(A[:, 0:1] * Bm[0:1, :], f)
        for j in range(1, q):
            acc = round_matrix(acc + round_matrix(A[:, j:j + 1] * Bm[j:j + 1, :], f), f)
        return acc

    B = np.zeros_like(X)
    for _, _, (a, b), (c, d), upper, lower in H.offdiag_blocks():
        B[a:b] = round_matrix(B[a:b] + mm(upper.U, mm(upper.V.T, X[c:d])), f)
        B[c:d] = round_matrix(B[c:d] + mm(lower.U, mm(lower.V.T, X[a:b])), f)
    for _, (a, b), D in H.leaves():
        B[a:b] = round_matrix(B[a:b] + mm(D, X[a:b]), f)
    return B[:, 0] if vec else B


def dense_of(H) -> np.ndarray:
    """Dense binary64 assembly (restates reconstruct_dense, hodlr.py:268-276)."""
    out = np.zeros((H.n, H.n))
    for _, (a, b), D in H.leaves():
        out[a:b, a:b] = D
    for _, _, (a, b), (c, d), upper, lower in H.offdiag_blocks():
        out[a:b, c:d] = upper.U @ upper.V.T
        out[c:d, a:b] = lower.U @ lower.V.T
    return out
