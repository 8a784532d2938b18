"""Error measures and the Theorem 3.5 bound of the HODLR matvec.

Restates the spec'd metrics: the relative backward error
||b_hat - K x||_F / (||K||_F ||x||_F) (numerator against the binary64 K x, see
SPEC.md "linops Open Questions") and the bound
2 (sqrt2 + 1) sqrt(2^(l+1) + 2^(l-1)) eps of Thm 3.5,
valid when the working unit roundoff u <= eps / n.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["matvec_bound", "matvec_backward_error", "hypothesis_holds", "construction_bound",
           "construction_error", "storage_ratio"]


def construction_bound(depth: int, eps: float) -> float:
    """Thm 3.1's global construction bound (2 sqrt(2 l) + 1) eps."""
    if depth < 1:
        raise ValueError("depth must be >= 1")
    return (2.0 * math.sqrt(2.0 * depth) + 1.0) * eps


def construction_error(A, H_dense) -> float:
    """||A - reconstruct_dense(H)||_F / ||A||_F; H_dense is the
    densified HODLR matrix."""
    na = float(np.linalg.norm(A))
    if na == 0.0:
        raise ValueError("zero matrix")
    return float(np.linalg.norm(np.asarray(A) - np.asarray(H_dense)) / na)


def storage_ratio(uniform, adaptive) -> float:
    """storage_bits(uniform build) / storage_bits(adaptive build)."""
    from .model import storage_bits

    return storage_bits(uniform) / storage_bits(adaptive)


def matvec_bound(depth: int, eps: float) -> float:
    if eps == 0:
        return 0.0
    return 2.0 * (math.sqrt(2.0) + 1.0) * math.sqrt(2.0 ** (depth + 1) + 2.0 ** (depth - 1)) * eps


def matvec_backward_error(kx, x, b_hat, norm_k: float) -> float:
    nx = float(np.linalg.norm(x))
    if norm_k == 0 or nx == 0:
        raise ValueError("zero matrix or vector")
    return float(np.linalg.norm(np.asarray(b_hat) - np.asarray(kx)) / (norm_k * nx))


def hypothesis_holds(working, eps: float, n: int) -> bool:
    return working.unit_roundoff <= eps / n
