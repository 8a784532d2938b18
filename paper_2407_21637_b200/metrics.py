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

__all__ = ["matvec_bound", "matvec_backward_error", "hypothesis_holds"]


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
