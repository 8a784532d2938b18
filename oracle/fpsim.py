"""Oracle restatement of the reference storage quantiser (TEST INFRASTRUCTURE).

Restates /root/reference/pkg/src/hodlrmp/fpsim.py:
  * the named format table (fpsim.py:110-114),
  * ``_round_array`` / ``round_matrix`` (fpsim.py:160-185): round-to-nearest,
    ties-to-even of binary64 values onto the grid of a format with t significand
    bits, exponent range [e_min, e_max]; magnitudes that round above x_max become
    +-inf; subnormals kept (optionally flushed); zeros/infs/nans pass through.

Used only by tests/ and bench.py's CPU baseline, never by the product package.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class OracleFormat:
    name: str
    t: int
    e_min: int
    e_max: int
    bits: int
    subnormals: bool = True

    @property
    def u(self) -> float:
        return math.ldexp(1.0, -self.t)

    @property
    def x_max(self) -> float:
        return math.ldexp(2.0 - math.ldexp(1.0, 1 - self.t), self.e_max)

    @property
    def identity(self) -> bool:
        return self.t >= 53 and self.e_min <= -1022 and self.e_max >= 1023 and self.subnormals


# fpsim.py:110-114
FORMATS = {
    "q52": OracleFormat("q52", 3, -14, 15, 8),
    "bf16": OracleFormat("bf16", 8, -126, 127, 16),
    "fp16": OracleFormat("fp16", 11, -14, 15, 16),
    "fp32": OracleFormat("fp32", 24, -126, 127, 32),
    "fp64": OracleFormat("fp64", 53, -1022, 1023, 64),
}


def as_oracle_format(fmt) -> OracleFormat:
    """Accept a name, an OracleFormat, or any object with the reference's
    PrecisionFormat fields (fpsim.py:48-68)."""
    if isinstance(fmt, OracleFormat):
        return fmt
    if isinstance(fmt, str):
        return FORMATS[fmt]
    return OracleFormat(
        str(fmt.name), int(fmt.t), int(fmt.e_min), int(fmt.e_max), int(fmt.bits),
        bool(getattr(fmt, "subnormals_enabled", True)),
    )


def unit_roundoff(fmt) -> float:
    return as_oracle_format(fmt).u


def round_matrix(a, fmt) -> np.ndarray:
    """RNE of every binary64 entry onto ``fmt``'s grid (fpsim.py:160-185).

    With |a| = f * 2**e, f in [0.5, 1), the grid spacing at |a| is 2**q with
    q = max(e - t, e_min - t + 1) (the floor is the subnormal spacing).  Scaling
    by powers of two is exact in binary64 and ``np.rint`` rounds half to even.
    """
    f = as_oracle_format(fmt)
    a = np.asarray(a, dtype=np.float64)
    if f.identity:
        return a.copy()
    with np.errstate(invalid="ignore", over="ignore"):
        mag = np.abs(a)
        e = np.frexp(mag)[1].astype(np.int64)
        q = np.maximum(e - f.t, f.e_min - f.t + 1)
        r = np.ldexp(np.rint(np.ldexp(mag, -q)), q)
        r = np.where(r > f.x_max, np.inf, r)
        if not f.subnormals:
            r = np.where(r < math.ldexp(1.0, f.e_min), 0.0, r)
        return np.copysign(r, a)
