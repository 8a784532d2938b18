"""Storage / working formats of the adaptive-precision HODLR.

Mirrors the reference's format model (/root/reference/pkg/src/hodlrmp/fpsim.py:48-157):
a format is (t significand bits incl. the implicit one, e_min, e_max, storage
bits, subnormals flag), with the five named formats of fpsim.py:110-114
(q52 = fp8 E5M2).  ``format_code`` maps either this module's formats or the
reference's ``PrecisionFormat`` objects onto the C-ABI ``hodlr_format`` codes;
custom formats have no GPU encoding and raise ``NotImplementedError``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

__all__ = [
    "PrecisionFormat", "Q52", "BF16", "FP16", "FP32", "FP64", "NAMED_FORMATS",
    "parse_format", "format_spec", "format_code", "format_from_code", "unit_roundoff",
    "bits_per_scalar", "CODE", "ELEMENT_BYTES",
]


@dataclass(frozen=True)
class PrecisionFormat:
    name: str
    t: int
    e_min: int
    e_max: int
    bits: int
    subnormals_enabled: bool = True

    def __post_init__(self):
        if self.t < 2:
            raise ValueError(f"significand width t={self.t} must be >= 2")
        if self.e_min >= self.e_max:
            raise ValueError(f"need e_min < e_max, got {self.e_min} >= {self.e_max}")
        if self.bits < 1:
            raise ValueError(f"storage width {self.bits} must be positive")

    @property
    def unit_roundoff(self) -> float:
        return math.ldexp(1.0, -self.t)

    @property
    def x_min(self) -> float:
        return math.ldexp(1.0, self.e_min)

    @property
    def x_max(self) -> float:
        return math.ldexp(2.0 - math.ldexp(1.0, 1 - self.t), self.e_max)

    @property
    def smallest_subnormal(self) -> float:
        return math.ldexp(1.0, self.e_min - self.t + 1)

    @property
    def is_exact_for_binary64(self) -> bool:
        return self.t >= 53 and self.e_min <= -1022 and self.e_max >= 1023 and self.subnormals_enabled

    def __str__(self):
        return self.name


Q52 = PrecisionFormat("q52", 3, -14, 15, 8)
BF16 = PrecisionFormat("bf16", 8, -126, 127, 16)
FP16 = PrecisionFormat("fp16", 11, -14, 15, 16)
FP32 = PrecisionFormat("fp32", 24, -126, 127, 32)
FP64 = PrecisionFormat("fp64", 53, -1022, 1023, 64)
NAMED_FORMATS = {f.name: f for f in (Q52, BF16, FP16, FP32, FP64)}

# hodlr_format codes of include/hodlr_b200.h
CODE = {"q52": 0, "bf16": 1, "fp16": 2, "fp32": 3, "fp64": 4}
ELEMENT_BYTES = {0: 1, 1: 2, 2: 2, 3: 4, 4: 8}
_BY_CODE = {v: NAMED_FORMATS[k] for k, v in CODE.items()}


def parse_format(spec: str) -> PrecisionFormat:
    """Format name or ``custom:t=..,emin=..,emax=..,bits=..[,subnormals=0|1]``
    (fpsim.py:119-149)."""
    spec = spec.strip()
    if spec in NAMED_FORMATS:
        return NAMED_FORMATS[spec]
    if spec.startswith("custom:"):
        kv = {}
        for item in spec[7:].split(","):
            key, _, val = item.partition("=")
            if not val:
                raise ValueError(f"malformed custom format field {item!r} in {spec!r}")
            kv[key.strip()] = int(val)
        try:
            return PrecisionFormat("custom", kv["t"], kv["emin"], kv["emax"], kv["bits"],
                                   bool(kv.get("subnormals", 1)))
        except KeyError as exc:
            raise ValueError(f"custom format {spec!r} is missing field {exc}") from None
    raise ValueError(f"unknown precision format {spec!r}; expected one of {sorted(NAMED_FORMATS)} "
                     "or custom:t=..,emin=..,emax=..,bits=..")


def format_spec(fmt) -> str:
    if fmt.name in NAMED_FORMATS and _same(fmt, NAMED_FORMATS[fmt.name]):
        return fmt.name
    sub = "" if getattr(fmt, "subnormals_enabled", True) else ",subnormals=0"
    return f"custom:t={fmt.t},emin={fmt.e_min},emax={fmt.e_max},bits={fmt.bits}{sub}"


def _same(a, b) -> bool:
    return (a.t, a.e_min, a.e_max, a.bits, bool(getattr(a, "subnormals_enabled", True))) == (
        b.t, b.e_min, b.e_max, b.bits, b.subnormals_enabled)


def format_code(fmt) -> int:
    """C-ABI code of a named format (ours or the reference's PrecisionFormat)."""
    if isinstance(fmt, str):
        fmt = parse_format(fmt)
    named = NAMED_FORMATS.get(getattr(fmt, "name", None))
    if named is None or not _same(fmt, named):
        raise NotImplementedError(
            f"format {format_spec(fmt)!r} has no B200 storage encoding; only "
            f"{sorted(NAMED_FORMATS)} are supported on the GPU path")
    return CODE[named.name]


def format_from_code(code: int) -> PrecisionFormat:
    return _BY_CODE[int(code)]


def unit_roundoff(fmt) -> float:
    return math.ldexp(1.0, -fmt.t)


def bits_per_scalar(fmt) -> int:
    return int(fmt.bits)
