"""HODLR object model used by the B200 matvec (input side of the hot path).

The drop-in accepts the reference's own ``HodlrMatrix`` (hodlr.py:95-135) and
this module's equivalent, which keeps the same public surface the matvec
needs -- ``n``, ``depth``, ``tree.ranges``, ``working_format``, ``plan``,
``eps``, ``offdiag_blocks()`` (hodlr.py:111-123: level-major, pair order,
yielding ``(k, i, rows_first, rows_second, upper, lower)``) and ``leaves()``
(hodlr.py:125-135) -- but stores the blocks flat, level by level, instead of
as a recursive node tree.  ``load_hodlr``/``save_hodlr`` read and write the
reference's ``.npz`` container v1 (hodlr.py:297-363), so matrices move between
the two packages bit-exactly.

Container v2 (``save_hodlr(..., narrow=True)``) is the narrow-payload variant
of the same schema: identical keys and metadata, ``container_version`` 2, and
every payload stored in its own format's encoding instead of binary64 (q52: one
byte, bf16 / fp16: two, fp32: four) -- 8x fewer bytes for a q52 level.
``load_hodlr`` decodes it back to the binary64 object model (exact);
``load_encoded`` keeps the narrow arrays so the device loader
(``HodlrOperator.from_container``) hands them to the C ABI as they are.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .formats import FP64, PrecisionFormat, format_spec, parse_format

__all__ = [
    "ClusterTree", "build_tree", "LowRankFactor", "PrecisionPlan", "HodlrMatrix",
    "storage_bits", "load_hodlr", "save_hodlr", "load_encoded", "EncodedHodlr",
    "CONTAINER_VERSION", "NARROW_CONTAINER_VERSION",
]

CONTAINER_VERSION = 1
NARROW_CONTAINER_VERSION = 2
# numpy carrier of each named format's encoding (bf16 / q52 have no numpy type:
# their bit patterns travel as unsigned integers)
ENCODED_DTYPE = {"q52": np.uint8, "bf16": np.uint16, "fp16": np.float16, "fp32": np.float32, "fp64": np.float64}


@dataclass(frozen=True)
class ClusterTree:
    """Balanced binary partition of range(n); ``ranges[k][i]`` is the half-open
    interval of node i at level k (tree.py:18-32)."""

    n: int
    depth: int
    ranges: tuple

    @property
    def leaf_ranges(self):
        return list(self.ranges[self.depth])


def build_tree(n: int, depth: int) -> ClusterTree:
    """Ceil split: the left child gets ceil(m/2) of a size-m parent (tree.py:35-54)."""
    if n < 1:
        raise ValueError(f"dimension {n} must be positive")
    if depth < 0:
        raise ValueError(f"depth {depth} must be nonnegative")
    if 2 ** depth > n:
        raise ValueError(f"tree too deep for dimension: 2**{depth} > {n}")
    levels = [((0, n),)]
    for _ in range(depth):
        nxt = []
        for a, b in levels[-1]:
            mid = a + (b - a + 1) // 2
            nxt += [(a, mid), (mid, b)]
        levels.append(tuple(nxt))
    return ClusterTree(n, depth, tuple(levels))


@dataclass(frozen=True, eq=False)
class LowRankFactor:
    """Block = U @ V.T, U rows x r, V cols x r, entries representable in fmt
    (lowrank.py:30-67)."""

    U: np.ndarray
    V: np.ndarray
    fmt: PrecisionFormat = field(default=FP64)

    def __post_init__(self):
        if self.U.ndim != 2 or self.V.ndim != 2 or self.U.shape[1] != self.V.shape[1]:
            raise ValueError(f"bad factor shapes U {self.U.shape}, V {self.V.shape}")

    rows = property(lambda self: self.U.shape[0])
    cols = property(lambda self: self.V.shape[0])
    rank = property(lambda self: self.U.shape[1])

    def dense(self) -> np.ndarray:
        return self.U @ self.V.T


@dataclass
class PrecisionPlan:
    """Per-level storage formats (index 0 = level 1), hodlr.py:72-92."""

    chosen: list
    xi: list | None = None
    thresholds: list | None = None
    fallback: list | None = None

    def level_format(self, k: int):
        return self.chosen[k - 1]

    @property
    def any_fallback(self) -> bool:
        return bool(self.fallback) and any(self.fallback)


@dataclass(eq=False)
class HodlrMatrix:
    """Flat HODLR container: ``blocks[k-1][i] = (upper, lower)`` for pair i of
    level k; ``leaf_blocks[i]`` the dense diagonal leaf i (working format)."""

    tree: ClusterTree
    leaf_blocks: list
    blocks: list
    eps: float
    plan: PrecisionPlan
    working_format: PrecisionFormat

    def __post_init__(self):
        if len(self.leaf_blocks) != 2 ** self.tree.depth or len(self.blocks) != self.tree.depth:
            raise ValueError("block lists do not match the cluster tree")

    n = property(lambda self: self.tree.n)
    depth = property(lambda self: self.tree.depth)

    def offdiag_blocks(self):
        for k in range(1, self.depth + 1):
            lvl = self.tree.ranges[k]
            for i, (upper, lower) in enumerate(self.blocks[k - 1]):
                yield k, i, lvl[2 * i], lvl[2 * i + 1], upper, lower

    def leaves(self):
        for i, block in enumerate(self.leaf_blocks):
            yield i, self.tree.ranges[self.depth][i], block


def storage_bits(H) -> int:
    """Bits of all leaves (working format) and factors (their formats),
    hodlr.py:279-287.  Works on either object model."""
    total = sum((b - a) ** 2 * H.working_format.bits for _, (a, b), _ in H.leaves())
    for _, _, _, _, up, lo in H.offdiag_blocks():
        total += sum((f.rows + f.cols) * f.rank * f.fmt.bits for f in (up, lo))
    return total


def _encode(a: np.ndarray, fmt) -> np.ndarray:
    """binary64 values representable in fmt -> the format's encoding, same
    shape and memory order (K0's host build: exact for representable values)."""
    from . import _lib
    from .formats import format_code

    code = format_code(fmt)
    a = np.asarray(a, dtype=np.float64)
    order = "F" if (a.ndim == 2 and a.flags.f_contiguous and not a.flags.c_contiguous) else "C"
    flat = np.ascontiguousarray(a.ravel(order=order))
    out = np.empty(flat.size, dtype=ENCODED_DTYPE[fmt.name])
    if flat.size:
        _lib.check(_lib.lib().hodlr_quantize_host(code, flat.ctypes.data, out.ctypes.data, flat.size))
    return out.reshape(a.shape, order=order)


def _decode(a: np.ndarray, fmt) -> np.ndarray:
    """Inverse of _encode: exact widening to binary64, memory order kept."""
    from . import _lib
    from .formats import format_code

    code = format_code(fmt)
    want = np.dtype(ENCODED_DTYPE[fmt.name])
    if a.dtype != want:
        raise ValueError(f"payload dtype {a.dtype} is not the {fmt.name} encoding ({want})")
    order = "F" if (a.ndim == 2 and a.flags.f_contiguous and not a.flags.c_contiguous) else "C"
    flat = np.ascontiguousarray(a.ravel(order=order))
    out = np.empty(flat.size, dtype=np.float64)
    if flat.size:
        _lib.check(_lib.lib().hodlr_dequantize_host(code, flat.ctypes.data, out.ctypes.data, flat.size))
    return out.reshape(a.shape, order=order)


def save_hodlr(H, path, narrow: bool = False) -> None:
    """Container writer: v1 (the schema of hodlr.py:297-324, binary64 payloads)
    or, with ``narrow=True``, v2 (same keys, payloads in their formats' encodings)."""
    meta = {
        "container_version": NARROW_CONTAINER_VERSION if narrow else CONTAINER_VERSION,
        "n": H.n, "depth": H.depth, "eps": H.eps,
        "working": format_spec(H.working_format),
        "level_formats": [format_spec(f) for f in H.plan.chosen],
        "xi": H.plan.xi, "thresholds": H.plan.thresholds, "fallback": H.plan.fallback,
    }
    enc = (lambda a, f: _encode(a, f)) if narrow else (lambda a, f: a)
    arrays = {f"leaf{i}": enc(blk, H.working_format) for i, _, blk in H.leaves()}
    for k, i, _, _, up, lo in H.offdiag_blocks():
        for tag, f in (("upper", up), ("lower", lo)):
            arrays[f"lvl{k}_pair{i}_{tag}_U"] = enc(f.U, f.fmt)
            arrays[f"lvl{k}_pair{i}_{tag}_V"] = enc(f.V, f.fmt)
    np.savez(path, __meta__=json.dumps(meta), **arrays)


@dataclass(eq=False)
class EncodedHodlr:
    """A stored matrix with its payloads still in their narrow encodings
    (container v2) or binary64 (v1): what the device loader consumes."""

    tree: ClusterTree
    leaf_blocks: list            # encoded arrays, working format
    blocks: list                 # blocks[k-1][i] = ((U, V), (U, V)) encoded arrays, level format
    eps: float
    plan: PrecisionPlan
    working_format: PrecisionFormat
    encoded: bool

    n = property(lambda self: self.tree.n)
    depth = property(lambda self: self.tree.depth)

    def payload_bytes(self) -> int:
        return sum(a.nbytes for a in self.leaf_blocks) + sum(
            a.nbytes for lvl in self.blocks for pair in lvl for fac in pair for a in fac)


def _read(path):
    with np.load(path, allow_pickle=False) as z:
        meta = json.loads(str(z["__meta__"][()]))
        ver = meta.get("container_version")
        if ver not in (CONTAINER_VERSION, NARROW_CONTAINER_VERSION):
            raise ValueError(f"unsupported container version {ver!r}")
        tree = build_tree(int(meta["n"]), int(meta["depth"]))
        working = parse_format(meta["working"])
        chosen = [parse_format(s) for s in meta["level_formats"]]
        if len(chosen) != tree.depth:
            raise ValueError("level_formats does not match the tree depth")
        plan = PrecisionPlan(chosen, meta.get("xi"), meta.get("thresholds"), meta.get("fallback"))
        leaves = [z[f"leaf{i}"] for i in range(2 ** tree.depth)]
        blocks = [[tuple((z[f"lvl{k}_pair{i}_{tag}_U"], z[f"lvl{k}_pair{i}_{tag}_V"]) for tag in ("upper", "lower"))
                   for i in range(2 ** (k - 1))] for k in range(1, tree.depth + 1)]
    return EncodedHodlr(tree, leaves, blocks, float(meta["eps"]), plan, working, ver == NARROW_CONTAINER_VERSION)


def load_encoded(path) -> EncodedHodlr:
    """Container v1 or v2 with the payloads as stored (no widening)."""
    return _read(path)


def load_hodlr(path) -> HodlrMatrix:
    """Container reader (v1: schema of hodlr.py:297-363; v2: narrow payloads,
    widened exactly) into the flat binary64 model."""
    E = _read(path)
    dl = (lambda a: _decode(a, E.working_format)) if E.encoded else (lambda a: a)
    leaves = [dl(a) for a in E.leaf_blocks]
    blocks = []
    for k in range(1, E.depth + 1):
        fmt = E.plan.chosen[k - 1]
        df = (lambda a, fmt=fmt: _decode(a, fmt)) if E.encoded else (lambda a: a)
        blocks.append([tuple(LowRankFactor(df(U), df(V), fmt) for U, V in pair) for pair in E.blocks[k - 1]])
    return HodlrMatrix(E.tree, leaves, blocks, E.eps, E.plan, E.working_format)
