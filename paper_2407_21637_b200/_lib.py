"""ctypes binding of the C ABI in include/hodlr_b200.h (libhodlr_b200.so, built in-tree).

There is no fallback: if the shared library is missing the import of the
operator layer raises, naming the build command.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HODLR_B200_LIB: load an instrumented build instead (diagnostics in tools/ only)
LIB_PATH = os.environ.get("HODLR_B200_LIB") or os.path.join(_HERE, "libhodlr_b200.so")

c_i32, c_i64, c_sz, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)

HODLR_OK, HODLR_ERR_INVALID, HODLR_ERR_UNSUPPORTED, HODLR_ERR_CUDA = 0, 1, 2, 3
PATH_GENERIC, PATH_FUSED_SV, PATH_MRHS, PATH_MRHS_SLAB, PATH_MRHS_TC, PATH_STRICT = 0, 1, 2, 3, 4, 5
PATH_NAMES = {PATH_GENERIC: "generic", PATH_FUSED_SV: "fused_sv", PATH_MRHS: "mrhs", PATH_MRHS_SLAB: "mrhs_slab",
              PATH_MRHS_TC: "mrhs_tc", PATH_STRICT: "strict"}
ABI_VERSION = 3


class FactorIn(ctypes.Structure):
    _fields_ = [("fmt", c_i32), ("rank", c_i32), ("rows", c_i64), ("cols", c_i64),
                ("U", c_dp), ("u_rs", c_i64), ("u_cs", c_i64),
                ("V", c_dp), ("v_rs", c_i64), ("v_cs", c_i64)]


class Desc(ctypes.Structure):
    _fields_ = [("n", c_i64), ("depth", c_i32), ("leaf_fmt", c_i32),
                ("leaf_bounds", ctypes.POINTER(c_i64)), ("leaves", ctypes.POINTER(c_dp)),
                ("leaf_ld", ctypes.POINTER(c_i64)), ("factors", ctypes.POINTER(FactorIn)),
                ("payload_encoded", c_i32)]


class Shard(ctypes.Structure):
    _fields_ = [("rank", c_i32), ("nranks", c_i32)]


class Info(ctypes.Structure):
    _fields_ = [("n_local", c_i64), ("row0", c_i64), ("matrix_bytes", c_i64),
                ("device_bytes", c_i64), ("depth", c_i32), ("leaf_fmt", c_i32),
                ("launches_per_matvec", c_i32), ("num_levels_external", c_i32)]


EXPORTS = {
    "hodlr_abi_version": (c_i32, []),
    "hodlr_last_error": (ctypes.c_char_p, []),
    "hodlr_create": (c_i32, [ctypes.POINTER(Desc), c_i32, ctypes.POINTER(c_vp)]),
    "hodlr_create_sharded": (c_i32, [ctypes.POINTER(Desc), c_i32, Shard, ctypes.POINTER(c_vp)]),
    "hodlr_destroy": (c_i32, [c_vp]),
    "hodlr_workspace_size": (c_i32, [c_vp, c_i64, ctypes.POINTER(c_sz)]),
    "hodlr_matvec": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_sz, c_vp]),
    "hodlr_matvec_strict": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_sz, c_vp]),
    "hodlr_workspace_size_for": (c_i32, [c_vp, c_i32, c_i32, c_i64, ctypes.POINTER(c_sz)]),
    "hodlr_matvec_host": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i64, c_vp]),
    "hodlr_shard_exchange_count": (c_i32, [c_vp, c_i64, ctypes.POINTER(c_i64)]),
    "hodlr_matvec_shard_begin": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "hodlr_matvec_shard_local": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_sz,
                                         c_vp]),
    "hodlr_matvec_shard_end": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp,
                                       c_sz, c_vp]),
    "hodlr_quantize": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_vp]),
    "hodlr_dequantize": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_vp]),
    "hodlr_quantize_host": (c_i32, [c_i32, c_vp, c_vp, c_i64]),
    "hodlr_dequantize_host": (c_i32, [c_i32, c_vp, c_vp, c_i64]),
    "hodlr_unpack_factor": (c_i32, [c_vp, c_i64, c_vp, c_vp]),
    "hodlr_unpack_leaf": (c_i32, [c_vp, c_i64, c_vp]),
    "hodlr_info": (c_i32, [c_vp, ctypes.POINTER(Info)]),
    "hodlr_matvec_path": (c_i32, [c_vp, c_i32, c_i64, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]),
}

_LIB = None


def lib():
    """Load (once) and return the CDLL.  Raises if the extension was not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or make -C "
                "paper_2407_21637_b200/csrc).  There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.hodlr_abi_version() != ABI_VERSION:
            raise ImportError("libhodlr_b200.so ABI version mismatch; rebuild the extension")
        _LIB = L
    return _LIB


def check(status: int, what: str = "") -> None:
    """Map a hodlr_status onto the reference's exception convention."""
    if status == HODLR_OK:
        return
    msg = lib().hodlr_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == HODLR_ERR_INVALID:
        raise ValueError(text)
    if status == HODLR_ERR_UNSUPPORTED:
        raise NotImplementedError(text)
    raise RuntimeError(text)
