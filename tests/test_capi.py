"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and its host-compiled K0 quantiser is bit-exact against the
reference's round_matrix golden vectors (same source as the device K0)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "hodlr_b200.h")
CODES = {"q52": 0, "bf16": 1, "fp16": 2, "fp32": 3, "fp64": 4}
NP_T = {0: np.uint8, 1: np.uint16, 2: np.uint16, 3: np.float32, 4: np.float64}


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\**\s+\**(hodlr_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2407_21637_b200 import _lib

    return _lib.lib()


def test_header_declares_entry_points():
    fns = header_functions()
    assert "hodlr_create" in fns and "hodlr_matvec" in fns and "hodlr_quantize" in fns
    assert len(fns) >= 18


def test_library_exports_every_declared_symbol(L):
    from paper_2407_21637_b200 import _lib

    for name in header_functions():
        assert hasattr(L, name), name
        assert name in _lib.EXPORTS, f"{name} not bound in _lib.EXPORTS"
    assert L.hodlr_abi_version() == _lib.ABI_VERSION == 3


def host_quantize(L, fmt, x):
    x = np.ascontiguousarray(x, np.float64)
    q = np.empty(x.size, NP_T[fmt])
    assert L.hodlr_quantize_host(fmt, x.ctypes.data, q.ctypes.data, x.size) == 0
    y = np.empty(x.size)
    assert L.hodlr_dequantize_host(fmt, q.ctypes.data, y.ctypes.data, x.size) == 0
    return q, y


@pytest.mark.parametrize("name", ["q52", "bf16", "fp16", "fp32"])
def test_host_k0_bit_exact_vs_reference(L, name):
    with np.load(os.path.join(GOLDEN, "round_golden.npz")) as z:
        x, want = z[f"x_{name}"], z[f"y_{name}"]
    _, y = host_quantize(L, CODES[name], x)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(y), nan)
    assert np.array_equal(y[~nan].view(np.uint64), want[~nan].view(np.uint64))


def test_host_k0_encodings_match_ieee(L):
    rng = np.random.default_rng(1)
    x = rng.standard_normal(10000) * 100
    q, _ = host_quantize(L, CODES["fp16"], x)
    assert np.array_equal(q, x.astype(np.float16).view(np.uint16))
    q, _ = host_quantize(L, CODES["fp32"], x)
    assert np.array_equal(q, x.astype(np.float32))
    # e5m2 is the high byte of the binary16 encoding of the same value
    q8, y8 = host_quantize(L, CODES["q52"], x)
    h = (q8.astype(np.uint16) << 8).view(np.float16).astype(np.float64)
    assert np.array_equal(h, y8)


def test_unsupported_format_maps_to_notimplemented(L):
    from paper_2407_21637_b200 import _lib

    x = np.zeros(4)
    st = L.hodlr_quantize_host(9, x.ctypes.data, x.ctypes.data, 4)
    assert st == _lib.HODLR_ERR_UNSUPPORTED
    with pytest.raises(NotImplementedError):
        _lib.check(st)
    assert b"format" in L.hodlr_last_error()


def test_create_rejects_bad_descriptor_without_gpu(L):
    """Validation happens before any CUDA call."""
    from paper_2407_21637_b200 import _lib

    bounds = np.array([0, 3, 8], dtype=np.int64)  # depth 1, n = 8
    D = np.eye(8)
    lptr = (_lib.c_dp * 2)(D.ctypes.data_as(_lib.c_dp), D.ctypes.data_as(_lib.c_dp))
    lds = np.array([8, 8], dtype=np.int64)
    U = np.zeros((4, 1))
    f = _lib.FactorIn(4, 1, 4, 4, U.ctypes.data_as(_lib.c_dp), 1, 1, U.ctypes.data_as(_lib.c_dp), 1, 1)
    fs = (_lib.FactorIn * 2)(f, f)
    d = _lib.Desc(8, 1, 4, bounds.ctypes.data_as(ctypes.POINTER(_lib.c_i64)), lptr,
                  lds.ctypes.data_as(ctypes.POINTER(_lib.c_i64)), fs, 0)
    h = _lib.c_vp()
    st = L.hodlr_create(ctypes.byref(d), 0, ctypes.byref(h))
    assert st == _lib.HODLR_ERR_INVALID  # factor rows 4 != leaf sizes 3 / 5
    with pytest.raises(ValueError):
        _lib.check(st)


def test_working_format_gate():
    from paper_2407_21637_b200 import linops
    from paper_2407_21637_b200.formats import parse_format
    from conftest import load_case

    H, _, _ = load_case("g512_fp64")
    custom = parse_format("custom:t=5,emin=-6,emax=7,bits=8")  # no GPU type: rejected before packing
    with pytest.raises(NotImplementedError):
        linops.matvec(H, np.zeros(H.n), custom)
