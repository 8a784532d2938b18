"""Pin the CPU oracle against the reference's own outputs (tests/golden/, made by
tests/golden/make_golden.py from /root/reference).  CPU only."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_case
from oracle import fpsim as ofp
from oracle import matvec as omv

FMTS = ["q52", "bf16", "fp16", "fp32"]


def same_bits(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.array_equal(a.view(np.uint64), b.view(np.uint64)) or (
        np.array_equal(np.isnan(a), np.isnan(b))
        and np.array_equal(a[~np.isnan(a)].view(np.uint64), b[~np.isnan(b)].view(np.uint64)))


@pytest.fixture(scope="module")
def rg():
    with np.load(os.path.join(GOLDEN, "round_golden.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("fmt", FMTS)
def test_round_matches_reference_golden(rg, fmt):
    x, y = rg[f"x_{fmt}"], rg[f"y_{fmt}"]
    assert same_bits(ofp.round_matrix(x, fmt), y)
    assert same_bits(omv.c_round(x, fmt), y)


def test_spec_kats(rg):
    kat = json.loads(str(rg["kat"][()]))
    assert ofp.round_matrix(7.0e4, "fp16") == np.inf == kat["7e4_fp16"]
    assert ofp.round_matrix(1 + 2.0 ** -9, "bf16") == 1.0 == kat["1p2m9_bf16"]
    assert ofp.unit_roundoff("fp16") == kat["u_fp16"]
    assert ofp.unit_roundoff("fp64") == kat["u_fp64"]
    assert ofp.unit_roundoff("q52") == kat["u_q52"] == 0.125


@pytest.mark.parametrize("fmt,dtype", [("fp16", np.float16)])
def test_exhaustive_fixed_points_fp16(fmt, dtype):
    # SPEC acceptance 1: every representable value is a fixed point.
    v = np.arange(2 ** 16, dtype=np.uint16).view(dtype).astype(np.float64)
    v = v[np.isfinite(v)]
    assert same_bits(ofp.round_matrix(v, fmt), v)


def test_exhaustive_fixed_points_bf16():
    v = (np.arange(2 ** 16, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)
    v = v[np.isfinite(v)]
    assert same_bits(ofp.round_matrix(v, "bf16"), v)


def test_round_matches_numpy_casts():
    rng = np.random.default_rng(0)
    x = np.ldexp(rng.random(200000) + 0.5, rng.integers(-160, 140, 200000))
    assert same_bits(ofp.round_matrix(x, "fp32"), x.astype(np.float32).astype(np.float64))
    y = np.ldexp(rng.random(200000) + 0.5, rng.integers(-30, 20, 200000))
    assert same_bits(ofp.round_matrix(y, "fp16"), y.astype(np.float16).astype(np.float64))


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matvec_matches_reference(name):
    H, vec, summ = load_case(name)
    X = vec["x"]
    b = omv.matvec_oracle(H, X)
    ref = vec["b_alg3"]
    if summ["working"] == "fp64":
        scale = np.linalg.norm(ref) or 1.0
        assert np.linalg.norm(b - ref) <= 1e-14 * scale
        assert np.linalg.norm(b - vec["b_dense"]) <= 1e-13 * scale
    else:
        # Strict-sequential per-op rounding is bit-identical to Arithmetic(fp32).
        assert same_bits(b, ref)


@pytest.mark.parametrize("name", ["rand96_fp32", "toep1024_e2_fp32", "depth0_fp32"])
def test_python_arith_equals_c_loop(name):
    H, vec, _ = load_case(name)
    assert same_bits(omv.matvec_arith_py(H, vec["x"]), omv.matvec_oracle(H, vec["x"]))


def test_oracle_dense_assembly():
    H, vec, _ = load_case("g512_fp64")
    D = omv.dense_of(H)
    assert np.allclose(D @ vec["x"], vec["b_dense"], rtol=0, atol=1e-12)


def test_oracle_length_mismatch():
    H, vec, _ = load_case("g512_fp64")
    with pytest.raises(ValueError):
        omv.matvec_oracle(H, np.ones(H.n + 1))


def test_cfg1_summary_is_consistent():
    with np.load(os.path.join(GOLDEN, "cfg1_summary.npz")) as z:
        s = json.loads(str(z["summary"][()]))
        assert s["formats"] == ["fp32", "fp64", "fp64", "fp64"]
        assert s["storage_bits"] == 81526784
        assert np.linalg.norm(z["b_alg3"] - z["b_dense"]) <= 1e-13 * np.linalg.norm(z["b_dense"])
