"""K0 on the device: bit-exact against the reference's round_matrix golden
vectors and exhaustive fixed-point checks (SPEC.md:649 acceptance 1)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.fpsim import round_matrix

pytestmark = pytest.mark.gpu
CODES = {"q52": 0, "bf16": 1, "fp16": 2, "fp32": 3, "fp64": 4}
TORCH_T = {0: "uint8", 1: "int16", 2: "int16", 3: "float32", 4: "float64"}


def dev_roundtrip(torch, fmt, x):
    from paper_2407_21637_b200 import _lib

    L = _lib.lib()
    xd = torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()
    q = torch.empty(x.size, dtype=getattr(torch, TORCH_T[fmt]), device="cuda")
    y = torch.empty_like(xd)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.hodlr_quantize(fmt, xd.data_ptr(), q.data_ptr(), x.size, s))
    _lib.check(L.hodlr_dequantize(fmt, q.data_ptr(), y.data_ptr(), x.size, s))
    torch.cuda.synchronize()
    return q.cpu().numpy(), y.cpu().numpy()


def assert_bits(y, want):
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(y), nan)
    assert np.array_equal(y[~nan].view(np.uint64), want[~nan].view(np.uint64))


@pytest.mark.parametrize("name", ["q52", "bf16", "fp16", "fp32"])
def test_device_k0_vs_reference_golden(cuda, name):
    with np.load(os.path.join(GOLDEN, "round_golden.npz")) as z:
        x, want = z[f"x_{name}"], z[f"y_{name}"]
    _, y = dev_roundtrip(cuda, CODES[name], x)
    assert_bits(y, want)


@pytest.mark.parametrize("name", ["q52", "bf16", "fp16", "fp32"])
def test_device_k0_adversarial_large(cuda, name):
    """1M fresh adversarial inputs per format against the oracle restatement
    (itself pinned to the reference by tests/test_oracle.py)."""
    rng = np.random.default_rng(CODES[name] + 100)
    from oracle.fpsim import FORMATS

    f = FORMATS[name]
    n = 1 << 20
    e = rng.integers(f.e_min - f.t - 2, f.e_max + 2, n)
    x = np.ldexp(rng.random(n) + 0.5, e)
    q = np.maximum(e - f.t, f.e_min - f.t + 1)
    mids = np.ldexp(np.floor(np.ldexp(x, -q)) + 0.5, q)
    x = np.concatenate([x, mids, np.nextafter(mids, 0), np.nextafter(mids, np.inf), -mids])
    _, y = dev_roundtrip(cuda, CODES[name], x)
    assert_bits(y, round_matrix(x, name))


def test_device_k0_exhaustive_fixed_points(cuda):
    v16 = np.arange(2 ** 16, dtype=np.uint16).view(np.float16).astype(np.float64)
    v16 = v16[np.isfinite(v16)]
    _, y = dev_roundtrip(cuda, CODES["fp16"], v16)
    assert_bits(y, v16)
    vb = (np.arange(2 ** 16, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)
    vb = vb[np.isfinite(vb)]
    _, y = dev_roundtrip(cuda, CODES["bf16"], vb)
    assert_bits(y, vb)
    v8 = (np.arange(256, dtype=np.uint16) << 8).view(np.float16).astype(np.float64)
    v8 = v8[np.isfinite(v8)]
    _, y = dev_roundtrip(cuda, CODES["q52"], v8)
    assert_bits(y, v8)


def test_device_encoding_is_native_layout(cuda):
    x = np.random.default_rng(3).standard_normal(4096) * 10
    q, _ = dev_roundtrip(cuda, CODES["fp16"], x)
    assert np.array_equal(q.view(np.uint16), x.astype(np.float16).view(np.uint16))
    q, _ = dev_roundtrip(cuda, CODES["bf16"], x)
    hi = (q.view(np.uint16).astype(np.uint32) << 16).view(np.float32)
    assert np.array_equal(hi.astype(np.float64), round_matrix(x, "bf16"))
