"""Round-2 golden fixtures, again generated FROM THE REFERENCE PACKAGE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_r2.py

Adds, next to the fixtures of ``make_golden.py``:

* ``narrow_golden.npz``: Algorithm 3 evaluated by the
  reference's own ``Arithmetic(working, "full-arithmetic")`` (arithmetic.py:14-67)
  in the simulated working precisions bf16, fp16 and q52 on reference-built
  matrices (the committed ``hodlr_<case>.npz`` plus ``nwhodlr_g600_bf16.npz``, a
  ragged matrix BUILT with bf16 working so its leaves are bf16 values,
  hodlr.py:193-194) -- the pins of the strict-order GPU kernels and of the
  oracle's C loop in those formats.
* ``builder_golden.json``: plan (formats, xi), per-block ranks and
  ``storage_bits`` of the reference ``build_adaptive`` (hodlr.py:227-265) on
  dense instances of the matrix-free sources: the Toeplitz kernel 1/(1+|i-j|)
  at n = 8192, the 2-D exponential kernel on Morton-sorted points and the 1-D
  Gaussian kernel (cfg3 / cfg4 analogues at sizes the reference can build).

The GPU box never sees /root/reference: tests only read these files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (puts the reference on sys.path)
from hodlrmp import fpsim, hodlr, tree  # noqa: E402

NARROW = (fpsim.BF16, fpsim.FP16, fpsim.Q52)
NARROW_CASES = ["g512_fp64", "toep1024_e4_fp64", "rand96_fp32", "toep512_e3_fp64", "depth0_fp32"]


def make_narrow():
    out = {}
    # a matrix whose leaves are bf16 values (built with bf16 working), ragged tree
    A = mg.gaussian_1d(600, 0.05, 1e-2, 11)
    H = hodlr.build_adaptive(A, tree.build_tree(600, 3), 1e-2, working=fpsim.BF16, available=mg.ALL)
    hodlr.save_hodlr(H, os.path.join(HERE, "nwhodlr_g600_bf16.npz"))  # (not hodlr_*: outside golden_cases())
    rng = np.random.default_rng(600)
    X = rng.uniform(-1.0, 1.0, size=(600, 2))
    out["g600_bf16__x"] = X
    out["g600_bf16__KX"] = A @ X
    out["g600_bf16__normA"] = np.linalg.norm(A)
    for w in NARROW + (fpsim.FP32,):
        out[f"g600_bf16__{w.name}"] = mg.alg3_reference(H, X, w)
    print("g600_bf16", mg.summary(H)["formats"], mg.summary(H)["ranks"])
    for name in NARROW_CASES:
        H = hodlr.load_hodlr(os.path.join(HERE, f"hodlr_{name}.npz"))
        with np.load(os.path.join(HERE, f"vec_{name}.npz")) as z:
            X = z["x"]
        X = X.reshape(H.n, -1)[:, :2]
        out[f"{name}__x"] = X
        for w in NARROW:
            out[f"{name}__{w.name}"] = mg.alg3_reference(H, X, w)
        print(name, "done")
    np.savez_compressed(os.path.join(HERE, "narrow_golden.npz"), **out)


def morton_order(P, bits=16):
    q = np.minimum((P * (1 << bits)).astype(np.uint64), (1 << bits) - 1)
    code = np.zeros(len(P), dtype=np.uint64)
    for b in range(bits):
        code |= ((q[:, 0] >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
        code |= ((q[:, 1] >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b + 1)
    return np.argsort(code, kind="stable")


def make_builder():
    cases = {}

    def record(name, A, depth, eps, working, extra):
        H = hodlr.build_adaptive(A, tree.build_tree(A.shape[0], depth), eps, working=working, available=mg.ALL)
        s = mg.summary(H)
        s.update(extra)
        cases[name] = s
        print(name, s["formats"], [r[0] for r in s["ranks"]][:6], s["storage_bits"])

    record("toeplitz_inv_8192", mg.toeplitz_inv(8192), 5, 1e-6, fpsim.FP64, {"kernel": "1/(1+|i-j|)"})
    record("toeplitz_inv_4096_e2", mg.toeplitz_inv(4096), 4, 1e-2, fpsim.FP32, {"kernel": "1/(1+|i-j|)"})
    P = np.random.default_rng(0).random((4096, 2))
    P = P[morton_order(P)]
    D = np.sqrt(((P[:, None, :] - P[None, :, :]) ** 2).sum(-1))
    record("exp2d_morton_4096", np.exp(-D / 0.2), 4, 1e-4, fpsim.FP32,
           {"kernel": "exp(-|p_i-p_j|/0.2), p = default_rng(0).random((4096,2)) Morton-sorted"})
    t = np.sort(np.random.default_rng(0).random(8192))
    record("gauss1d_8192", np.exp(-((t[:, None] - t[None, :]) ** 2) / (2 * 0.01 ** 2)), 5, 1e-6, fpsim.FP64,
           {"kernel": "exp(-(t_i-t_j)^2/(2*0.01^2)), t = sort(default_rng(0).random(8192))"})
    with open(os.path.join(HERE, "builder_golden.json"), "w") as f:
        json.dump(cases, f, indent=1)


if __name__ == "__main__":
    make_narrow()
    make_builder()
