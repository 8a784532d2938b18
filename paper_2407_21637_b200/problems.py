"""Seeded synthetic inputs of the BASELINE configurations (BASELINE.json).

The paper's experiments use kernel matrices on point
sets; BASELINE.json fixes five configurations.  Everything is generated from
the seeds recorded here:

  cfg1  n=4096, l=4:  A = exp(-(t_i-t_j)^2 / (2*0.05^2)) + 1e-2 I,
        t = sort(default_rng(0).random(n)); eps 1e-8; fp64 working;
        x = default_rng(1).standard_normal(n).
  cfg2  n=65536, l=8: A = 1/(1+|i-j|) (Toeplitz); eps 1e-6; fp64 working;
        x = default_rng(2).standard_normal(n).
  cfg5  n=262144, l=10: cfg2's kernel; eps in {1e-2,...,1e-10};
        fp32 working for eps >= 1e-4, else fp64.
(cfg3 / cfg4 sources are listed in DESIGN.md as next rows.)
"""

from __future__ import annotations

import math

import numpy as np

from .construct import BlockSource, DenseSource, build_adaptive
from .formats import BF16, FP16, FP32, FP64, Q52
from .model import build_tree

ALL_FORMATS = (Q52, BF16, FP16, FP32, FP64)


def gaussian_1d_dense(n: int, sigma: float, nugget: float, seed: int) -> np.ndarray:
    t = np.sort(np.random.default_rng(seed).random(n))
    A = np.exp(-((t[:, None] - t[None, :]) ** 2) / (2.0 * sigma * sigma))
    if nugget:
        A[np.diag_indices(n)] += nugget
    return A


class ToeplitzInvSource(BlockSource):
    """A_ij = 1 / (1 + |i - j|).

    Blocks up to ``dense_max`` rows are generated densely on the GPU; larger
    off-diagonal blocks (cfg5's level 1 is 131072^2 = 137 GB dense) are never
    formed: they are Toeplitz, so ||B||_F^2 comes exactly from the distance
    counts and the randomized range finder applies B and B^T by FFT
    convolution (O(m log m) per column)."""

    dense_max = 32768
    sketch = 96

    @staticmethod
    def f(t):
        return 1.0 / (1.0 + np.abs(t))

    def block(self, a, b, c, d):
        import torch

        i = torch.arange(a, b, device=self.device, dtype=torch.float64)[:, None]
        j = torch.arange(c, d, device=self.device, dtype=torch.float64)[None, :]
        return 1.0 / (1.0 + (i - j).abs())

    def frob2_all(self) -> float:
        n = self.n
        dist = np.arange(1, n, dtype=np.float64)
        return float(n) + 2.0 * math.fsum((n - dist) / (1.0 + dist) ** 2)

    def block_frob2(self, a, b, c, d) -> float:
        m, k = b - a, d - c
        delta = np.arange(-(m - 1), k, dtype=np.int64)      # j - i
        cnt = np.where(delta >= 0, np.minimum(m, k - delta), np.minimum(k, m + delta)).astype(np.float64)
        return math.fsum(cnt * self.f((c - a) + delta).astype(np.float64) ** 2)

    # B X for B = A[a:b, c:d], B_ij = f(o + j - i) with o = c - a (f is even, so
    # B^T has the same form with o -> -o), X: k x L, by FFT correlation.
    def _apply(self, a, b, c, d, X, transpose=False):
        m, k, o = b - a, d - c, c - a
        if transpose:
            m, k, o = k, m, -o
        h = self.f(o + np.arange(-(m - 1), k, dtype=np.int64))   # h[t + m - 1] = f(o + t)
        nfft = 1 << int(np.ceil(np.log2(len(h) + k)))
        full = np.fft.irfft(np.fft.rfft(h[::-1], nfft)[:, None] * np.fft.rfft(X, nfft, axis=0), nfft, axis=0)
        return full[k - 1:k - 1 + m]                              # y_i = conv[k - 1 + i]

    def compress(self, a, b, c, d, eps, cache=None):
        if min(b - a, d - c) <= self.dense_max:
            return super().compress(a, b, c, d, eps, cache)
        import torch

        from .construct import truncation_rank

        key = (a, b, c, d, eps)
        if cache is not None and key in cache:
            return cache[key]
        m, k = b - a, d - c
        rng = np.random.default_rng(self.seed)
        Lw = min(self.sketch, m, k)
        Om = rng.standard_normal((k, Lw))
        Q, _ = np.linalg.qr(self._apply(a, b, c, d, Om))
        for _ in range(self.power_iters):
            Z, _ = np.linalg.qr(self._apply(a, b, c, d, Q, transpose=True))
            Q, _ = np.linalg.qr(self._apply(a, b, c, d, Z))
        Ct = self._apply(a, b, c, d, Q, transpose=True)          # B^T Q  (k x Lw) = C^T
        Uc, s, Vh = np.linalg.svd(Ct.T, full_matrices=False)
        frob2 = self.block_frob2(a, b, c, d)
        # the sketch resolves the spectrum far below eps (kernel decays exponentially);
        # the unresolved remainder is bounded by s[-1] and dropped
        r = truncation_rank(s, eps, max(m, k), resid2=0.0, frob=math.sqrt(frob2))
        U = torch.from_numpy(np.ascontiguousarray(Q @ Uc[:, :r])).to(self.device)
        V = torch.from_numpy(np.ascontiguousarray(Vh[:r].T * s[:r])).to(self.device)
        out = (U, V)
        if cache is not None:
            cache[key] = out
        return out


def cfg1(seed_x: int = 1):
    """BASELINE config 1, built exactly as the reference does (dense, LAPACK)."""
    n, depth, eps = 4096, 4, 1e-8
    A = gaussian_1d_dense(n, 0.05, 1e-2, 0)
    H = build_adaptive(DenseSource(A), build_tree(n, depth), eps, FP64, ALL_FORMATS)
    x = np.random.default_rng(seed_x).standard_normal(n)
    return H, x, A


def toeplitz_config(n: int, depth: int, eps: float, working, seed_x: int, svd_cache=None):
    src = ToeplitzInvSource(n)
    H = build_adaptive(src, build_tree(n, depth), eps, working, ALL_FORMATS, svd_cache=svd_cache,
                       same_blocks_per_level=True, symmetric=True)
    x = np.random.default_rng(seed_x).standard_normal(n)
    return H, x, src


def cfg2():
    return toeplitz_config(65536, 8, 1e-6, FP64, 2)


CFG5_EPS = (1e-2, 1e-4, 1e-6, 1e-8, 1e-10)


def cfg5(eps: float, svd_cache=None):
    working = FP32 if eps >= 1e-4 else FP64
    return toeplitz_config(262144, 10, eps, working, 5, svd_cache)


def toeplitz_times(x: np.ndarray, device=None) -> np.ndarray:
    """K x for A = 1/(1+|i-j|) in binary64 on the GPU, exactly evaluated in
    row blocks (harness: the judged tolerance's reference product)."""
    import torch

    X = torch.from_numpy(np.asarray(x, np.float64).reshape(len(x), -1)).cuda(device)
    n = X.shape[0]
    out = torch.empty_like(X)
    j = torch.arange(n, device=X.device, dtype=torch.float64)[None, :]
    step = max(1, (1 << 27) // n)
    for a in range(0, n, step):
        b = min(n, a + step)
        i = torch.arange(a, b, device=X.device, dtype=torch.float64)[:, None]
        out[a:b] = (1.0 / (1.0 + (i - j).abs())) @ X
    r = out.cpu().numpy()
    return r[:, 0] if np.ndim(x) == 1 else r
