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
  cfg3  n=262144, l=10: A = exp(-||p_i - p_j|| / 0.2), p = default_rng(0).random((n, 2))
        sorted by Morton order (16-bit quantisation per axis, x bits even, y bits
        odd, stable argsort); eps 1e-4; fp32 working; X = default_rng(3)
        .standard_normal((n, 64)) rounded to fp32.
  cfg4  n=2^20, l=12: A = exp(-(t_i-t_j)^2 / (2*0.01^2)), t = sort(default_rng(0)
        .random(n)) (no nugget); eps 1e-6; fp64 working; X = default_rng(4)
        .standard_normal((n, 16)).
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


class PointKernelSource(BlockSource):
    """A_ij = f(||p_i - p_j||) for points p (n x dim), generated tile by tile on
    the GPU in binary64; nothing n x n is ever formed.

    * norms: exact sums of squares over tiles (tiles farther apart than
      ``cutoff`` -- where f is below 1e-20 of its peak -- are skipped; only the
      1-D sorted case uses it);
    * blocks up to ``dense_max`` per side: dense GPU SVD / randomized SVD of the
      generated block (BlockSource);
    * larger blocks: randomized range finder (oversampled, power iterations)
      whose products B @ Om, B^T @ Q and Q^T @ B stream the block in tiles,
      with the truncation tail taken from the explicitly computed residual
      ||B - Q Q^T B||_F^2 (also tiled)."""

    dense_max = 8192
    tile = 8192

    def __init__(self, points, f, cutoff=None, device=None):
        import torch

        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim == 1:
            pts = pts[:, None]
        super().__init__(len(pts), device)
        self.dim = pts.shape[1]
        self.f = f
        self.cutoff = cutoff
        self.pts_np = pts
        self.pts = torch.from_numpy(pts).to(self.device)

    # ---- tiles
    def block(self, a, b, c, d):
        return self.f(self._dist(self.pts[a:b], self.pts[c:d]))

    def _dist(self, P, Q):
        """Exact pairwise distances (no |p|^2 + |q|^2 - 2 p.q expansion).
        P: (..., m, dim), Q: (..., k, dim)."""
        import torch

        if self.dim == 1:
            return (P[..., :, 0:1] - Q[..., :, 0].unsqueeze(-2)).abs()
        acc = None
        for k in range(self.dim):
            t = (P[..., :, k:k + 1] - Q[..., :, k].unsqueeze(-2)) ** 2
            acc = t if acc is None else acc + t
        return torch.sqrt(acc)

    def _far(self, a, b, c, d):
        """Every entry of A[a:b, c:d] negligible (1-D sorted points only)."""
        if self.cutoff is None or self.dim != 1:
            return False
        t = self.pts_np[:, 0]
        gap = max(t[c] - t[b - 1], t[a] - t[d - 1], 0.0)
        return gap > self.cutoff

    def _tiles(self, a, b, c, d):
        T = self.tile
        for i0 in range(a, b, T):
            i1 = min(b, i0 + T)
            for j0 in range(c, d, T):
                j1 = min(d, j0 + T)
                if not self._far(i0, i1, j0, j1):
                    yield i0, i1, j0, j1

    def block_frob2(self, a, b, c, d) -> float:
        tot = 0.0
        for i0, i1, j0, j1 in self._tiles(a, b, c, d):
            B = self.block(i0, i1, j0, j1)
            tot += float((B * B).sum())
        return tot

    def frob2_all(self) -> float:
        n, T = self.n, self.tile
        tot = 0.0
        for i0 in range(0, n, T):
            i1 = min(n, i0 + T)
            tot += self.block_frob2(i0, i1, i0, i1)
            if i1 < n:
                tot += 2.0 * self.block_frob2(i0, i1, i1, n)
        return tot

    # ---- tiled products with B = A[a:b, c:d]
    def _apply(self, a, b, c, d, X):  # B @ X, X: (d-c) x L
        import torch

        Y = torch.zeros((b - a, X.shape[1]), dtype=torch.float64, device=self.device)
        for i0, i1, j0, j1 in self._tiles(a, b, c, d):
            Y[i0 - a:i1 - a] += self.block(i0, i1, j0, j1) @ X[j0 - c:j1 - c]
        return Y

    def _apply_t(self, a, b, c, d, X):  # B^T @ X, X: (b-a) x L
        import torch

        Y = torch.zeros((d - c, X.shape[1]), dtype=torch.float64, device=self.device)
        for i0, i1, j0, j1 in self._tiles(a, b, c, d):
            Y[j0 - c:j1 - c] += self.block(i0, i1, j0, j1).T @ X[i0 - a:i1 - a]
        return Y

    def _resid2(self, a, b, c, d, Q, C):
        tot = 0.0
        for i0, i1, j0, j1 in self._tiles(a, b, c, d):
            R = self.block(i0, i1, j0, j1) - Q[i0 - a:i1 - a] @ C[:, j0 - c:j1 - c]
            tot += float((R * R).sum())
        # skipped (far) tiles hold B ~ 0, where the residual is -Q C ~ 0 as well
        return tot

    def compress(self, a, b, c, d, eps, cache=None):
        if min(b - a, d - c) <= self.dense_max:
            return super().compress(a, b, c, d, eps, cache)
        import torch

        from .construct import truncation_rank

        key = (a, b, c, d, eps)
        if cache is not None and key in cache:
            return cache[key]
        m, k = b - a, d - c
        frob = math.sqrt(self.block_frob2(a, b, c, d))
        if frob == 0.0:
            z = torch.zeros((m, 0), dtype=torch.float64, device=self.device)
            return z, torch.zeros((k, 0), dtype=torch.float64, device=self.device)
        g = torch.Generator(device=self.device)
        g.manual_seed(self.seed)
        L = 64
        while True:
            Om = torch.randn((k, L), dtype=torch.float64, device=self.device, generator=g)
            Q, _ = torch.linalg.qr(self._apply(a, b, c, d, Om))
            for _ in range(self.power_iters):
                Z, _ = torch.linalg.qr(self._apply_t(a, b, c, d, Q))
                Q, _ = torch.linalg.qr(self._apply(a, b, c, d, Z))
            C = self._apply_t(a, b, c, d, Q).T  # Q^T B  (L x k)
            resid2 = self._resid2(a, b, c, d, Q, C)
            Uc, s, Vh = torch.linalg.svd(C, full_matrices=False)
            r = truncation_rank(s.cpu().numpy(), eps, max(m, k), resid2=resid2, frob=frob)
            if r < L - 8 or L >= min(m, k):
                out = ((Q @ Uc[:, :r]).contiguous(), Vh[:r].T * s[:r])
                if cache is not None:
                    cache[key] = out
                return out
            L *= 2


    def compress_level(self, rects, eps, cache=None):
        """Compress equal-shape blocks [(a, b, c, d), ...] of one level together:
        batched generation and a batched randomized range finder (one set of
        GPU launches per level instead of per block).  Same truncation rule as
        ``compress``: explicit residual, smallest rank meeting eps ||B||_F."""
        import torch

        from .construct import truncation_rank

        m, k = rects[0][1] - rects[0][0], rects[0][3] - rects[0][2]
        if any((b - a, d - c) != (m, k) for a, b, c, d in rects) or min(m, k) > self.dense_max:
            return [self.compress(*r, eps, cache) for r in rects]
        out = [None] * len(rects)
        per = max(1, int((1 << 31) // (8 * m * k * 3)))  # ~2 GB of blocks per batch
        for i0 in range(0, len(rects), per):
            chunk = rects[i0:i0 + per]
            ia = torch.tensor([a for a, _, _, _ in chunk], device=self.device)
            ic = torch.tensor([c for _, _, c, _ in chunk], device=self.device)
            ri = ia[:, None] + torch.arange(m, device=self.device)[None, :]
            ci = ic[:, None] + torch.arange(k, device=self.device)[None, :]
            B = self.f(self._dist(self.pts[ri], self.pts[ci]))  # (nb, m, k)
            frob = torch.linalg.norm(B, dim=(1, 2)).cpu().numpy()
            L = min(64, m, k)
            todo = list(range(len(chunk)))
            g = torch.Generator(device=self.device)
            g.manual_seed(self.seed)
            while todo:
                Bt = B[todo]
                Om = torch.randn((k, L), dtype=torch.float64, device=self.device, generator=g)
                Q, _ = torch.linalg.qr(Bt @ Om)
                for _ in range(self.power_iters):
                    Z, _ = torch.linalg.qr(Bt.transpose(1, 2) @ Q)
                    Q, _ = torch.linalg.qr(Bt @ Z)
                C = Q.transpose(1, 2) @ Bt
                R = Bt - Q @ C
                resid2 = (R * R).sum(dim=(1, 2)).cpu().numpy()
                del R
                Uc, sv, Vh = torch.linalg.svd(C, full_matrices=False)
                sv_np = sv.cpu().numpy()
                again = []
                for j, bi in enumerate(todo):
                    if frob[bi] == 0.0:
                        out[i0 + bi] = (torch.zeros((m, 0), dtype=torch.float64, device=self.device),
                                        torch.zeros((k, 0), dtype=torch.float64, device=self.device))
                        continue
                    r = truncation_rank(sv_np[j], eps, max(m, k), resid2=float(resid2[j]), frob=float(frob[bi]))
                    if r < L - 8 or L >= min(m, k):
                        out[i0 + bi] = ((Q[j] @ Uc[j, :, :r]).contiguous(), Vh[j, :r].T * sv[j, :r])
                    else:
                        again.append(bi)
                todo = again
                L = min(2 * L, m, k)
            del B
        return out


def morton_order(P: np.ndarray, bits: int = 16) -> np.ndarray:
    """Stable argsort by Morton code: coordinates quantised to 2^bits levels,
    x bits at even positions, y bits at odd positions."""
    q = np.minimum((P * (1 << bits)).astype(np.int64), (1 << bits) - 1)
    code = np.zeros(len(P), dtype=np.int64)
    for bit in range(bits):
        code |= ((q[:, 0] >> bit) & 1) << (2 * bit)
        code |= ((q[:, 1] >> bit) & 1) << (2 * bit + 1)
    return np.argsort(code, kind="stable")


def cfg3(n: int = 262144, depth: int = 10, s: int = 64):
    """BASELINE config 3 (or a same-distribution analog at smaller n)."""
    import torch

    from .formats import FP32 as W

    P = np.random.default_rng(0).random((n, 2))
    P = P[morton_order(P)]
    src = PointKernelSource(P, lambda r: torch.exp(-r / 0.2))
    H = build_adaptive(src, build_tree(n, depth), 1e-4, W, ALL_FORMATS, symmetric=True)
    X = np.random.default_rng(3).standard_normal((n, s)).astype(np.float32).astype(np.float64)
    return H, X, src


def cfg4(n: int = 1 << 20, depth: int = 12, s: int = 16):
    """BASELINE config 4 (or a same-distribution analog at smaller n)."""
    import torch

    sigma = 0.01
    t = np.sort(np.random.default_rng(0).random(n))
    src = PointKernelSource(t, lambda r: torch.exp(-(r * r) / (2.0 * sigma * sigma)),
                            cutoff=sigma * math.sqrt(2.0 * 46.1))  # exp(-46.1) = 1e-20
    H = build_adaptive(src, build_tree(n, depth), 1e-6, FP64, ALL_FORMATS, symmetric=True)
    X = np.random.default_rng(4).standard_normal((n, s))
    return H, X, src


def kernel_times(src, X, device=None):
    """K X in binary64 on the GPU, exactly, tile by tile (harness: the judged
    tolerance's reference product for the point-kernel configs)."""
    import torch

    Xd = torch.from_numpy(np.asarray(X, np.float64).reshape(src.n, -1)).to(src.device)
    Y = src._apply(0, src.n, 0, src.n, Xd)
    r = Y.cpu().numpy()
    return r[:, 0] if np.ndim(X) == 1 else r


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
