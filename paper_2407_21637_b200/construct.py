"""Adaptive-precision HODLR construction -- the input producer of the matvec.

Restates the reference builder so the BASELINE configurations can be built
where the reference cannot (its ``build_adaptive`` needs the dense n x n
matrix, an n x n temporary and a dense SVD per block: configs 2-5 need
0.07-8.8 TB):

* Alg. 2 / ``build_adaptive`` (hodlr.py:227-265): level
  weights xi_k = max_pair ||off-diagonal block||_F / ||A||_F from the original
  blocks in binary64; admissible roundoff eps / (2^(k/2) xi_k)
  (``admissible_roundoff``, hodlr.py:138-144); coarsest admissible format of
  {working} u available, else working + fallback flag (``select_level_format``,
  hodlr.py:147-161).
* Truncation (``_truncation_rank`` / ``truncate_from_svd``, lowrank.py:80-99):
  smallest r with ||s[r:]||_2 <= eps ||B||_F; U = left singular vectors,
  V = right singular vectors scaled by s.
* ``store_factor`` (lowrank.py:117-119) and leaf rounding (hodlr.py:193-194):
  quantisation through K0 (bit-exact ``round_matrix``) -- the device kernel
  when the builder runs on the GPU, its host compilation otherwise.

Backends: ``DenseSource`` (numpy A, LAPACK gesdd with gesvd fallback -- the
reference's own SVD path, lowrank.py:70-77) and ``BlockSource`` subclasses that
generate blocks on the GPU in binary64 (torch: cuBLAS / cuSOLVER, harness code,
not the hot path) with a randomized range finder whose truncation tail is
computed from the explicit residual, so the rank rule is applied to
sigma_{r..L} plus the residual norm without cancellation.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .formats import FP64, format_code, format_spec
from .model import HodlrMatrix, LowRankFactor, PrecisionPlan

__all__ = [
    "admissible_roundoff", "select_level_format", "truncation_rank", "quantize",
    "DenseSource", "BlockSource", "build_adaptive",
]

_NP_ENC = {0: np.uint8, 1: np.uint16, 2: np.uint16, 3: np.float32, 4: np.float64}


def admissible_roundoff(eps: float, k: int, xi: float) -> float:
    if xi < 0:
        raise ValueError("level weight must be nonnegative")
    if xi == 0.0:
        return math.inf
    return eps / (2.0 ** (k / 2.0) * xi)


def select_level_format(threshold: float, working, available):
    cands = {format_spec(f): f for f in (working, *available)}
    ok = [f for f in cands.values() if f.unit_roundoff <= threshold]
    if not ok:
        return working, True
    return max(ok, key=lambda f: (f.unit_roundoff, f.name)), False


def truncation_rank(s: np.ndarray, eps: float, nmax: int, resid2: float = 0.0,
                    frob: float | None = None) -> int:
    """Smallest r with ||s[r:]|| (plus an unresolved residual) <= eps * ||B||_F.

    With a full SVD (resid2 = 0, frob = None) this is lowrank.py:80-91 exactly:
    tails[0] = ||s|| = ||B||_F; eps == 0 keeps the numerical rank."""
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0:
        return 0
    if eps == 0.0:
        return int(np.count_nonzero(s > nmax * 2.0 ** -53 * s[0]))
    tails = np.sqrt(np.cumsum(s[::-1] ** 2)[::-1] + resid2)
    ref = tails[0] if frob is None else frob
    ok = np.concatenate([tails <= eps * ref, [True]])
    return int(np.argmax(ok))


def quantize(a, fmt):
    """round_matrix(a, fmt) through K0 (host build, or the device kernel for
    CUDA tensors): returns binary64 values on the input's side."""
    code = format_code(fmt)
    L = _lib.lib()
    try:
        import torch

        if isinstance(a, torch.Tensor):
            a = a.contiguous().double()
            if code == 4:
                return a.clone()
            enc = torch.empty(a.numel() * _lib_bytes(code), dtype=torch.uint8, device=a.device)
            out = torch.empty_like(a)
            st = torch.cuda.current_stream(a.device).cuda_stream
            _lib.check(L.hodlr_quantize(code, a.data_ptr(), enc.data_ptr(), a.numel(), st))
            _lib.check(L.hodlr_dequantize(code, enc.data_ptr(), out.data_ptr(), a.numel(), st))
            return out
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(a, dtype=np.float64)
    if code == 4:
        return a.copy()
    enc = np.empty(a.size, _NP_ENC[code])
    out = np.empty_like(a)
    _lib.check(L.hodlr_quantize_host(code, a.ctypes.data, enc.ctypes.data, a.size))
    _lib.check(L.hodlr_dequantize_host(code, enc.ctypes.data, out.ctypes.data, a.size))
    return out


def _lib_bytes(code):
    return {0: 1, 1: 2, 2: 2, 3: 4, 4: 8}[code]


# ---------------------------------------------------------------- sources
class DenseSource:
    """A dense binary64 matrix in host memory; SVDs by LAPACK like the reference."""

    def __init__(self, A):
        A = np.asarray(A, dtype=np.float64)
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise ValueError(f"expected a square matrix, got shape {A.shape}")
        self.A = A
        self.n = A.shape[0]

    def frob2_all(self) -> float:
        return float(np.sum(self.A * self.A))

    def block_frob2(self, a, b, c, d) -> float:
        return float(np.sum(self.A[a:b, c:d] ** 2))

    def leaf(self, a, b):
        return self.A[a:b, a:b]

    def compress(self, a, b, c, d, eps, cache=None):
        key = (a, b, c, d)
        if cache is not None and key in cache:
            U, s, Vt = cache[key]
        else:
            B = self.A[a:b, c:d]
            if not np.all(np.isfinite(B)):
                raise ValueError("cannot compress a block with non-finite entries")
            try:
                U, s, Vt = np.linalg.svd(B, full_matrices=False)
            except np.linalg.LinAlgError:
                import scipy.linalg

                U, s, Vt = scipy.linalg.svd(B, full_matrices=False, lapack_driver="gesvd")
            if cache is not None:
                cache[key] = (U, s, Vt)
        r = truncation_rank(s, eps, max(b - a, d - c))
        return np.ascontiguousarray(U[:, :r]), Vt[:r].T * s[:r]


class BlockSource:
    """Matrix-free source: subclasses generate blocks A[a:b, c:d] on the GPU
    (torch float64).  Truncation by a randomized range finder (oversampled,
    power iterations, re-orthonormalised) with the residual norm measured
    explicitly; blocks up to ``dense_svd_max`` use a full GPU SVD."""

    dense_svd_max = 2048
    power_iters = 2
    seed = 1234

    def __init__(self, n: int, device=None):
        import torch

        self.n = int(n)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)

    # subclasses implement these two
    def block(self, a, b, c, d):  # -> torch (b-a) x (d-c) float64 on self.device
        raise NotImplementedError

    def frob2_all(self) -> float:
        raise NotImplementedError

    def block_frob2(self, a, b, c, d) -> float:
        B = self.block(a, b, c, d)
        return float((B * B).sum())

    def leaf(self, a, b):
        return self.block(a, b, a, b)

    def compress(self, a, b, c, d, eps, cache=None):
        import torch

        key = (a, b, c, d, eps)
        if cache is not None and key in cache:
            return cache[key]
        B = self.block(a, b, c, d)
        m, k = B.shape
        frob = float(torch.linalg.norm(B))
        if frob == 0.0:
            out = (torch.zeros((m, 0), dtype=B.dtype, device=B.device),
                   torch.zeros((k, 0), dtype=B.dtype, device=B.device))
        elif min(m, k) <= self.dense_svd_max:
            U, s, Vh = torch.linalg.svd(B, full_matrices=False)
            r = truncation_rank(s.cpu().numpy(), eps, max(m, k))
            out = (U[:, :r].contiguous(), Vh[:r].T * s[:r])
        else:
            out = self._rsvd(B, eps, frob)
        if cache is not None:
            cache[key] = out
        return out

    def _rsvd(self, B, eps, frob):
        import torch

        m, k = B.shape
        g = torch.Generator(device=B.device)
        g.manual_seed(self.seed)
        L = 48
        while True:
            L = min(L, min(m, k))
            Om = torch.randn((k, L), dtype=B.dtype, device=B.device, generator=g)
            Q, _ = torch.linalg.qr(B @ Om)
            for _ in range(self.power_iters):
                Z, _ = torch.linalg.qr(B.T @ Q)
                Q, _ = torch.linalg.qr(B @ Z)
            C = Q.T @ B
            R = B - Q @ C
            resid2 = float((R * R).sum())
            del R
            Uc, s, Vh = torch.linalg.svd(C, full_matrices=False)
            s_np = s.cpu().numpy()
            r = truncation_rank(s_np, eps, max(m, k), resid2=resid2, frob=frob)
            if r < L - 8 or L >= min(m, k):
                U = Q @ Uc[:, :r]
                return U.contiguous(), Vh[:r].T * s[:r]
            L *= 2


# ---------------------------------------------------------------- builder
def build_adaptive(source, tree, eps: float, working=FP64, available=(), svd_cache=None,
                   same_blocks_per_level: bool = False, symmetric: bool = False) -> HodlrMatrix:
    """Alg. 2 over ``source`` (DenseSource or a BlockSource).

    ``same_blocks_per_level``: every sibling pair of a level has the same upper
    block and the same lower block (Toeplitz kernels on a uniform grid with a
    uniform tree) -- compressed once per level and shared.  ``symmetric``: the
    lower block is the transpose of the upper one (A = A^T).
    """
    if not 0.0 <= eps < 1.0:
        raise ValueError(f"tolerance {eps} outside [0, 1)")
    if source.n != tree.n:
        raise ValueError(f"dimension mismatch: matrix {source.n}, tree {tree.n}")
    gpu = isinstance(source, BlockSource)
    nrm_all = source.frob2_all()
    xi, thr, chosen, fb = [], [], [], []
    for k in range(1, tree.depth + 1):
        lvl = tree.ranges[k]
        nrm = 0.0
        pairs = [0] if same_blocks_per_level else range(0, 2 ** k, 2)
        for p in pairs:
            (a, b), (c, d) = lvl[p], lvl[p + 1]
            up = source.block_frob2(a, b, c, d)
            lo = up if symmetric else source.block_frob2(c, d, a, b)
            nrm = max(nrm, up, lo)
        x = math.sqrt(nrm / nrm_all) if nrm_all > 0.0 else 0.0
        t = admissible_roundoff(eps, k, x)
        f, flag = select_level_format(t, working, available)
        xi.append(x)
        thr.append(t)
        chosen.append(f)
        fb.append(flag)
    plan = PrecisionPlan(chosen, xi, thr, fb)

    def to_host(a):
        return a.cpu().numpy() if gpu else a

    def store(U, V, fmt):
        return LowRankFactor(to_host(quantize(U, fmt)), np.asfortranarray(to_host(quantize(V, fmt))), fmt)

    leaves = []
    leaf_cache = {}
    for a, b in tree.ranges[tree.depth]:
        key = (b - a) if same_blocks_per_level else None
        if key is not None and key in leaf_cache:
            leaves.append(leaf_cache[key])
            continue
        blk = to_host(quantize(source.leaf(a, b), working))
        if key is not None:
            leaf_cache[key] = blk
        leaves.append(blk)
    blocks = []
    for k in range(1, tree.depth + 1):
        lvl = tree.ranges[k]
        fmt = chosen[k - 1]
        row = []
        shared = None
        batch = None
        if hasattr(source, "compress_level") and not same_blocks_per_level:
            rects = [(*lvl[2 * i], *lvl[2 * i + 1]) for i in range(2 ** (k - 1))]
            batch = source.compress_level(rects, eps, svd_cache)
        for i in range(2 ** (k - 1)):
            if same_blocks_per_level and shared is not None:
                row.append(shared)
                continue
            (a, b), (c, d) = lvl[2 * i], lvl[2 * i + 1]
            Uu, Vu = batch[i] if batch is not None else source.compress(a, b, c, d, eps, svd_cache)
            if symmetric:
                # lower = upper^T = (V/s)(s)(U)^T : re-normalise so lower.U is orthonormal
                if gpu:
                    import torch

                    sv = torch.linalg.norm(Vu, dim=0)
                    safe = torch.where(sv > 0, sv, torch.ones_like(sv))
                    Ul, Vl = Vu / safe, Uu * sv
                else:
                    sv = np.linalg.norm(Vu, axis=0)
                    safe = np.where(sv > 0, sv, 1.0)
                    Ul, Vl = Vu / safe, Uu * sv
            else:
                Ul, Vl = source.compress(c, d, a, b, eps, svd_cache)
            pair = (store(Uu, Vu, fmt), store(Ul, Vl, fmt))
            if same_blocks_per_level:
                shared = pair
            row.append(pair)
        blocks.append(row)
    return HodlrMatrix(tree, leaves, blocks, eps, plan, working)
