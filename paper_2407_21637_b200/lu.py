"""HODLR LU factorisation and triangular solves (Algorithm 4, HODLR_LU).

The other kernel the paper analyses (Cor. 3.8
PAPER.md:1132-1140), spec'd as ``lu / solve_lower / solve_upper_right /
schur_update / reconstruct_lu``; the
reference package ships only its building blocks (``factor_product``,
``recompress_sum``, lowrank.py:122-157).  The recursion is the paper's:

    leaf:      dense LU without pivoting (a pivot below ``pivot_tol`` raises,
               naming the leaf);
    node:      (L11, U11) = lu(H11)
               U12 = solve_lower(L11, H12)          -- thin solve on U of H12, rank kept
               L21 = solve_upper_right(H21, U11)    -- thin solve on V of H21, rank kept
               H22 <- H22 - L21 U12                 -- schur_update: the low-rank product
                                                       restricted to every block of H22,
                                                       off-diagonal blocks recompressed to
                                                       eps (QR + small SVD), leaves dense
               (L22, U22) = lu(H22)

Everything runs on the GPU in the working precision (fp64 or fp32 tensors;
stored factors are widened on access, computed factors stay in the working
format): cuBLAS products, cuSOLVER QR / SVD / triangular solves
through torch.  The factorisation is sequential by nature;
this module is the "next" row of the scope table, not the matvec hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .construct import truncation_rank
from .formats import FP64, format_code

__all__ = ["HodlrLuFactors", "SingularPivotError", "lu", "solve_lower", "solve_upper_right", "solve_upper",
           "schur_update", "reconstruct_lu", "lu_solve", "lu_backward_error", "lu_bound", "to_nodes"]


class SingularPivotError(ArithmeticError):
    """A leaf pivot fell below the pivot tolerance."""


def _torch():
    import torch

    return torch


def _device(device):
    torch = _torch()
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("HODLR LU runs on the GPU: no CUDA device (pass device='cpu' explicitly to "
                               "run the recursion on the host, e.g. in logic tests)")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _dtype(working):
    torch = _torch()
    code = format_code(working)
    if code == 4:
        return torch.float64
    if code == 3:
        return torch.float32
    raise NotImplementedError("HODLR LU: working precision must be fp64 or fp32")


# ---------------------------------------------------------------- node tree
class Node:
    """A HODLR (sub)matrix on the device: a dense leaf, or two children plus the
    two off-diagonal low-rank blocks ``upper = (U, V)`` (rows first, columns
    second child) and ``lower = (U, V)`` (rows second, columns first child).
    Triangular factors use the same type with one block absent (None)."""

    __slots__ = ("a", "b", "dense", "c1", "c2", "upper", "lower", "leaf_index")

    def __init__(self, a, b, dense=None, c1=None, c2=None, upper=None, lower=None, leaf_index=-1):
        self.a, self.b, self.dense, self.c1, self.c2 = a, b, dense, c1, c2
        self.upper, self.lower, self.leaf_index = upper, lower, leaf_index

    n = property(lambda self: self.b - self.a)
    is_leaf = property(lambda self: self.dense is not None)


def to_nodes(H, working=None, device=None) -> Node:
    """The recursive device tree of a ``HodlrMatrix`` (reference object or the
    flat mirror), factors widened to the working dtype."""
    torch = _torch()
    dev = _device(device)
    dt = _dtype(working if working is not None else H.working_format)
    depth = H.depth
    ranges = H.tree.ranges
    leaves = {i: D for i, _, D in H.leaves()}
    pairs = {(k, i): (up, lo) for k, i, _, _, up, lo in H.offdiag_blocks()}

    def t(a):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

    def build(k, j):
        a, b = ranges[k][j]
        if k == depth:
            return Node(a, b, dense=t(leaves[j]), leaf_index=j)
        up, lo = pairs[(k + 1, j)]
        return Node(a, b, c1=build(k + 1, 2 * j), c2=build(k + 1, 2 * j + 1),
                    upper=(t(up.U), t(up.V)), lower=(t(lo.U), t(lo.V)))

    return build(0, 0)


def _dense(node: Node):
    torch = _torch()
    if node.is_leaf:
        return node.dense.clone()
    m1 = node.c1.n
    ref = node.c1
    while not ref.is_leaf:
        ref = ref.c1
    out = torch.zeros((node.n, node.n), dtype=ref.dense.dtype, device=ref.dense.device)
    out[:m1, :m1] = _dense(node.c1)
    out[m1:, m1:] = _dense(node.c2)
    if node.upper is not None:
        out[:m1, m1:] = node.upper[0] @ node.upper[1].T
    if node.lower is not None:
        out[m1:, :m1] = node.lower[0] @ node.lower[1].T
    return out


# ---------------------------------------------------------------- low-rank algebra
def _recompress_sum(a, b, eps):
    """a + b (each (U, V)) recompressed to relative tolerance eps: thin QR of the
    stacked factors, SVD of the small core (lowrank.py:122-138)."""
    torch = _torch()
    rows, cols = a[0].shape[0], a[1].shape[0]
    joint = a[0].shape[1] + b[0].shape[1]
    if joint == 0:
        return a[0].new_zeros((rows, 0)), a[1].new_zeros((cols, 0))
    Qu, Ru = torch.linalg.qr(torch.cat([a[0], b[0]], dim=1))
    Qv, Rv = torch.linalg.qr(torch.cat([a[1], b[1]], dim=1))
    X, s, Yt = torch.linalg.svd(Ru @ Rv.T, full_matrices=False)
    s_np = s.double().cpu().numpy()
    # noise floor: a sum that cancelled down to rounding level (relative to the
    # summands) is rank 0 -- the relative rule would otherwise keep its noise
    floor = max(rows, cols) * float(torch.finfo(s.dtype).eps) * float(torch.linalg.norm(Ru)) * float(torch.linalg.norm(Rv))
    r = 0 if s_np.size == 0 or s_np[0] <= floor else truncation_rank(s_np, eps, max(rows, cols))
    return Qu @ X[:, :r], Qv @ (Yt[:r].T * s[:r])


def _factor_product(a, b):
    """(U_a V_a^T)(U_b V_b^T) as a factor of rank min(r_a, r_b) (lowrank.py:141-157)."""
    ra, rb = a[0].shape[1], b[0].shape[1]
    if min(ra, rb) == 0:
        return a[0].new_zeros((a[0].shape[0], 0)), b[1].new_zeros((b[1].shape[0], 0))
    core = a[1].T @ b[0]
    if ra <= rb:
        return a[0], b[1] @ core.T
    return a[0] @ core, b[1]


# ---------------------------------------------------------------- triangular solves
def _solve_lower_dense(Lt: Node, B):
    """L W = B for a HODLR unit-lower-triangular L and a dense thin B."""
    torch = _torch()
    if B.shape[1] == 0:
        return B
    if Lt.is_leaf:
        return torch.linalg.solve_triangular(Lt.dense, B, upper=False, unitriangular=True)
    m1 = Lt.c1.n
    W1 = _solve_lower_dense(Lt.c1, B[:m1])
    W2 = _solve_lower_dense(Lt.c2, B[m1:] - Lt.lower[0] @ (Lt.lower[1].T @ W1))
    return torch.cat([W1, W2], dim=0)


def _solve_upper_t_dense(Ut: Node, B):
    """U^T W = B for a HODLR upper-triangular U (so U^T is lower triangular)."""
    torch = _torch()
    if B.shape[1] == 0:
        return B
    if Ut.is_leaf:
        return torch.linalg.solve_triangular(Ut.dense.T, B, upper=False)
    m1 = Ut.c1.n
    W1 = _solve_upper_t_dense(Ut.c1, B[:m1])
    W2 = _solve_upper_t_dense(Ut.c2, B[m1:] - Ut.upper[1] @ (Ut.upper[0].T @ W1))
    return torch.cat([W1, W2], dim=0)


def _solve_upper_dense(Ut: Node, B):
    """U W = B (back substitution through the HODLR structure)."""
    torch = _torch()
    if B.shape[1] == 0:
        return B
    if Ut.is_leaf:
        return torch.linalg.solve_triangular(Ut.dense, B, upper=True)
    m1 = Ut.c1.n
    W2 = _solve_upper_dense(Ut.c2, B[m1:])
    W1 = _solve_upper_dense(Ut.c1, B[:m1] - Ut.upper[0] @ (Ut.upper[1].T @ W2))
    return torch.cat([W1, W2], dim=0)


def _is_factor(B):
    return isinstance(B, tuple) and len(B) == 2


def solve_lower(L: Node, B):
    """L X = B.  B low-rank ``(U, V)``: only L W = U is solved and ``(W, V)``
    returned, rank preserved; B dense: forward substitution through the tree
    (SPEC.md:352-360)."""
    rows = B[0].shape[0] if _is_factor(B) else B.shape[0]
    if rows != L.n:
        raise ValueError(f"shape mismatch: L is {L.n} x {L.n}, right-hand side has {rows} rows")
    if _is_factor(B):
        return _solve_lower_dense(L, B[0]), B[1]
    return _solve_lower_dense(L, B)


def solve_upper_right(B, U: Node):
    """X U = B.  B low-rank ``(U_B, V_B)``: U^T W = V_B is solved and
    ``(U_B, W)`` returned, rank preserved; B dense: X = (U^{-T} B^T)^T
    (SPEC.md:361-369)."""
    cols = B[1].shape[0] if _is_factor(B) else B.shape[1]
    if cols != U.n:
        raise ValueError(f"shape mismatch: U is {U.n} x {U.n}, right-hand side has {cols} columns")
    if _is_factor(B):
        return B[0], _solve_upper_t_dense(U, B[1])
    return _solve_upper_t_dense(U, B.T.contiguous()).T


def solve_upper(U: Node, B):
    """U X = B for a dense B (the back-substitution half of a linear solve)."""
    if B.shape[0] != U.n:
        raise ValueError(f"shape mismatch: U is {U.n} x {U.n}, right-hand side has {B.shape[0]} rows")
    return _solve_upper_dense(U, B)


# ---------------------------------------------------------------- Schur update
def schur_update(H22: Node, L21, U12, eps: float) -> Node:
    """H22 - L21 U12 as a HODLR node: Z = factor_product(L21, U12) restricted to
    every block of H22 -- off-diagonal blocks by recompress_sum to eps, leaves by
    dense subtraction."""
    if L21[0].shape[0] != H22.n or U12[1].shape[0] != H22.n or L21[1].shape[0] != U12[0].shape[0]:
        raise ValueError("schur_update: shapes do not conform")
    Zu, Zv = _factor_product(L21, U12)
    return _subtract_lowrank(H22, Zu, Zv, eps)


def _subtract_lowrank(node: Node, Zu, Zv, eps):
    if Zu.shape[1] == 0:
        return node
    if node.is_leaf:
        return Node(node.a, node.b, dense=node.dense - Zu @ Zv.T, leaf_index=node.leaf_index)
    m1 = node.c1.n
    upper = _recompress_sum(node.upper, (Zu[:m1], -Zv[m1:]), eps)
    lower = _recompress_sum(node.lower, (Zu[m1:], -Zv[:m1]), eps)
    return Node(node.a, node.b, c1=_subtract_lowrank(node.c1, Zu[:m1], Zv[:m1], eps),
                c2=_subtract_lowrank(node.c2, Zu[m1:], Zv[m1:], eps), upper=upper, lower=lower)


# ---------------------------------------------------------------- factorisation
@dataclass
class HodlrLuFactors:
    """L: HODLR unit-lower-triangular tree (``lower`` blocks only), U: HODLR
    upper-triangular tree (``upper`` blocks only); both in the working format
    (SPEC.md:326-331)."""

    L: Node
    U: Node
    tree: object
    working_format: object
    eps: float

    n = property(lambda self: self.L.n)


def _leaf_lu(D, leaf_index, pivot_tol):
    """Dense LU without pivoting (Doolittle: unit diagonal in L)."""
    torch = _torch()
    m = D.shape[0]
    tol = pivot_tol if pivot_tol is not None else m * 2.0 ** -53 * float(torch.linalg.norm(D))
    if D.is_cuda:
        LU = torch.linalg.lu_factor_ex(D, pivot=False).LU  # (no raise on a zero pivot: checked below)
    else:
        LU = D.clone()
        for j in range(m - 1):
            if abs(float(LU[j, j])) <= tol:
                break
            LU[j + 1:, j] /= LU[j, j]
            LU[j + 1:, j + 1:] -= torch.outer(LU[j + 1:, j], LU[j, j + 1:])
    piv = torch.diagonal(LU).abs()
    if not bool(torch.isfinite(LU).all()) or float(piv.min()) <= tol:
        raise SingularPivotError(f"singular pivot encountered in leaf {leaf_index} "
                                 f"(|pivot| {float(piv.min()):.3e} <= tolerance {tol:.3e})")
    Lm = torch.tril(LU, -1) + torch.eye(m, dtype=D.dtype, device=D.device)
    return Lm, torch.triu(LU)


def _lu_node(node: Node, eps, pivot_tol):
    if node.is_leaf:
        Lm, Um = _leaf_lu(node.dense, node.leaf_index, pivot_tol)
        return (Node(node.a, node.b, dense=Lm, leaf_index=node.leaf_index),
                Node(node.a, node.b, dense=Um, leaf_index=node.leaf_index))
    L11, U11 = _lu_node(node.c1, eps, pivot_tol)
    U12 = solve_lower(L11, node.upper)
    L21 = solve_upper_right(node.lower, U11)
    S = schur_update(node.c2, L21, U12, eps)
    L22, U22 = _lu_node(S, eps, pivot_tol)
    return (Node(node.a, node.b, c1=L11, c2=L22, lower=L21),
            Node(node.a, node.b, c1=U11, c2=U22, upper=U12))


def lu(H, eps: float | None = None, working=None, pivot_tol: float | None = None, device=None) -> HodlrLuFactors:
    """Algorithm 4 on ``H`` (a ``HodlrMatrix`` or a device ``Node``): Schur
    truncation tolerance ``eps`` (default ``H.eps``), all arithmetic in
    ``working`` (default ``H.working_format``)."""
    if isinstance(H, Node):
        root, tree, wf = H, None, (working if working is not None else FP64)
    else:
        wf = working if working is not None else H.working_format
        root, tree = to_nodes(H, wf, device), H.tree
        eps = H.eps if eps is None else eps
    if eps is None or not 0.0 <= eps < 1.0:
        raise ValueError(f"tolerance {eps} outside [0, 1)")
    _dtype(wf)
    Lt, Ut = _lu_node(root, float(eps), pivot_tol)
    return HodlrLuFactors(Lt, Ut, tree, wf, float(eps))


def reconstruct_lu(F: HodlrLuFactors):
    """(dense L, dense U) in binary64 with exact triangular structure."""
    torch = _torch()
    Ld = torch.tril(_dense(F.L).double())
    Ld.fill_diagonal_(1.0)
    return Ld.cpu().numpy(), torch.triu(_dense(F.U).double()).cpu().numpy()


def lu_solve(F: HodlrLuFactors, b):
    """x with (L U) x = b: forward then back substitution through the HODLR
    triangular factors.  b: numpy (n,) / (n, s) or a device tensor."""
    torch = _torch()
    ref = F.L
    while not ref.is_leaf:
        ref = ref.c1
    host = not isinstance(b, torch.Tensor)
    B = torch.as_tensor(np.asarray(b), dtype=ref.dense.dtype, device=ref.dense.device) if host else b.to(ref.dense.dtype)
    vec = B.dim() == 1
    B2 = B.reshape(-1, 1) if vec else B
    if B2.shape[0] != F.n:
        raise ValueError(f"length mismatch: b has {B2.shape[0]} rows, factors are {F.n} x {F.n}")
    X = solve_upper(F.U, solve_lower(F.L, B2))
    X = X[:, 0] if vec else X
    return X.double().cpu().numpy() if host else X


# ---------------------------------------------------------------- metrics
def lu_backward_error(A, F: HodlrLuFactors) -> float:
    """||L U - A||_F / ||A||_F with the densified factors (§4.3)."""
    A = np.asarray(A, dtype=np.float64)
    na = float(np.linalg.norm(A))
    if na == 0.0:
        raise ValueError("zero matrix")
    Ld, Ud = reconstruct_lu(F)
    return float(np.linalg.norm(Ld @ Ud - A) / na)


def lu_bound(ell: int, eps: float, normA: float, normL: float, normU: float) -> float:
    """Cor. 3.8 as a relative bound: (2 (2^l - 1) eps ||A|| + 11 (2^l - 1) eps ||L|| ||U||) / ||A||."""
    if normA == 0.0:
        raise ValueError("zero matrix")
    c = 2.0 ** ell - 1.0
    return (2.0 * c * eps * normA + 11.0 * c * eps * normL * normU) / normA


def hypothesis_holds(working, eps: float, n: int) -> bool:
    """u <~ eps / n, the hypothesis under which Cor. 3.8 is claimed."""
    return working.unit_roundoff <= eps / n if eps > 0 else False

