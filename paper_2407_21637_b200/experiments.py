"""The paper's matvec experiment on the GPU path (SPEC.md:600-607 ``cmd_matvec``,
PAPER.md:1264-1279, Fig. 4): for each kernel matrix mat-1..mat-4 (n = 2000,
l = 8), each tolerance eps and each working precision in {fp64, fp32, bf16},
build the adaptive-precision HODLR matrix (Alg. 2), multiply ``trials`` random
vectors with entries uniform on (-1, 1) (Alg. 3, on the B200 through the C
ABI) and report the mean backward error ||b_hat - K x|| / (||K||_F ||x||)
next to the Theorem 3.5 bound and the hypothesis flag u <= eps / n
(a cell with the flag false is "hypothesis unmet", never a
violation).

Test matrices (Eq. (4.1)): point sets s1 = n equispaced
points of [0, 1], s2 = the first n points (row-major) of the ceil(sqrt n)^2
uniform grid on [-1, 1]^2; kernels (i) 1/(x - y) (diagonal 1), (ii)
log ||x_i - x_j|| (0 for coincident points), (iii) exp(-||x_i - x_j||^2 / (2 h^2)).
mat-1 = (i) on s1, mat-2 = (ii) on s2, mat-3 / mat-4 = (iii) on s2 with
h = 1 / h = 20.

fp64 and fp32 working run the throughput kernels; bf16 (and fp16 / q52) run
the strict-order kernels, bit-identical to the reference's
``Arithmetic(working)``.  The trial vectors come from numpy's Philox
counter-based generator (seed recorded in the CSV header), so every row is
reproducible.

    python -m paper_2407_21637_b200.experiments matvec --out fig4.csv
"""

from __future__ import annotations

import argparse
import math
import sys

import numpy as np

from . import metrics
from .construct import DenseSource, build_adaptive
from .formats import BF16, FP16, FP32, FP64, Q52, parse_format
from .model import build_tree, storage_bits

ALL_FORMATS = (Q52, BF16, FP16, FP32, FP64)
CSV_SCHEMA = 1
MATRICES = ("mat-1", "mat-2", "mat-3", "mat-4")
DEFAULT_EPS = tuple(10.0 ** -k for k in range(1, 11))
DEFAULT_WORKINGS = (FP64, FP32, BF16)


# ---------------------------------------------------------------- problems
def grid_1d(n: int) -> np.ndarray:
    """n equispaced points covering [0, 1] inclusive."""
    if n < 1:
        raise ValueError("n must be positive")
    return np.linspace(0.0, 1.0, n).reshape(n, 1) if n > 1 else np.zeros((1, 1))


def grid_2d(n: int) -> np.ndarray:
    """First n points, row-major, of the m x m grid on [-1, 1]^2, m = ceil(sqrt n)
    (SPEC.md:440-446)."""
    if n < 1:
        raise ValueError("n must be positive")
    m = math.isqrt(n - 1) + 1
    ax = np.linspace(-1.0, 1.0, m) if m > 1 else np.array([-1.0])
    P = np.stack(np.meshgrid(ax, ax, indexing="ij"), axis=-1).reshape(-1, 2)
    return P[:n]


def kernel_matrix(kind: str, pts: np.ndarray, h: float | None = None) -> np.ndarray:
    """Eq. (4.1).  kind: "i" | "ii" | "iii"."""
    pts = np.asarray(pts, dtype=np.float64)
    if kind == "i":
        if pts.shape[1] != 1:
            raise ValueError("kernel (i) needs a 1-D point set")
        d = pts[:, 0][:, None] - pts[:, 0][None, :]
        with np.errstate(divide="ignore"):
            K = np.where(d != 0.0, 1.0 / d, 1.0)
        return K
    D2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
    if kind == "ii":
        with np.errstate(divide="ignore"):
            return np.where(D2 > 0.0, 0.5 * np.log(np.where(D2 > 0.0, D2, 1.0)), 0.0)
    if kind == "iii":
        if h is None or h <= 0:
            raise ValueError("kernel (iii) needs a bandwidth h > 0")
        return np.exp(-D2 / (2.0 * h * h))
    raise ValueError(f"unknown kernel kind {kind!r}")


def paper_matrix(name: str, n: int = 2000) -> np.ndarray:
    if name == "mat-1":
        return kernel_matrix("i", grid_1d(n))
    if name == "mat-2":
        return kernel_matrix("ii", grid_2d(n))
    if name == "mat-3":
        return kernel_matrix("iii", grid_2d(n), 1.0)
    if name == "mat-4":
        return kernel_matrix("iii", grid_2d(n), 20.0)
    raise ValueError(f"unknown matrix {name!r} (expected one of {MATRICES})")


# ---------------------------------------------------------------- the sweep
def trial_vectors(n: int, trials: int, seed: int) -> np.ndarray:
    """n x trials, entries uniform on (-1, 1), Philox counter-based stream."""
    return np.random.Generator(np.random.Philox(seed)).uniform(-1.0, 1.0, size=(n, trials))


def sweep_matvec(matrices=MATRICES, n: int = 2000, depth: int = 8, eps_grid=DEFAULT_EPS,
                 workings=DEFAULT_WORKINGS, trials: int = 10, seed: int = 20240731, device: int = 0,
                 log=None):
    """Rows of the Fig. 4 sweep: one dict per (matrix, eps, working) cell."""
    import torch

    from .linops import HodlrOperator

    rows = []
    tree = build_tree(n, depth)
    X = trial_vectors(n, trials, seed)
    for name in matrices:
        K = paper_matrix(name, n)
        src = DenseSource(K)
        norm_k = float(np.linalg.norm(K))
        KX = K @ X
        cache = {}
        for eps in eps_grid:
            for w in workings:
                H = build_adaptive(src, tree, eps, working=w, available=ALL_FORMATS, svd_cache=cache)
                op = HodlrOperator(H, device=device)
                Xd = torch.from_numpy(X).cuda(device)
                B = op.matvec(Xd, working=w).double().cpu().numpy()
                path, _ = op.path(trials, w)
                op.close()
                errs = [metrics.matvec_backward_error(KX[:, j], X[:, j], B[:, j], norm_k) for j in range(trials)]
                err = float(np.mean(errs))
                bound = metrics.matvec_bound(depth, eps)
                hyp = metrics.hypothesis_holds(w, eps, n)
                row = {
                    "matrix": name, "n": n, "depth": depth, "eps": eps, "working": w.name, "trials": trials,
                    "backward_error": err, "bound": bound, "hypothesis_met": hyp,
                    "satisfied": bool(err <= bound),
                    "status": ("ok" if err <= bound else ("hypothesis-unmet" if not hyp else "VIOLATED")),
                    "formats": "/".join(f.name for f in H.plan.chosen),
                    "fallback": bool(H.plan.any_fallback), "storage_bits": storage_bits(H), "kernel_path": path,
                }
                rows.append(row)
                if log:
                    log(f"{name} eps={eps:.0e} {w.name:5s} err={err:.3e} bound={bound:.3e} "
                        f"{row['status']} [{path}]")
    rows.sort(key=lambda r: (r["matrix"], -r["eps"], r["working"]))
    return rows


COLUMNS = ["matrix", "n", "depth", "eps", "working", "trials", "backward_error", "bound", "hypothesis_met",
           "satisfied", "status", "formats", "fallback", "storage_bits", "kernel_path"]


def write_csv(rows, fh, seed: int) -> None:
    fh.write(f"# hodlr-b200 matvec sweep, csv schema {CSV_SCHEMA}; vectors: numpy Philox(seed={seed}) "
             "uniform(-1,1); error = ||b_hat - K x|| / (||K||_F ||x||), mean over trials\n")
    fh.write(",".join(COLUMNS) + "\n")
    for r in rows:
        fh.write(",".join(f"{r[c]:.6e}" if isinstance(r[c], float) else str(r[c]) for c in COLUMNS) + "\n")


def sweep_lu(sizes=(256, 512), depths=(2, 8), eps_grid=(1e-2, 1e-4, 1e-6, 1e-8, 1e-10), workings=(FP64, FP32),
             seed: int = 20240731, device=None, log=None):
    """The LU experiment (SPEC.md:608-615 ``cmd_lu``, §4.3) on diagonally
    dominant random matrices: ||L U - A|| / ||A|| of the HODLR LU (Alg. 4, on
    the GPU) against the Cor. 3.8 bound with the measured ||L|| ||U||, the
    hypothesis flag, and "pivot-breakdown" cells reported, not raised."""
    from . import lu as hl

    rows = []
    for n in sizes:
        rng = np.random.Generator(np.random.Philox(seed + n))
        A = rng.standard_normal((n, n))
        A = A + np.diag(np.abs(A).sum(axis=1) + 1.0)
        src = DenseSource(A)
        for depth in depths:
            tree = build_tree(n, depth)
            cache = {}
            for eps in eps_grid:
                for w in workings:
                    H = build_adaptive(src, tree, eps, working=w, available=ALL_FORMATS, svd_cache=cache)
                    from .lu import _dense, to_nodes

                    Ah = _dense(to_nodes(H, FP64, device)).cpu().numpy()
                    row = {"matrix": f"dd-random:{n}", "n": n, "depth": depth, "eps": eps, "working": w.name}
                    try:
                        F = hl.lu(H, device=device)
                        Ld, Ud = hl.reconstruct_lu(F)
                        err = hl.lu_backward_error(Ah, F)
                        bound = hl.lu_bound(depth, eps, float(np.linalg.norm(Ah)), float(np.linalg.norm(Ld)),
                                            float(np.linalg.norm(Ud)))
                        hyp = hl.hypothesis_holds(w, eps, n)
                        row.update(backward_error=err, bound=bound, hypothesis_met=hyp, satisfied=bool(err <= bound),
                                   status="ok" if err <= bound else ("hypothesis-unmet" if not hyp else "VIOLATED"))
                    except hl.SingularPivotError:
                        row.update(backward_error=float("nan"), bound=float("nan"), hypothesis_met=False,
                                   satisfied=False, status="pivot-breakdown")
                    rows.append(row)
                    if log:
                        log(f"lu n={n} l={depth} eps={eps:.0e} {w.name}: err={row['backward_error']:.3e} "
                            f"bound={row['bound']:.3e} {row['status']}")
    return rows


LU_COLUMNS = ["matrix", "n", "depth", "eps", "working", "backward_error", "bound", "hypothesis_met", "satisfied", "status"]


def main(argv=None) -> int:
    """Exit codes: 0 success, 1 usage error, 3 a bound violated
    with the hypothesis met."""
    ap = argparse.ArgumentParser(prog="paper_2407_21637_b200.experiments")
    sub = ap.add_subparsers(dest="cmd", required=True)
    mv = sub.add_parser("matvec", help="Fig. 4 sweep (SPEC.md:600-607)")
    mv.add_argument("--source", action="append", help="mat-1 .. mat-4 (repeatable; default all four)")
    mv.add_argument("--n", type=int, default=2000)
    mv.add_argument("--depth", type=int, default=8)
    mv.add_argument("--eps", type=float, action="append", help="repeatable; default 1e-1 .. 1e-10")
    mv.add_argument("--working", action="append", help="fp64 | fp32 | bf16 | fp16 | q52 (repeatable)")
    mv.add_argument("--trials", type=int, default=10)
    mv.add_argument("--seed", type=int, default=20240731)
    mv.add_argument("--device", type=int, default=0)
    mv.add_argument("--out", default="-")
    lp = sub.add_parser("lu", help="LU sweep on diagonally dominant randoms (SPEC.md:608-615)")
    lp.add_argument("--seed", type=int, default=20240731)
    lp.add_argument("--out", default="-")
    try:
        a = ap.parse_args(argv)
        if a.cmd == "lu":
            rows = sweep_lu(seed=a.seed, log=lambda s: print(s, file=sys.stderr))
            fh = sys.stdout if a.out == "-" else open(a.out, "w")
            fh.write(f"# hodlr-b200 lu sweep, csv schema {CSV_SCHEMA}; matrices: Philox(seed={a.seed}+n) normal + "
                     "row-sum diagonal\n" + ",".join(LU_COLUMNS) + "\n")
            for r in rows:
                fh.write(",".join(f"{r[c]:.6e}" if isinstance(r[c], float) else str(r[c]) for c in LU_COLUMNS) + "\n")
            if fh is not sys.stdout:
                fh.close()
            return 3 if any(r["status"] == "VIOLATED" for r in rows) else 0
        if a.trials < 1:
            raise ValueError("trials must be >= 1")
        workings = tuple(parse_format(w) for w in a.working) if a.working else DEFAULT_WORKINGS
        mats = tuple(a.source) if a.source else MATRICES
        for m in mats:
            if m not in MATRICES:
                raise ValueError(f"unknown source {m!r}")
    except (ValueError, SystemExit) as exc:
        if isinstance(exc, SystemExit) and exc.code == 0:
            return 0
        print(f"usage error: {exc}", file=sys.stderr)
        return 1
    rows = sweep_matvec(mats, a.n, a.depth, tuple(a.eps) if a.eps else DEFAULT_EPS, workings, a.trials, a.seed,
                        a.device, log=lambda s: print(s, file=sys.stderr))
    fh = sys.stdout if a.out == "-" else open(a.out, "w")
    try:
        write_csv(rows, fh, a.seed)
    finally:
        if fh is not sys.stdout:
            fh.close()
    return 3 if any(r["status"] == "VIOLATED" for r in rows) else 0


if __name__ == "__main__":
    sys.exit(main())
