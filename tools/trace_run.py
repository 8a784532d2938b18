"""Phase timeline of the fused kernel from an HODLR_TRACE build.

  tools/build_trace.sh && python tools/trace_run.py --config 2 --cache /tmp/cfg2.npz

Stamps (per CTA, ns of %globaltimer, relative to the earliest entry):
  0 entry  2 last A leaf issued  3 first BC item  4/5 first R wait start/end
  6 coefficients ready (producer sees every R piece)  7 queue exhausted
  8 last U piece issued  9 consumers done  10 exit; 11/12/13 A / BC / R counts.
"""
import argparse
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def summarize(path):
    raw = open(path, "rb").read()
    grid, w, num_a, num_r = np.frombuffer(raw[:16], dtype=np.int32)
    T = np.frombuffer(raw[16:], dtype=np.uint64).reshape(grid, w).astype(np.float64)
    t0 = T[:, 0].min()
    rel = lambda i: (T[:, i][T[:, i] > 0] - t0) / 1000.0  # us

    def line(name, i):
        v = rel(i)
        if len(v) == 0:
            print(f"  {name:28s} (none)")
            return
        print(f"  {name:28s} n={len(v):4d} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")

    print(f"grid {grid}  A leaves {num_a}  R pieces {num_r}")
    for name, i in [("entry", 0), ("epoch loaded", 21), ("tables ready", 22), ("first queue items", 23), ("first entry known", 30), ("first piece issued", 1), ("A piece 1 arrived", 24), ("A piece 2 arrived", 25),
                    ("A piece 3 arrived", 26), ("A piece 4 arrived", 27), ("last A piece issued", 2), ("first BC item", 3), ("R wait start", 4),
                    ("R wait end (all A done)", 5), ("coefficients ready", 6), ("queue exhausted", 7),
                    ("first U issued", 14), ("first U consumed", 15), ("last U issued", 8), ("consumers done", 9), ("exit", 10),
                    ("A publish: fence start", 16), ("A publish: fence end", 17), ("R stage issued", 20),
                    ("R publish: fence start", 18), ("R publish: fence end", 19)]:
        line(name, i)
    wait, tot = T[:, 28], T[:, 29]
    if tot.max() > 0:
        fr = wait / np.maximum(tot, 1)
        print(f"  consumer warp 0 waiting for data: {100 * fr.mean():.1f}% of its loop (min {100 * fr.min():.1f}%, "
              f"max {100 * fr.max():.1f}%), loop {tot.mean() / 1.965e3:.1f} us @1.965GHz")
    if T.shape[1] >= 44:
        names = {1: "A", 2: "D", 3: "U", 5: "R"}
        parts = []
        for i, nm in names.items():
            nb = T[:, 38 + i].sum()
            if nb:
                parts.append(f"{nm} {T[:, 32 + i].sum() / nb / 1.965e3:.3f} us x {nb / len(T):.1f}")
        print("  consumer warp 0 busy per piece: " + ", ".join(parts))
        na, nd = T[:, 39].sum(), T[:, 40].sum()
        sp = T[:, 44:48].sum(axis=0) / 1.965e3
        if na and nd:
            print(f"  A: compute {sp[0] / na:.3f} us + combine {sp[1] / na:.3f} us per piece;  "
                  f"D: compute {sp[2] / nd:.3f} us per piece + combine {sp[3] / (nd / 4):.3f} us per item")
    cnt = T[:, 11:14]
    print(f"  items per CTA: A {cnt[:, 0].mean():.2f} (max {cnt[:, 0].max():.0f})  BC {cnt[:, 1].mean():.2f} "
          f"(max {cnt[:, 1].max():.0f})  R {cnt[:, 2].sum():.0f} total")
    print(f"  kernel span {(T[:, 10].max() - t0) / 1000:.2f} us")
    # who ends last?  per-CTA rows sorted by exit time (first / last 8) and correlations
    us = lambda i: np.where(T[:, i] > 0, (T[:, i] - t0) / 1000.0, np.nan)
    ex = us(10)
    cols = [("A", cnt[:, 0]), ("BC", cnt[:, 1]), ("R", cnt[:, 2]), ("firstBC", us(3)), ("coefReady", us(6)),
            ("qExhaust", us(7)), ("firstU", us(14)), ("lastU", us(8)), ("consDone", us(9)), ("exit", ex)]
    order = np.argsort(ex)
    print("  per-CTA (sorted by exit):  cta " + " ".join(f"{n:>9s}" for n, _ in cols))
    for i in list(order[:8]) + [-1] + list(order[-8:]):
        if i < 0:
            print("    ...")
            continue
        print(f"    {i:4d} " + " ".join(f"{v[i]:9.2f}" for _, v in cols))
    for n, v in cols[:-1]:
        ok = ~np.isnan(v)
        if ok.sum() > 2 and np.std(v[ok]) > 0:
            print(f"  corr(exit, {n}) = {np.corrcoef(ex[ok], v[ok])[0, 1]:+.2f}")
    sm_lo, sm_hi = ex[: grid // 2], ex[grid // 2:]
    print(f"  exit by CTA index half: first {np.nanmean(sm_lo):.2f}  second {np.nanmean(sm_hi):.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--cache", default=None)
    ap.add_argument("--iters", type=int, default=6)
    args = ap.parse_args()
    tf = os.path.join(ROOT, "gpurun_out", f"trace_cfg{args.config.replace(':', '_')}.bin")
    os.makedirs(os.path.dirname(tf), exist_ok=True)
    env = dict(os.environ, HODLR_B200_LIB=os.path.join(ROOT, "tools", "libhodlr_b200_trace.so"),
               HODLR_B200_TRACE_FILE=tf)
    cmd = [sys.executable, os.path.join(ROOT, "tools", "run_matvec.py"), "--config", args.config,
           "--iters", str(args.iters)]
    if args.cache:
        cmd += ["--cache", args.cache]
    subprocess.check_call(cmd, env=env)
    summarize(tf)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1].endswith(".bin"):
        summarize(sys.argv[1])
    else:
        main()
