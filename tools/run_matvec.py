"""Run the B200 matvec on a BASELINE workload (profiling / variant-timing target).

  python tools/run_matvec.py --config 2 [--iters 10] [--time] [--cache path.npz]

--cache saves the built matrix on first use and reloads it afterwards, so ncu
never sees the builder's cuSOLVER kernels.  --time prints the mean device time
of one matvec (L2 flushed before each, CUDA events on the launching stream).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--cache", default=None)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2407_21637_b200 import linops, model

    if args.cache and os.path.exists(args.cache):
        H = model.load_hodlr(args.cache)
        x = np.random.default_rng(2).standard_normal(H.n)
        desc = f"cached {args.cache}"
    else:
        import bench

        H, x, desc, _, _ = bench.build_workload(args.config)
        if args.cache:
            model.save_hodlr(H, args.cache)
    op = linops.HodlrOperator(H, 0)
    dt = torch.float64 if H.working_format.name == "fp64" else torch.float32
    xd = torch.from_numpy(x).cuda().to(dt)
    bd = torch.empty_like(xd)
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    times = []
    st = torch.cuda.current_stream()
    for i in range(args.iters):
        flush.sum()  # read-only L2 flush: evicts the matrix, leaves no dirty lines
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        op.matvec(xd, out=bd.view(-1, 1))
        e1.record(st)
        times.append((e0, e1))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in times[3:]] if len(times) > 3 else [0.0]
    if args.time:
        print(f"TIME {os.environ.get('VARIANT', '')} mean_us {1000 * sum(ms) / len(ms):.2f} min_us {1000 * min(ms):.2f}")
    print("ok", desc, "launches/matvec", op.launches_per_matvec)


if __name__ == "__main__":
    main()
