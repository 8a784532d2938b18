"""Run the B200 matvec on a BASELINE workload a few times (profiling target:
`ncu ... python tools/run_matvec.py --config 2`)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2407_21637_b200 import linops

    H, x, desc, _, _ = bench.build_workload(args.config)
    op = linops.HodlrOperator(H, 0)
    dt = torch.float64 if H.working_format.name == "fp64" else torch.float32
    xd = torch.from_numpy(x).cuda().to(dt)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for i in range(args.iters):
        flush.fill_(float(i))
        op.matvec(xd)
    torch.cuda.synchronize()
    print("ok", desc, "launches/matvec", op.launches_per_matvec)


if __name__ == "__main__":
    main()
