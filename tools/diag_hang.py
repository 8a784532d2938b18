"""Locate a hang: build a workload, run one matvec, dump Python stacks after a delay."""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(float(sys.argv[2]) if len(sys.argv) > 2 else 150, exit=True)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_21637_b200 import linops  # noqa: E402

t0 = time.time()
H, x, desc, Kx, normA = bench.build_workload(sys.argv[1])
print("built", desc, f"{time.time() - t0:.1f}s", [f.name for f in H.plan.chosen],
      [H.blocks[k][0][0].rank for k in range(H.depth)], flush=True)
op = linops.HodlrOperator(H, 0)
print("packed; launches/matvec", op.launches_per_matvec, flush=True)
dt = torch.float64 if H.working_format.name == "fp64" else torch.float32
b = op.matvec(torch.from_numpy(x).cuda().to(dt))
torch.cuda.synchronize()
print("matvec ok", f"{time.time() - t0:.1f}s", flush=True)
from oracle.matvec import matvec_oracle  # noqa: E402

bo = matvec_oracle(H, x)
print("oracle ok", f"{time.time() - t0:.1f}s", float(abs(b.double().cpu().numpy() - bo).max()), flush=True)
