"""Build a config (timed) and time the matvec on it: python tools/time_configs.py 3|4 [n depth s]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2407_21637_b200 import linops, problems, storage_bits

cfg = sys.argv[1]
kw = {}
if len(sys.argv) > 2:
    kw = dict(n=int(sys.argv[2]), depth=int(sys.argv[3]), s=int(sys.argv[4]))
t0 = time.perf_counter()
H, X, src = (problems.cfg3 if cfg == "3" else problems.cfg4)(**kw)
t1 = time.perf_counter()
print(f"cfg{cfg} {kw} build {t1 - t0:.1f}s formats {[f.name for f in H.plan.chosen]} "
      f"ranks {[max(u.rank, l.rank) for u, l in (H.blocks[k][0] for k in range(H.depth))]} "
      f"storage {storage_bits(H) / 8e6:.1f} MB", flush=True)
op = linops.HodlrOperator(H)
dt = torch.float64 if H.working_format.name == "fp64" else torch.float32
Xd = torch.from_numpy(X).cuda().to(dt)
B = torch.empty_like(Xd)
for _ in range(3):
    op.matvec(Xd, out=B)
torch.cuda.synchronize()
flush = torch.ones(64 << 20, device="cuda")
ev = []
for _ in range(20):
    flush.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    op.matvec(Xd, out=B)
    b.record()
    ev.append((a, b))
torch.cuda.synchronize()
us = np.mean([a.elapsed_time(b) for a, b in ev]) * 1e3
nbytes = storage_bits(H) / 8 + 2 * X.size * (8 if dt == torch.float64 else 4)
print(f"matvec s={X.shape[1]}: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s  launches {op.launches_per_matvec}", flush=True)
