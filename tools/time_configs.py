"""Build a config (timed) and time the matvec on it:
    python tools/time_configs.py 3|4|2|5:1e-6 [n depth s] [--prof]
--prof: per-kernel device times from CUPTI (torch.profiler), L2 flushed between calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2407_21637_b200 import linops, problems, storage_bits

args = [a for a in sys.argv[1:] if not a.startswith("--")]
prof = "--prof" in sys.argv
cfg = args[0]
kw = {}
if len(args) > 1:
    kw = dict(n=int(args[1]), depth=int(args[2]), s=int(args[3]))
t0 = time.perf_counter()
if cfg == "3":
    H, X, src = problems.cfg3(**kw)
elif cfg == "4":
    H, X, src = problems.cfg4(**kw)
elif cfg == "2":
    H, X, src = problems.cfg2()
elif cfg.startswith("5:"):
    H, X, src = problems.cfg5(float(cfg[2:]))
X = X.reshape(H.n, -1)
t1 = time.perf_counter()
print(f"cfg{cfg} {kw} build {t1 - t0:.1f}s formats {[f.name for f in H.plan.chosen]} "
      f"ranks {[max(u.rank, l.rank) for u, l in (H.blocks[k][0] for k in range(H.depth))]} "
      f"storage {storage_bits(H) / 8e6:.1f} MB", flush=True)
op = linops.HodlrOperator(H)
dt = torch.float64 if H.working_format.name == "fp64" else torch.float32
Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda().to(dt)
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
s = X.shape[1]
print(f"matvec s={s}: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s  path {op.path(s)}", flush=True)
if prof:
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as pr:
        for _ in range(10):
            flush.sum()
            op.matvec(Xd, out=B)
        torch.cuda.synchronize()
    tot = {}
    for e in pr.events():
        if e.device_type.name == "CUDA":
            nm = e.name[:90]
            t, c = tot.get(nm, (0.0, 0))
            tot[nm] = (t + e.device_time, c + 1)
    for nm, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        print(f"  {t / c:10.1f} us x{c:3d}  {nm}")
