"""Where the e2e (host-buffer) matvec time goes on cfg2: full host call vs its parts.
Usage: python tools/e2e_breakdown.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2407_21637_b200 import linops

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
H, X, desc, _, _ = bench.build_workload(cfg)
n, s = X.shape
op = linops.HodlrOperator(H, 0)
st = torch.cuda.current_stream()
xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()
bh = torch.empty_like(xh).pin_memory()
xd = xh.cuda()
bd = torch.empty_like(xd)
K = 400


def timeit(name, fn):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(K):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"{name:40s} events {e0.elapsed_time(e1) / K * 1e3:8.1f} us   wall {(t1 - t0) / K * 1e6:8.1f} us", flush=True)


timeit("host call (hodlr_matvec_host)", lambda: op.matvec_host_ptr(xh.data_ptr(), bh.data_ptr(), s, stream=st.cuda_stream))


def copies():
    xd.copy_(xh, non_blocking=True)
    bh.copy_(bd, non_blocking=True)
    torch.cuda.current_stream().synchronize()


timeit("H2D + D2H + sync", copies)


def kern_sync():
    op.matvec(xd, out=bd)
    torch.cuda.current_stream().synchronize()


timeit("device matvec + sync", kern_sync)
timeit("device matvec (async)", lambda: op.matvec(xd, out=bd))


def h2d():
    xd.copy_(xh, non_blocking=True)


timeit("H2D only (async)", h2d)
timeit("D2H only (async)", lambda: bh.copy_(bd, non_blocking=True))
