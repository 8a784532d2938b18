"""Per-rank device time of the sharded matvec on ONE GPU:
rank 0's handle of a P-way shard runs shard_begin / shard_local / shard_end
with a zero-filled receive buffer (no other rank exists; the all-gather itself
is not timed).  python tools/shard_time.py 4|2|s4 [P ...]   (s4: synthetic matrix of cfg4's shape)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2407_21637_b200 import linops, problems, storage_bits

cfg = sys.argv[1]
Ps = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
if cfg == "s4":
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from synth_time import SHAPES, synthetic

    n_, d_, f_, r_, w_, s_ = SHAPES["4"]
    H = synthetic(n_, d_, f_, r_, w_)
    X = np.random.default_rng(1).standard_normal((n_, s_))
else:
    H, X, src = (problems.cfg4() if cfg == "4" else problems.cfg3() if cfg == "3" else problems.cfg2())
X = np.asarray(X).reshape(H.n, -1)
s = X.shape[1]
dt = torch.float64 if H.working_format.name == "fp64" else torch.float32
wb = 8 if dt == torch.float64 else 4
flush = torch.ones(64 << 20, device="cuda")
for P in Ps:
    op = linops.HodlrOperator(H, rank=0, nranks=P) if P > 1 else linops.HodlrOperator(H)
    nl = op.n_local
    xl = torch.from_numpy(np.ascontiguousarray(X[:nl])).cuda().to(dt)
    bl = torch.empty_like(xl)
    if P > 1:
        cnt = op.exchange_count(s)
        send = torch.zeros(cnt, dtype=dt, device="cuda")
        recv = torch.zeros(cnt * P, dtype=dt, device="cuda")

    def step():
        if P == 1:
            op.matvec(xl, out=bl)
        else:
            op.shard_begin(xl, send)
            op.shard_local(xl, bl)
            op.shard_end(xl, recv, bl)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = []
    for _ in range(10):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    us = float(np.mean([a.elapsed_time(b) for a, b in ev])) * 1e3
    byts = op.matrix_bytes + 2 * nl * s * wb
    print(f"P={P} rank0 n_local={nl} path={op.path(s)} {us:.1f} us/matvec  {byts / us / 1e3:.0f} GB/s  "
          f"exchange {op.exchange_count(s) * wb if P > 1 else 0} B", flush=True)
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as pr:
        for _ in range(5):
            flush.sum()
            step()
        torch.cuda.synchronize()
    tot = {}
    for e in pr.events():
        if e.device_type.name == "CUDA" and "reduce_kernel<512" not in e.name:
            import re
            mm = re.search(r"(k_\w+)", e.name)
            nm = mm.group(1) if mm else e.name[:40]
            t, c = tot.get(nm, (0.0, 0))
            tot[nm] = (t + e.device_time, c + 1)
    for nm, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        print(f"    {t / c:9.1f} us x{c // 5}  {nm}", flush=True)
    del op
