"""Event-timing overhead check: a 1-element kernel vs the fused matvec, both
timed like bench.py (L2 flush, then events around the call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2407_21637_b200 import linops, model

H = model.load_hodlr(sys.argv[1])
x = np.random.default_rng(2).standard_normal(H.n)
op = linops.HodlrOperator(H, 0)
xd = torch.from_numpy(x).cuda()
bd = torch.empty_like(xd)
tiny = torch.zeros(1, device="cuda")
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()


def timeit(fn, n=200, do_flush=True):
    ev = []
    for i in range(n):
        if do_flush:
            flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        ev.append((a, b))
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1000 for a, b in ev[5:]]
    return np.mean(t), np.min(t)


for name, fn in [("tiny add", lambda: tiny.add_(1.0)), ("matvec", lambda: op.matvec(xd, out=bd.view(-1, 1)))]:
    for fl in (True, False):
        m, mn = timeit(fn, do_flush=fl)
        print(f"{name:10s} flush={fl!s:5s} mean {m:7.2f} us  min {mn:7.2f} us")
# back-to-back: 50 matvecs between two events
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(50):
    op.matvec(xd, out=bd.view(-1, 1))
b.record(st)
torch.cuda.synchronize()
print(f"back-to-back (L2 warm) per matvec {a.elapsed_time(b) * 1000 / 50:.2f} us")

# event floor and CUDA-graph replays
print("events only      mean %7.2f us  min %7.2f us" % timeit(lambda: None))
for name, fn in [("tiny add", lambda: tiny.add_(1.0)), ("matvec", lambda: op.matvec(xd, out=bd.view(-1, 1)))]:
    s2 = torch.cuda.Stream()
    s2.wait_stream(st)
    with torch.cuda.stream(s2):
        fn()
    st.wait_stream(s2)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    print(f"graph {name:10s} mean %7.2f us  min %7.2f us" % timeit(lambda: g.replay()))
