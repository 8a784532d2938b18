"""Stress: alternating fp32/fp64 calls and repeated calls on one handle."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from conftest import random_hodlr
from oracle.matvec import matvec_oracle
from paper_2407_21637_b200 import linops, FP32, FP64

H = random_hodlr(2048, 3, ["fp32", "fp32", "fp16"], [10, 8, 6], "fp32", seed=4)
op = linops.HodlrOperator(H, 0)
print("launches", op.launches_per_matvec, flush=True)
x = np.random.default_rng(3).standard_normal(H.n)
ref = {w.name: matvec_oracle(H, x, w.name) for w in (FP32, FP64)}
bad = 0
pattern = sys.argv[1] if len(sys.argv) > 1 else "alt"
for i in range(400):
    if pattern == "alt":
        w = FP64 if i % 2 else FP32
    elif pattern == "fp32":
        w = FP32
    else:
        w = FP64
    dt = torch.float64 if w is FP64 else torch.float32
    b = op.matvec(torch.from_numpy(x).cuda().to(dt), working=w).double().cpu().numpy()
    r = np.linalg.norm(b - ref[w.name]) / np.linalg.norm(ref[w.name])
    tol = 1e-12 if w is FP64 else 1e-5
    if r > tol:
        bad += 1
        if bad < 10:
            d = np.abs(b - ref[w.name]); idx = np.argsort(d)[-5:]
            print(pattern, "iter", i, w.name, "rel", r, "worst rows", idx, d[idx], flush=True)
print(pattern, "bad", bad, "of 400", flush=True)
