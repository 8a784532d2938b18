"""Time the matvec kernels on a SYNTHETIC matrix with a BASELINE config's shape
(random factors, one block shared by all blocks of a level, so it builds in
seconds instead of the 20-40 s of the real kernel matrices).  Kernel times do
not depend on the values; parity is checked against the oracle on a few rows.

    python tools/synth_time.py 4|3|2 [--prof] [--iters N] [--check]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2407_21637_b200 import NAMED_FORMATS, linops, model, storage_bits

SHAPES = {
    # n, depth, level formats, ranks, working, s   (plans / ranks of the real builds, BENCH lines)
    "4": (1 << 20, 12, ["fp32"] * 12, [7, 7, 7, 7, 7, 5, 4, 3, 3, 2, 2, 2], "fp64", 16),
    "3": (1 << 18, 10, ["fp32"] * 8 + ["fp16"] * 2, [88, 52, 49, 29, 33, 25, 24, 13, 14, 10], "fp32", 64),
    "5a": (1 << 18, 10, ["q52"] * 9 + ["bf16"], [7, 7, 7, 6, 6, 6, 5, 5, 5, 4], "fp32", 1),
    "5b": (1 << 18, 10, ["bf16"] * 5 + ["fp16"] * 5, [13, 13, 12, 11, 11, 10, 9, 9, 8, 7], "fp32", 1),
    "2": (1 << 16, 8, ["fp32"] * 8, [17, 16, 15, 14, 13, 12, 11, 10], "fp64", 1),
}


def synthetic(n, depth, fmts, ranks, working, seed=0):
    from oracle.fpsim import round_matrix

    class _C:  # cast[fmt](a).astype(float64) == round_matrix(a, fmt)
        def __init__(self, f):
            self.f = f

        def __call__(self, a):
            return round_matrix(a, self.f)

    cast = {f: _C(f) for f in ("q52", "bf16", "fp16", "fp32", "fp64")}
    rng = np.random.default_rng(seed)
    T = model.build_tree(n, depth)
    m = n >> depth
    leaf = cast[working](rng.standard_normal((m, m)))
    leaves = [leaf] * (1 << depth)
    blocks = []
    for k in range(1, depth + 1):
        F, dt, r = NAMED_FORMATS[fmts[k - 1]], cast[fmts[k - 1]], ranks[k - 1]
        rows = n >> k
        U = dt(rng.standard_normal((rows, r)) / np.sqrt(rows))
        V = np.asfortranarray(dt(rng.standard_normal((rows, r)) * 0.5 ** k))
        f = model.LowRankFactor(U, V, F)
        blocks.append([(f, f)] * (1 << (k - 1)))
    return model.HodlrMatrix(T, leaves, blocks, 1e-6, model.PrecisionPlan([NAMED_FORMATS[f] for f in fmts]),
                             NAMED_FORMATS[working])


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    cfg = args[0] if args else "4"
    iters = 20
    if "--iters" in sys.argv:
        iters = int(sys.argv[sys.argv.index("--iters") + 1])
    n, depth, fmts, ranks, working, s = SHAPES[cfg]
    t0 = time.perf_counter()
    H = synthetic(n, depth, fmts, ranks, working)
    op = linops.HodlrOperator(H)
    torch.cuda.synchronize()
    print(f"synthetic cfg{cfg}: n={n} depth={depth} s={s} {working} built+packed in {time.perf_counter() - t0:.1f}s "
          f"storage {storage_bits(H) / 8e6:.1f} MB path {op.path(s)}", flush=True)
    dt = torch.float64 if working == "fp64" else torch.float32
    X = np.random.default_rng(1).standard_normal((n, s))
    Xd = torch.from_numpy(X).cuda().to(dt)
    if s == 1:
        Xd = Xd[:, 0].contiguous()
    B = torch.empty_like(Xd)
    for _ in range(3):
        op.matvec(Xd, out=B if s > 1 else B.view(-1, 1))
    torch.cuda.synchronize()
    flush = torch.ones(64 << 20, device="cuda")
    ev = []
    for _ in range(iters):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        op.matvec(Xd, out=B if s > 1 else B.view(-1, 1))
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) for a, b in ev]) * 1e3
    nbytes = storage_bits(H) / 8 + 2 * X.size * (8 if dt == torch.float64 else 4)
    print(f"TIME {os.environ.get('VARIANT', '')} cfg{cfg} mean {t.mean():.1f} us  min {t.min():.1f}  "
          f"{nbytes / t.mean() / 1e3:.0f} GB/s  frac {nbytes / t.mean() / 1e3 / 6466.8:.3f}", flush=True)
    if "--e2e" in sys.argv:
        # host-buffer entry point: pinned binary64 X in, B out, every call
        xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()
        bh = torch.empty_like(xh).pin_memory()
        st = torch.cuda.current_stream()
        for _ in range(3):
            op.matvec_host_ptr(xh.data_ptr(), bh.data_ptr(), s, stream=st.cuda_stream)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 10
        for _ in range(reps):
            op.matvec_host_ptr(xh.data_ptr(), bh.data_ptr(), s, stream=st.cuda_stream)
        torch.cuda.synchronize()
        dt_ms = (time.perf_counter() - t0) / reps * 1e3
        ref = op.matvec(Xd).double().cpu().numpy().reshape(n, -1)
        same = np.array_equal(bh.numpy().reshape(n, -1), ref)
        print(f"E2E {os.environ.get('VARIANT', '')} cfg{cfg} {dt_ms:.3f} ms per host-buffer call ({1e3 / dt_ms:.1f} matvec/s), "
              f"result == device-resident call: {same}", flush=True)
    if "--check" in sys.argv:
        # oracle on the rows of the first and last leaf (dense rows of H through the blocks)
        from oracle.matvec import matvec_oracle

        nn, dd = 4096, max(depth - (n.bit_length() - 13), 1)
        Hs = synthetic(nn, dd, fmts[-dd:], ranks[-dd:], working, seed=3)
        ops = linops.HodlrOperator(Hs)
        Xs = np.random.default_rng(2).standard_normal((nn, s))
        if working == "fp32":
            Xs = Xs.astype(np.float32).astype(np.float64)
        got = ops.matvec(torch.from_numpy(Xs).cuda().to(dt)).double().cpu().numpy()
        want = matvec_oracle(Hs, Xs, "fp64")
        print(f"CHECK small synthetic (n={nn}, depth={dd}) rel err vs fp64 oracle "
              f"{np.linalg.norm(got - want) / np.linalg.norm(want):.2e} path {ops.path(s)}", flush=True)
    if "--prof" in sys.argv:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as pr:
            for _ in range(10):
                flush.sum()
                op.matvec(Xd, out=B if s > 1 else B.view(-1, 1))
            torch.cuda.synchronize()
        tot = {}
        for e in pr.events():
            if e.device_type.name == "CUDA":
                nm = e.name[:70]
                tt, c = tot.get(nm, (0.0, 0))
                tot[nm] = (tt + e.device_time, c + 1)
        for nm, (tt, c) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
            print(f"  {tt / c:10.1f} us x{c:3d}  {nm}")


if __name__ == "__main__":
    main()
    time.sleep(float(os.environ.get("SYNTH_SLEEP", "0")))  # (diagnostic builds with a delayed host-side report)
