"""Benchmark of the B200 HODLR matvec (BASELINE.json metric: HODLR matvecs/s and
effective HBM GB/s as a fraction of roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl reference]

* Workload at N=1: BASELINE config 2 (n=65536, depth 8, Toeplitz 1/(1+|i-j|),
  eps=1e-6, adaptive formats, fp64 working, one right-hand side), built by the
  package's restatement of Alg. 2 on the GPU from seeded inputs.
* ``value``: matvecs/s with x, b and the packed matrix resident in HBM; every
  timed step is bracketed by CUDA events on the launching stream and preceded
  by an (untimed) L2 flush (reading a 256 MiB buffer), so the matrix streams from HBM.
* ``e2e``: the same metric through the public host-buffer entry point
  (hodlr_matvec_host): pinned binary64 x copied in, matvec, b copied out, every
  step, timed by events around the whole call.
* ``roofline``: algorithmic bytes per matvec = storage_bits(H)/8 + n*s*(w_x+w_b)
  (hodlr.py:279-287) / the kernel's average event time, against
  the measured HBM copy bandwidth of MEASURED_PEAKS.json.
* ``cpu_baseline``: the CPU oracle (Alg. 3 restatement, numpy/OpenBLAS fp64) on
  the same H and x, all host threads, bounded sample.
* ``--impl reference``: the reference-side CPU implementation of the path (the
  oracle port -- the reference package has no matvec of its own), same line shape.
Multi-GPU (torchrun, N>1): the tree is sharded at level log2(N); one NCCL
all-gather of V^T x coefficient partials per matvec; time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded (multi-GPU) code path even at one rank")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def build_workload(cfg: str):
    """(H, X (n x s), description, K-times function, ||K||_F) for a BASELINE config."""
    from paper_2407_21637_b200 import problems

    if cfg == "2":
        H, x, src = problems.cfg2()
        desc = ("cfg2: n=65536 depth=8 leaf=256, A_ij=1/(1+|i-j|), eps=1e-6, adaptive over "
                "{q52,bf16,fp16,fp32,fp64}, fp64 working, 1 rhs")
        return H, x.reshape(-1, 1), desc, (lambda v: problems.toeplitz_times(v)), src.frob2_all() ** 0.5
    if cfg == "1":
        H, x, A = problems.cfg1()
        desc = ("cfg1: n=4096 depth=4 leaf=256, Gaussian sigma=0.05 + 1e-2 I, eps=1e-8, adaptive, "
                "fp64 working, 1 rhs")
        return H, x.reshape(-1, 1), desc, (lambda v: A @ v), float(np.linalg.norm(A))
    if cfg == "3":
        H, X, src = problems.cfg3()
        desc = ("cfg3: n=262144 depth=10 leaf=256, A_ij=exp(-|p_i-p_j|/0.2), 2-D uniform points, Morton "
                "order, eps=1e-4, adaptive, fp32 working, 64 rhs (tensor-core multi-RHS path)")
        return H, X, desc, (lambda v: problems.kernel_times(src, v)), src.frob2_all() ** 0.5
    if cfg == "4":
        H, X, src = problems.cfg4()
        desc = ("cfg4: n=1048576 depth=12 leaf=256, Gaussian sigma=0.01 on sorted uniform 1-D points, "
                "eps=1e-6, adaptive, fp64 working, 16 rhs")
        return H, X, desc, (lambda v: problems.kernel_times(src, v)), src.frob2_all() ** 0.5
    if cfg.startswith("5:"):
        eps = float(cfg.split(":")[1])
        H, x, src = problems.cfg5(eps)
        w = H.working_format.name
        desc = (f"cfg5: n=262144 depth=10 leaf=256, A_ij=1/(1+|i-j|), eps={eps:g}, adaptive, "
                f"{w} working, 1 rhs")
        return H, x.reshape(-1, 1), desc, (lambda v: problems.toeplitz_times(v)), src.frob2_all() ** 0.5
    raise SystemExit(f"unknown --config {cfg}")


def alg_flops(H, s):
    """F_alg = 2 s (sum_leaves m^2 + sum_factors (rows + cols) rank)."""
    f = sum((b - a) ** 2 for _, (a, b), _ in H.leaves())
    for _, _, _, _, up, lo in H.offdiag_blocks():
        for F in (up, lo):
            f += (F.U.shape[0] + F.V.shape[0]) * F.rank
    return 2 * s * f


def alg_bytes(H, s, wbytes):
    from paper_2407_21637_b200 import storage_bits

    return storage_bits(H) // 8 + H.n * s * (wbytes + wbytes)


def cpu_time_oracle(H, X, seconds):
    """Mean wall time of the CPU oracle (Alg. 3 restatement) over a bounded
    sample.  Multi-RHS fp32 working uses the strict-sequential loop per column:
    the sample is one column, scaled by s."""
    from oracle.matvec import matvec_oracle

    s = X.shape[1]
    cols = 1 if (s > 1 and H.working_format.name != "fp64") else s
    Xs = np.ascontiguousarray(X[:, :cols])
    matvec_oracle(H, Xs)  # warm
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 2:
        t0 = time.perf_counter()
        matvec_oracle(H, Xs)
        times.append(time.perf_counter() - t0)
        if len(times) >= 3 and time.perf_counter() > t_end:
            break
    scale = s / cols
    return float(np.mean(times)) * scale, len(times), cols


def main():
    args = parse()
    # the driver reads ONE JSON line from stdout: keep NCCL's version banner off it
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not launched by torchrun: relaunch one rank per GPU
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if world > 1 or args.sharded:
        from paper_2407_21637_b200 import dist

        if "WORLD_SIZE" not in os.environ:  # --sharded without torchrun: a one-rank group
            import socket

            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(port))

        return dist.bench_sharded(args, build_workload, alg_bytes, peaks, ClockSampler)
    return run_single(args)


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    H, X, desc, _, _ = build_workload(args.config)
    wb = 8 if H.working_format.name == "fp64" else 4
    s = X.shape[1]
    budget = max(args.cpu_seconds, 5.0)
    dt, nrep, cols = cpu_time_oracle(H, X, budget)
    cores = os.cpu_count()
    value = 1.0 / dt
    sample = (f"{nrep} full matvecs of the workload" if cols == s else
              f"{nrep} matvecs on {cols} of the {s} right-hand sides, time scaled by {s // cols}")
    line = {
        "impl": "reference", "metric": "HODLR matvecs/sec", "value": value, "unit": "matvec/s",
        "n_gpus": args.gpus, "steps": nrep, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if wb == 8 else "f32", "data": "synthetic (seeded, BASELINE shapes)",
        "config": {"workload": desc, "n": H.n, "depth": H.depth, "s": s,
                   "effective_GBps": alg_bytes(H, s, wb) / dt / 1e9},
        "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} (oracle Alg. 3, numpy/OpenBLAS fp64 or strict-sequential fp32 C "
                                   f"loop, {cores} threads)"},
        "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_single(args):
    import torch

    from paper_2407_21637_b200 import linops

    dev = 0
    torch.cuda.set_device(dev)
    t_build = time.perf_counter()
    H, X, desc, Kx, normA = build_workload(args.config)
    t_build = time.perf_counter() - t_build
    working = H.working_format
    wb = 8 if working.name == "fp64" else 4
    dt = torch.float64 if wb == 8 else torch.float32
    n, s = X.shape
    op = linops.HodlrOperator(H, dev)
    path, launches = op.path(s)
    stream = torch.cuda.current_stream()
    xd = torch.from_numpy(np.ascontiguousarray(X)).cuda().to(dt)
    bd = torch.empty_like(xd)
    flush = torch.ones(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def step():
        op.matvec(xd, out=bd)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- parity on the bench workload (GPU vs oracle; backward error vs K x)
    from oracle.matvec import matvec_oracle

    b_gpu = bd.double().cpu().numpy()
    xw = X.astype(np.float32).astype(np.float64) if wb == 4 else X
    # fp64 oracle (BLAS) on the same H: both working precisions approximate it
    b_or = matvec_oracle(H, xw, "fp64")
    rel_or = float(np.linalg.norm(b_gpu - b_or) / np.linalg.norm(b_or))
    kx = Kx(xw if s > 1 else xw[:, 0])
    from paper_2407_21637_b200.metrics import matvec_backward_error, matvec_bound

    beta = matvec_backward_error(np.asarray(kx).reshape(n, s), xw, b_gpu, normA)
    bound = matvec_bound(H.depth, H.eps)

    # ---- timed region: K steps, L2 flushed (untimed) before each
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    hot0, hot1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        for i in range(K):
            flush.sum()  # read-only L2 flush: evicts the matrix and leaves no dirty lines
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        # hot-cache (L2-resident where it fits) back-to-back for reference
        hot0.record(stream)
        for _ in range(K):
            step()
        hot1.record(stream)
        torch.cuda.synchronize()
        # e2e through the host-buffer entry point, pinned buffers
        Ke = max(10, K // 4)
        xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()
        bh = torch.empty_like(xh).pin_memory()
        for _ in range(3):
            op.matvec_host_ptr(xh.data_ptr(), bh.data_ptr(), s, stream=stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(Ke):
            op.matvec_host_ptr(xh.data_ptr(), bh.data_ptr(), s, stream=stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    ms_hot = hot0.elapsed_time(hot1) / K
    ms_e2e = e0.elapsed_time(e1) / Ke
    tol = 1e-12 if wb == 8 else 1e-5
    e2e_ok = bool(np.linalg.norm(bh.numpy() - b_gpu) <= tol * np.linalg.norm(b_gpu))

    B = alg_bytes(H, s, wb)
    F = alg_flops(H, s)
    peak, peak_src = peaks()
    achieved = B / (ms * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_cfg{args.config.replace(':', '_')}.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    cpu = None
    if not args.no_cpu_baseline:
        t_cpu, nrep, cols = cpu_time_oracle(H, X, args.cpu_seconds)
        cores = os.cpu_count()
        smp = (f"{nrep} full matvecs of the workload" if cols == s else
               f"{nrep} matvecs on {cols} of the {s} right-hand sides, time scaled by {s // cols}")
        cpu = {"value": 1.0 / t_cpu, "unit": "matvec/s", "cores": cores, "kind": "port",
               "sample": f"{smp} (oracle Alg. 3, numpy/OpenBLAS fp64 or strict-sequential fp32 C loop, "
                         f"{cores} threads), mean wall time"}
    value = 1000.0 / ms
    kernels = {"fused_sv": "k_stream (fused single-vector kernel, one launch per matvec)",
               "mrhs_slab": "k_mr2_a + k_mr_reduce + k_mr2_b (multi-RHS, fragment slabs, "
                            + ("DMMA fp64" if wb == 8 else "3xTF32 mma.sync") + ")",
               "mrhs": "k_mr_a + k_mr_reduce + k_mr_b (multi-RHS, arena)",
               "mrhs_tc": "k_tc_a + k_mr_reduce + k_tc_b (multi-RHS, tcgen05 kind::tf32 3xTF32, A in TMEM)",
               "generic": "generic three-launch kernels"}
    line = {
        "metric": "HODLR matvecs/sec", "value": value, "unit": "matvec/s", "n_gpus": 1,
        "steps": K, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if wb == 8 else "f32",
        "data": "synthetic (seeded, BASELINE shapes)",
        "config": {
            "workload": desc, "n": H.n, "depth": H.depth, "s": s, "eps": H.eps,
            "level_formats": [f.name for f in H.plan.chosen],
            "ranks": [max(u.rank, l.rank) for u, l in (H.blocks[k][0] for k in range(H.depth))],
            "matrix_bytes": int(op.matrix_bytes), "alg_bytes_per_matvec": int(B), "alg_flops_per_matvec": int(F),
            "l2": "flushed before every timed step (256 MiB read, untimed)",
            "effective_GBps": achieved, "alg_TFLOPs": F / (ms * 1e-3) / 1e12,
            "vector_matvecs_per_s": value * s,
            "hot_cache_ms": ms_hot, "hot_cache_matvecs_per_s": 1000.0 / ms_hot,
            "build_seconds": t_build, "parallelism": "single GPU", "kernel_path": path,
        },
        "parity": {"rel_err_vs_oracle_fp64": rel_or, "backward_error": beta, "bound_thm35": bound,
                   "within_10x_bound": beta <= 10 * bound, "e2e_matches": e2e_ok},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": kernels.get(path, path)},
        "e2e": {"value": 1000.0 / ms_e2e, "unit": "matvec/s", "h2d_bytes_per_step": int(n * s * 8),
                "d2h_bytes_per_step": int(n * s * 8), "ms_per_step": ms_e2e},
        "gpu_launches": K * launches,
        "clocks": clocks.summary(),
    }
    if path == "mrhs_tc":
        # tensor-pipe view: executed tf32 MMA flops (hi*hi + hi*lo for every block, + lo*hi for
        # fp32-stored blocks) against the kind::tf32 dense peak = half the measured bf16 peak
        passes = 3.0
        tpeak = _measured_bf16() / 2.0
        line["tensor"] = {"kind": "tcgen05.mma kind::tf32 (3xTF32 split, fp32 accumulate in TMEM)",
                          "executed_TFLOPs": passes * F / (ms * 1e-3) / 1e12, "peak_TFLOPs": tpeak,
                          "frac": passes * F / (ms * 1e-3) / 1e12 / tpeak if tpeak else None,
                          "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (tf32 = half-rate kind)"}
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    return 0


def _measured_bf16():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        return 2250.0


if __name__ == "__main__":
    sys.exit(main())
