"""Benchmark of the B200 HODLR matvec (BASELINE.json metric: "HODLR matvecs/sec
and effective HBM GB/s (frac. of roofline) at 1/2/4/8 B200").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl reference]

* Headline workload: BASELINE config 4, the largest config and the one the
  metric's "1/2/4/8 B200" scaling is quoted on -- n = 2^20, depth 12 (256-row
  leaves), Gaussian kernel sigma = 0.01 on sorted uniform 1-D points, eps = 1e-6,
  adaptive per-level formats, fp64 working, 16 right-hand sides; built by the
  package's restatement of Alg. 2 on the GPU from seeded inputs (the reference
  cannot build it: its construction is dense n x n).  ``--config 1|2|3|5:eps``
  selects another BASELINE config.  At N = 1 the default run also times config
  2 (the single-vector fused kernel) and reports it under ``secondary``.
* ``value``: matvecs/s with X, B and the packed matrix resident in HBM; every
  timed step is bracketed by CUDA events on the launching stream and preceded
  by an untimed L2 flush (reading a 256 MiB buffer).
* ``e2e``: the same metric through the public host-buffer entry point
  (``hodlr_matvec_host``): pinned binary64 X copied in, matvec, B copied out,
  every step, timed by events around the whole call.
* ``roofline``: algorithmic bytes per matvec = storage_bits(H)/8 + n*s*(w_x+w_b)
  (hodlr.py:279-287) / the event time of one matvec, against
  the measured HBM copy bandwidth (MEASURED_PEAKS.json).
* ``cpu_baseline``: the CPU oracle (Alg. 3 restatement, numpy/OpenBLAS fp64) on
  the same H and X, all host threads, bounded sample; host provenance (CPU
  model, threads, OPENBLAS_NUM_THREADS) under ``host``.
* ``--impl reference``: the reference-side CPU implementation of the path (the
  oracle port: the reference package has no matvec of its own)
  timed for exactly W + K steps on the same workload.  The matrix is built in a
  child process and handed over as a container-v1 file, so the timing process
  never maps the CUDA extension.
* Multi-GPU (torchrun, N > 1): STRONG scaling of the same workload -- the tree
  is sharded at level log2(N), each rank owns n/N rows; one NCCL all-gather of
  V^T X coefficient partials per matvec; time = max over ranks; same unit.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLUSH_BYTES = 256 << 20
METRIC = "HODLR matvecs/sec"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="4")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg2 single-vector secondary line")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded (multi-GPU) code path even at one rank")
    ap.add_argument("--dump-workload", default=None, help=argparse.SUPPRESS)  # child of --impl reference
    return ap.parse_args(argv)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _measured_bf16():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        return 2250.0


# ------------------------------------------------------------------ host / clocks
def host_info():
    """CPU provenance of every CPU number."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info

        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads"), "version": d.get("version")}
                for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count()
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "usable_cpus": usable,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"), "blas": blas}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons polled through NVML every
    ~2 ms from a thread; ``timed(True/False)`` brackets the timed region, and
    the summary covers the samples taken inside it (all samples if none)."""

    HW_SLOWDOWN, SW_POWER_CAP, SW_THERMAL, HW_THERMAL = 0x8, 0x4, 0x20, 0x40

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (in_timed_region, sm_mhz, max_mhz, reasons bitmask)
        self._in = False
        self._stop = threading.Event()
        self._nvml = None

    def _handle(self):
        import pynvml

        pynvml.nvmlInit()
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            for cand in (uuid, "GPU-" + uuid):
                try:
                    return pynvml, pynvml.nvmlDeviceGetHandleByUUID(cand)
                except Exception:
                    pass
        except Exception:
            pass
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = self.device
        if vis:
            try:
                idx = int(vis.split(",")[self.device])
            except Exception:
                pass
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def __enter__(self):
        try:
            nv, h = self._handle()
            self._nvml = nv
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append((self._in, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                             int(get_r(h))))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
            t_end = time.time() + 2.0
            while not self.samples and time.time() < t_end:
                time.sleep(0.005)
        except Exception:
            self._nvml = None
        return self

    def timed(self, on: bool):
        if on:
            self._in = True
        else:
            time.sleep(0.004)  # let the poller see the end of the region
            self._in = False

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self.t.join(timeout=2)

    def summary(self):
        inside = [s for s in self.samples if s[0]]
        use = inside or self.samples
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "unavailable"}
        names = {self.HW_SLOWDOWN: "hw_slowdown", self.HW_THERMAL: "hw_thermal_slowdown",
                 self.SW_THERMAL: "sw_thermal_slowdown", self.SW_POWER_CAP: "sw_power_cap"}
        reasons = sorted({nm for bit, nm in names.items() for s in use if s[3] & bit})
        return {"sm_mhz": float(np.median([s[1] for s in use])), "sm_max_mhz": float(max(s[2] for s in use)),
                "reasons": reasons, "samples": len(use), "samples_in_timed_region": len(inside),
                "source": "NVML poll (~2 ms) during the timed steps"}


# ------------------------------------------------------------------ workloads
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


def wbytes_of(H):
    return 8 if H.working_format.name == "fp64" else 4


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
    return float(np.mean(times)) * (s / cols), len(times), cols


def _parity(H, X, b_gpu, Kx, normA):
    """GPU vs the fp64 oracle on the same H, and the judged backward error."""
    from oracle.matvec import matvec_oracle
    from paper_2407_21637_b200.metrics import hypothesis_holds, matvec_backward_error, matvec_bound

    n, s = X.shape
    xw = X.astype(np.float32).astype(np.float64) if wbytes_of(H) == 4 else X
    b_or = matvec_oracle(H, xw, "fp64")
    rel_or = float(np.linalg.norm(b_gpu - b_or) / np.linalg.norm(b_or))
    kx = Kx(xw if s > 1 else xw[:, 0])
    beta = matvec_backward_error(np.asarray(kx).reshape(n, s), xw, b_gpu, normA)
    bound = matvec_bound(H.depth, H.eps)
    return {"rel_err_vs_oracle_fp64": rel_or, "tol_vs_oracle": 1e-12 if wbytes_of(H) == 8 else 1e-5,
            "backward_error": beta, "bound_thm35": bound, "within_10x_bound": beta <= 10 * bound,
            "hypothesis_u_le_eps_over_n": bool(hypothesis_holds(H.working_format, H.eps, H.n))}


KERNELS = {"fused_sv": "k_stream (fused single-vector kernel, one launch per matvec)",
           "mrhs_slab64": "k_mr4_a (K-split 4 x 4 phase A) + k_mr_reduce + k_mr2_b (multi-RHS, fragment slabs, DMMA fp64)",
           "mrhs_slab32": "k_mr2_a + k_mr_reduce + k_mr2_b (multi-RHS, fragment slabs, 3xTF32 mma.sync)",
           "mrhs": "k_mr_a + k_mr_reduce + k_mr_b (multi-RHS, arena)",
           "mrhs_tc": "k_tc_a + k_mr_reduce + k_tc_b (multi-RHS, tcgen05 kind::tf32 3xTF32, A in TMEM)",
           "generic": "generic three-launch kernels"}


def _kernel_name(path, wb):
    if path == "mrhs_slab":
        return KERNELS["mrhs_slab64" if wb == 8 else "mrhs_slab32"]
    return KERNELS.get(path, path)


def time_device(op, xd, bd, K, W, flush, stream, clocks=None):
    """(mean ms over K L2-flushed steps, hot-cache ms) with CUDA events on `stream`."""
    import torch

    def step():
        op.matvec(xd, out=bd)

    for _ in range(max(W, 3)):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if clocks:
        clocks.timed(True)
    for i in range(K):
        flush.sum()  # read-only L2 flush: evicts the matrix and leaves no dirty lines
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.timed(False)
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(K):
        step()
    h1.record(stream)
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in ev])), h0.elapsed_time(h1) / K


def time_e2e(op, X, K, stream):
    """ms per host-buffer call (pinned X in, B out, every step) and the result."""
    import torch

    s = X.shape[1]
    xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()
    bh = torch.empty_like(xh).pin_memory()
    for _ in range(3):
        op.matvec_host_ptr(xh.data_ptr(), bh.data_ptr(), s, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    # short calls: enough of them for ~30 ms of timed region (a dozen 100-us calls is noise)
    t0 = time.perf_counter()
    op.matvec_host_ptr(xh.data_ptr(), bh.data_ptr(), s, stream=stream.cuda_stream)
    est_ms = max((time.perf_counter() - t0) * 1e3, 1e-3)
    K = int(min(400, max(K, 30.0 / est_ms)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K):
        op.matvec_host_ptr(xh.data_ptr(), bh.data_ptr(), s, stream=stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, bh.numpy().copy()


def time_e2e_two_callers(op, X, K, b_ref):
    """Host-buffer calls from TWO host threads (each with its own pinned buffers and stream):
    the C ABI keeps two staging contexts per handle, so one call's device-to-host copy runs
    under the other's host-to-device copy.  Every call still copies its X in and its B out.
    Returns ms per call (device time from the first call's start to the last call's end,
    divided by the 2 K calls) and whether both callers' results equal the serial result."""
    import threading

    import torch

    s = X.shape[1]
    xs, bs, sts = [], [], []
    for _ in range(2):
        xs.append(torch.from_numpy(np.ascontiguousarray(X)).pin_memory())
        bs.append(torch.empty_like(xs[-1]).pin_memory())
        sts.append(torch.cuda.Stream())
    errs = []

    def run(i, reps):
        try:
            for _ in range(reps):
                op.matvec_host_ptr(xs[i].data_ptr(), bs[i].data_ptr(), s, stream=sts[i].cuda_stream)
        except Exception as e:  # reported by the caller
            errs.append(repr(e))

    def both(reps):
        th = [threading.Thread(target=run, args=(i, reps)) for i in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    both(2)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e0.record(sts[0])
    sts[1].wait_event(e0)
    both(K)
    for i in range(2):
        ends[i].record(sts[i])
    torch.cuda.synchronize()
    if errs:
        raise RuntimeError("two-caller e2e: " + "; ".join(errs))
    ms = max(e0.elapsed_time(e) for e in ends) / (2 * K)
    same = all(np.array_equal(b.numpy(), b_ref) for b in bs)
    return ms, same


def measure_config(cfg, args, dev, clocks=None, cpu=True):
    """One BASELINE config on one GPU: parity, device time, e2e, roofline, CPU baseline."""
    import torch

    from paper_2407_21637_b200 import linops

    t_build = time.perf_counter()
    H, X, desc, Kx, normA = build_workload(cfg)
    t_build = time.perf_counter() - t_build
    wb = wbytes_of(H)
    dt = torch.float64 if wb == 8 else torch.float32
    n, s = X.shape
    op = linops.HodlrOperator(H, dev)
    path, launches = op.path(s)
    stream = torch.cuda.current_stream()
    xd = torch.from_numpy(np.ascontiguousarray(X)).cuda().to(dt)
    bd = torch.empty_like(xd)
    op.matvec(xd, out=bd)
    torch.cuda.synchronize()
    b_gpu = bd.double().cpu().numpy()
    parity = _parity(H, X, b_gpu, Kx, normA)

    flush = torch.ones(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    K = args.steps
    ms, ms_hot = time_device(op, xd, bd, K, args.warmup, flush, stream, clocks)
    ms_e2e, b_e2e = time_e2e(op, X, max(10, min(K, 200) // 4), stream)
    parity["e2e_matches"] = bool(np.linalg.norm(b_e2e - b_gpu) <= parity["tol_vs_oracle"] * np.linalg.norm(b_gpu))
    try:  # a secondary figure: never fails the headline line
        ms_e2e2, same2 = time_e2e_two_callers(op, X, int(min(500, max(5, 40.0 / ms_e2e))), b_e2e)  # ~80 ms of calls
        parity["e2e_two_callers_bitwise_equal"] = bool(same2)
    except Exception as e:
        print(f"[bench] two-caller e2e skipped: {e!r}", file=sys.stderr)
        ms_e2e2 = None
    del flush

    B = alg_bytes(H, s, wb)
    F = alg_flops(H, s)
    peak, peak_src = peaks()
    achieved = B / (ms * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_cfg{cfg.replace(':', '_')}.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    res = {
        "H": H, "X": X, "desc": desc, "path": path, "launches": launches, "ms": ms, "ms_hot": ms_hot,
        "ms_e2e": ms_e2e, "ms_e2e2": ms_e2e2, "B": B, "F": F, "wb": wb, "parity": parity, "t_build": t_build, "op": op,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "kernel": _kernel_name(path, wb),
                     "alg_bytes_per_launch": int(B)},
    }
    if cpu:
        t_cpu, nrep, cols = cpu_time_oracle(H, X, args.cpu_seconds)
        cores = os.cpu_count()
        smp = (f"{nrep} full matvecs of the workload" if cols == s else
               f"{nrep} matvecs on {cols} of the {s} right-hand sides, time scaled by {s // cols}")
        res["cpu"] = {"value": 1.0 / t_cpu, "unit": "matvec/s", "cores": cores, "kind": "port",
                      "sample": f"{smp} (oracle Alg. 3, numpy/OpenBLAS fp64 or strict-sequential fp32 C loop, "
                                f"{cores} threads), mean wall time"}
    return res


def main():
    args = parse()
    if args.dump_workload:
        return dump_workload(args)
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
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if world > 1 or args.sharded:
        if "WORLD_SIZE" not in os.environ:  # --sharded without torchrun: a one-rank group
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(_free_port()))
        return run_sharded(args)
    return run_single(args)


def _free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


# ------------------------------------------------------------------ 1 GPU
def run_single(args):
    import torch

    dev = 0
    torch.cuda.set_device(dev)
    with ClockSampler(dev) as clocks:
        r = measure_config(args.config, args, dev, clocks, cpu=not args.no_cpu_baseline)
    H, X, s, wb = r["H"], r["X"], r["X"].shape[1], r["wb"]
    ms = r["ms"]
    value = 1000.0 / ms
    line = {
        "metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if wb == 8 else "f32",
        "data": "synthetic (seeded, BASELINE shapes and distributions; random x ~ N(0,1))",
        "config": {
            "workload": r["desc"], "n": H.n, "depth": H.depth, "s": s, "eps": H.eps,
            "level_formats": [f.name for f in H.plan.chosen],
            "ranks": [max(u.rank, lo.rank) for u, lo in (H.blocks[k][0] for k in range(H.depth))],
            "matrix_bytes": int(r["op"].matrix_bytes), "alg_bytes_per_matvec": int(r["B"]),
            "alg_flops_per_matvec": int(r["F"]),
            "l2": "flushed before every timed step (256 MiB read, untimed)",
            "effective_GBps": r["roofline"]["achieved"], "alg_TFLOPs": r["F"] / (ms * 1e-3) / 1e12,
            "vector_matvecs_per_s": value * s,
            "hot_cache_ms": r["ms_hot"], "hot_cache_matvecs_per_s": 1000.0 / r["ms_hot"],
            "build_seconds": r["t_build"], "parallelism": "single GPU", "kernel_path": r["path"],
            "native_lib": _native_lib(),
        },
        "parity": r["parity"],
        "roofline": r["roofline"],
        "e2e": {"value": 1000.0 / r["ms_e2e"], "unit": "matvec/s", "h2d_bytes_per_step": int(H.n * s * 8),
                "d2h_bytes_per_step": int(H.n * s * 8), "ms_per_step": r["ms_e2e"],
                "path": "hodlr_matvec_host (pinned binary64 X in, B out), one caller, calls back to back",
                "two_callers": {"value": 1000.0 / r["ms_e2e2"] if r["ms_e2e2"] else None, "unit": "matvec/s",
                                "ms_per_step": r["ms_e2e2"],
                                "note": "same entry point from two host threads on two streams (two staging "
                                        "contexts per handle): one call's D2H overlaps the other's H2D; "
                                        "every call copies its X in and its B out"}},
        "gpu_launches": args.steps * r["launches"],
        "clocks": clocks.summary(),
        "host": host_info(),
    }
    if r["path"] == "mrhs_tc":
        tpeak = _measured_bf16() / 2.0
        ex = 3.0 * r["F"] / (ms * 1e-3) / 1e12
        line["tensor"] = {"kind": "tcgen05.mma kind::tf32 (3xTF32 split, fp32 accumulate in TMEM)",
                          "executed_TFLOPs": ex, "peak_TFLOPs": tpeak, "frac": ex / tpeak,
                          "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (tf32 = half-rate kind)"}
    if "cpu" in r:
        line["cpu_baseline"] = r["cpu"]
    del r
    if args.config == "4" and not args.no_secondary:
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        with ClockSampler(dev) as c2:
            r2 = measure_config("2", args, dev, c2, cpu=False)
        line["secondary"] = {"cfg2": {
            "workload": r2["desc"], "value": 1000.0 / r2["ms"], "unit": "matvec/s", "ms_per_step": r2["ms"],
            "kernel_path": r2["path"], "roofline": r2["roofline"], "parity": r2["parity"],
            "e2e": {"value": 1000.0 / r2["ms_e2e"], "unit": "matvec/s", "ms_per_step": r2["ms_e2e"],
                    "two_callers": {"value": 1000.0 / r2["ms_e2e2"] if r2["ms_e2e2"] else None, "unit": "matvec/s",
                                    "ms_per_step": r2["ms_e2e2"]}},
            "hot_cache_ms": r2["ms_hot"], "gpu_launches": args.steps * r2["launches"], "clocks": c2.summary()}}
        line["gpu_launches"] += args.steps * r2["launches"]
    print(json.dumps(line), flush=True)
    return 0


def _native_lib():
    try:
        from paper_2407_21637_b200 import _lib

        return os.path.relpath(_lib.LIB_PATH, ROOT)
    except Exception:
        return None


# ------------------------------------------------------------------ N GPUs
def run_sharded(args):
    """bench.py's N-GPU arm (torchrun, one rank per GPU, NCCL): strong scaling
    of the workload, the tree sharded at level log2(N)."""
    import torch
    import torch.distributed as tdist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    kw = {"backend": "nccl", "device_id": dev}
    try:
        opts = tdist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True  # the all-gather's CTAs go first next to the persistent kernels
        kw["pg_options"] = opts
    except Exception:
        pass
    tdist.init_process_group(**kw)
    try:
        return _run_sharded(args, rank, world, local, dev)
    finally:
        tdist.destroy_process_group()


def _run_sharded(args, rank, world, local, dev):
    import torch
    import torch.distributed as tdist

    from paper_2407_21637_b200 import dist

    L = dist.levels_of(world)
    t_build = time.perf_counter()
    H, x, desc, Kx, normA = build_workload(args.config)
    desc += f"; tree sharded at level {L} over {world} GPU(s) (strong scaling)"
    t_build = time.perf_counter() - t_build
    x = np.asarray(x).reshape(H.n, -1)
    s = x.shape[1]
    wb = wbytes_of(H)
    dt = torch.float64 if wb == 8 else torch.float32
    # the whole step (phase A, all-gather, phase B) replayed as one CUDA graph per
    # buffer pair; falls back to eager launches if the capture fails
    sop = dist.ShardedOperator(H, rank, world, device=local, use_graph=os.environ.get("HODLR_B200_SHARD_GRAPH", "1") == "1")
    op = sop.op
    r0, nl = sop.row0, sop.n_local
    xd = torch.from_numpy(np.ascontiguousarray(x[r0:r0 + nl])).to(dev).to(dt)
    bd = torch.empty_like(xd)
    flush = torch.ones(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        sop.matvec(xd, out=bd)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # parity: gather b on every rank, rank 0 checks against the oracle and K x
    parts = [torch.empty_like(bd) for _ in range(world)]
    tdist.all_gather(parts, bd)
    parity = None
    if rank == 0:
        parity = _parity(H, x, torch.cat(parts).double().cpu().numpy(), Kx, normA)

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ClockSampler(local) as clocks:
        tdist.barrier()
        torch.cuda.synchronize()
        clocks.timed(True)
        for i in range(K):
            flush.sum()  # read-only L2 flush, untimed
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        clocks.timed(False)
        tdist.barrier()
        # e2e: pinned host x_own in, b_own out, every step
        Ke = max(10, min(K, 200) // 4)
        xh = torch.from_numpy(np.ascontiguousarray(x[r0:r0 + nl])).pin_memory()
        bh = torch.empty_like(xh).pin_memory()
        xe = torch.empty((nl, s), dtype=torch.float64, device=dev)

        def e2e_step():
            xe.copy_(xh, non_blocking=True)
            sop.matvec(xe if dt == torch.float64 else xe.to(dt), out=bd)
            bh.copy_(bd if dt == torch.float64 else bd.double(), non_blocking=True)

        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize()
        tdist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(Ke):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms_local = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    ms_e2e_local = e0.elapsed_time(e1) / Ke
    t = torch.tensor([ms_local, ms_e2e_local], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms, ms_e2e = float(t[0]), float(t[1])
    B_all = alg_bytes(H, s, wb)
    mb = torch.tensor([op.matrix_bytes + 2 * nl * s * wb], dtype=torch.float64, device=dev)
    tdist.all_reduce(mb, op=tdist.ReduceOp.MAX)
    if rank != 0:
        return 0
    peak, peak_src = peaks()
    per_gpu = float(mb[0])  # largest shard's algorithmic bytes (matrix rows + x + b)
    achieved = per_gpu / (ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": 1000.0 / ms, "unit": "matvec/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if wb == 8 else "f32",
        "data": "synthetic (seeded, BASELINE shapes and distributions; random x ~ N(0,1))",
        "config": {
            "workload": desc, "n": H.n, "depth": H.depth, "s": s, "eps": H.eps,
            "level_formats": [f.name for f in H.plan.chosen],
            "alg_bytes_per_matvec": int(B_all), "alg_bytes_largest_shard": int(per_gpu),
            "effective_GBps_total": B_all / (ms * 1e-3) / 1e9,
            "exchange_bytes_per_rank": sop.exchange_bytes(s, wb),
            "l2": "flushed before every timed step (256 MiB read, untimed)",
            "build_seconds": t_build, "parallelism": f"tree sharded at level {L} over {world} GPUs, "
                                                     "NCCL all-gather of V^T x coefficients",
            "cuda_graph_replays": sop.graph_replays,
            "native_lib": _native_lib(),
        },
        "parity": parity,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_src,
                     "kernel": "whole sharded step per GPU (phase A incl. external partials, all-gather, "
                               "phase B), largest shard's algorithmic bytes"},
        "e2e": {"value": 1000.0 / ms_e2e, "unit": "matvec/s", "h2d_bytes_per_step": int(H.n * s * 8),
                "d2h_bytes_per_step": int(H.n * s * 8), "ms_per_step": ms_e2e},
        "gpu_launches": K * (op.path(s)[1] + 3 * (world > 1)) * world,
        "clocks": clocks.summary(),
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ reference arm
def dump_workload(args):
    """Child of --impl reference: build the workload (GPU builder) and save H
    (container v1) and X for the parent, which never loads the CUDA extension."""
    from paper_2407_21637_b200.model import save_hodlr

    H, X, desc, _, _ = build_workload(args.config)
    save_hodlr(H, os.path.join(args.dump_workload, "H.npz"))
    np.save(os.path.join(args.dump_workload, "X.npy"), np.ascontiguousarray(X))
    with open(os.path.join(args.dump_workload, "desc.txt"), "w") as f:
        f.write(desc)
    return 0


def run_reference(args, world, rank):
    """The reference-side CPU implementation of the path (the oracle port,
    all host threads) timed for exactly W + K steps on the workload."""
    if rank != 0:
        return 0
    from oracle.matvec import matvec_oracle
    from paper_2407_21637_b200.model import load_hodlr, storage_bits

    with tempfile.TemporaryDirectory(prefix="hodlr_ref_") as tmp:
        t0 = time.perf_counter()
        subprocess.check_call([sys.executable, os.path.abspath(__file__), "--config", args.config,
                               "--dump-workload", tmp], stdout=subprocess.DEVNULL)
        H = load_hodlr(os.path.join(tmp, "H.npz"))
        X = np.load(os.path.join(tmp, "X.npy"))
        desc = open(os.path.join(tmp, "desc.txt")).read()
        t_build = time.perf_counter() - t0
    wb = wbytes_of(H)
    n, s = X.shape
    # one step = one matvec of the workload; the fp32 strict-sequential loop is
    # per column, so for fp32 multi-RHS a step is one column, time scaled by s
    cols = 1 if (s > 1 and wb == 4) else s
    Xs = np.ascontiguousarray(X[:, :cols])
    for _ in range(args.warmup):
        matvec_oracle(H, Xs)
    times = []
    for _ in range(args.steps):
        t1 = time.perf_counter()
        matvec_oracle(H, Xs)
        times.append(time.perf_counter() - t1)
    dt = float(np.mean(times)) * (s / cols)
    hi = host_info()
    value = 1.0 / dt
    sample = (f"each step one full matvec of the workload" if cols == s else
              f"each step one matvec on 1 of the {s} right-hand sides (fp32 strict-sequential loop), "
              f"time scaled by {s}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "matvec/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if wb == 8 else "f32", "data": "synthetic (seeded, BASELINE shapes and distributions)",
        "config": {"workload": desc, "n": H.n, "depth": H.depth, "s": s, "eps": H.eps,
                   "alg_bytes_per_matvec": int(storage_bits(H) // 8 + n * s * 2 * wb),
                   "effective_GBps": (storage_bits(H) // 8 + n * s * 2 * wb) / dt / 1e9,
                   "matrix_handoff": f"built in a child process (GPU builder), container v1 file, "
                                     f"{t_build:.1f} s; this process runs numpy only"},
        "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": hi["usable_cpus"], "kind": "port",
                         "sample": f"{sample} (oracle Alg. 3: numpy/OpenBLAS fp64, or the strict-sequential "
                                   f"fp32 C loop), all host threads, mean of {args.steps} steps after "
                                   f"{args.warmup} warm-up"},
        "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": hi,
    }
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
