#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out/sv_sweep3.txt; : > $O
HODLR_SV_STATIC=1 timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_matvec.py -x -q > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
run() {
  env "$@" timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step']*1e3,2), 'us hot', round(d['config']['hot_cache_ms']*1e3,2), 'err', d['parity']['rel_err_vs_oracle_fp64'])" >> $O 2>&1
}
run HODLR_SV_STATIC=0
run HODLR_SV_STATIC=1
run HODLR_SV_STATIC=0
run HODLR_SV_STATIC=1
run HODLR_SV_STATIC=1 HODLR_R_BYTES=8192
HODLR_SV_STATIC=0 python tools/trace_run.py --config 2 > gpurun_out/trace_cfg2_s0.txt 2>&1
HODLR_SV_STATIC=1 python tools/trace_run.py --config 2 > gpurun_out/trace_cfg2_s1.txt 2>&1
