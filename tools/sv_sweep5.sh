#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out/sv_sweep5.txt; : > $O
HODLR_B200_A_GROUP=2 timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_matvec.py -x -q > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
run() {
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg$cfg $*', round(d['ms_per_step']*1e3,2), 'us hot', round(d['config']['hot_cache_ms']*1e3,2), 'err', d['parity']['rel_err_vs_oracle_fp64'])" >> $O 2>&1
}
for g in 1 2 4 1 2; do run 2 HODLR_B200_A_GROUP=$g; done
for g in 1 2; do run 5:1e-4 HODLR_B200_A_GROUP=$g; run 5:1e-8 HODLR_B200_A_GROUP=$g; done
HODLR_B200_A_GROUP=2 python tools/trace_run.py --config 2 > gpurun_out/trace_cfg2_ag2.txt 2>&1
