#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out/sv_sweep4.txt; : > $O
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_matvec.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
run() {
  env "$@" timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step']*1e3,2), 'us hot', round(d['config']['hot_cache_ms']*1e3,2), 'err', d['parity']['rel_err_vs_oracle_fp64'])" >> $O 2>&1
}
run X=0
run HODLR_R_BYTES=8192
run X=0
run HODLR_R_BYTES=8192
python tools/trace_run.py --config 2 > gpurun_out/trace_cfg2_rjob.txt 2>&1
