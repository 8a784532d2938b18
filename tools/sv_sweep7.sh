#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out/sv_sweep7.txt; : > $O
run() {
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg$cfg $*', round(d['ms_per_step']*1e3,2), 'us hot', round(d['config']['hot_cache_ms']*1e3,2), 'err', d['parity']['rel_err_vs_oracle_fp64'])" >> $O 2>&1
}
for rep in 1 2; do
run 2 X=0
run 2 HODLR_POS_R=64
run 2 HODLR_POS_R=96
run 2 HODLR_POS_R=192
run 2 HODLR_R_BYTES=12288
done
python tools/trace_run.py --config 2 > gpurun_out/trace_cfg2_final.txt 2>&1
