#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out/sv_sweep6.txt; : > $O
run() {
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg$cfg $*', round(d['ms_per_step']*1e3,2), 'us hot', round(d['config']['hot_cache_ms']*1e3,2), 'err', d['parity']['rel_err_vs_oracle_fp64'])" >> $O 2>&1
}
for rep in 1; do
run 2 X=0
run 2 HODLR_R_BYTES=16384
run 2 HODLR_R_BYTES=8192
run 2 HODLR_R_BYTES=4096
run 2 HODLR_POS_R=32
run 2 HODLR_POS_R=256
done
