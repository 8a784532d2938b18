#!/bin/bash
# Fused-kernel knob sweep on cfg2 (A item grouping, R piece size, R queue position).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out/sv_sweep.txt; : > $O
run() {
  env "$@" timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step']*1e3,2), 'us hot', round(d['config']['hot_cache_ms']*1e3,2), 'err', d['parity']['rel_err_vs_oracle_fp64'])" >> $O 2>&1
}
run X=0
run HODLR_B200_A_GROUP=2
for rb in 16384 8192 4096; do run HODLR_R_BYTES=$rb; run HODLR_B200_A_GROUP=2 HODLR_R_BYTES=$rb; done
run HODLR_B200_A_GROUP=2 HODLR_POS_R=0
run HODLR_B200_A_GROUP=2 HODLR_POS_R=40
run HODLR_R_BYTES=8192 HODLR_POS_R=40
