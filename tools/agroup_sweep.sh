#!/bin/bash
# Runtime knobs of the fused kernel on the binary32-working cfg5 cases (geometry 1), run on the GPU box:
#   tools/agroup_sweep.sh            A-item grouping (HODLR_B200_A_GROUP), R piece bytes, R queue position
cd "$(dirname "$0")/.."
run() {  # run <label> <env assignments...>
  echo -n "$1: "; shift
  env "$@" HODLR_B200_VERBOSE=1 timeout 120 python tools/run_matvec.py --config $CFG --iters 200 --time --cache $C 2>&1 | grep -E "TIME|rror|fused path" | sed 's/.*items/items/' | tr '\n' ' '
  echo
}
for CFG in 5:1e-2 5:1e-4; do
C=/tmp/sweep_cfg${CFG//:/_}.npz
python tools/run_matvec.py --config $CFG --iters 4 --cache $C > /dev/null 2>&1
for r in 1 2; do
  run "cfg $CFG default" X=1
  for g in 1 2 99; do run "cfg $CFG A_GROUP $g" HODLR_B200_A_GROUP=$g; done
  for b in 2048 4096 16384 20800; do run "cfg $CFG R_BYTES $b" HODLR_R_BYTES=$b; done
  for p in 0 64 256 1024; do run "cfg $CFG POS_R $p" HODLR_POS_R=$p; done
  run "cfg $CFG STATIC" HODLR_SV_STATIC=1
done; done
