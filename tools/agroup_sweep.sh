#!/bin/bash
# A-item grouping of the fused kernel on the binary32-working cfg5 cases (geometry 1), run on the GPU box
cd "$(dirname "$0")/.."
for CFG in 5:1e-2 5:1e-4; do
C=/tmp/sweep_cfg${CFG//:/_}.npz
python tools/run_matvec.py --config $CFG --iters 4 --cache $C > /dev/null 2>&1
for r in 1 2; do
for g in default 1 2 99; do
  echo -n "cfg $CFG A_GROUP $g: "
  if [ $g = default ]; then
    HODLR_B200_VERBOSE=1 timeout 120 python tools/run_matvec.py --config $CFG --iters 200 --time --cache $C 2>&1 | grep -E "TIME|rror|fused path" | tr '\n' ' '
  else
    HODLR_B200_VERBOSE=1 HODLR_B200_A_GROUP=$g timeout 120 python tools/run_matvec.py --config $CFG --iters 200 --time --cache $C 2>&1 | grep -E "TIME|rror|fused path" | tr '\n' ' '
  fi
  echo
done; done; done
