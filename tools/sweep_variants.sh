#!/bin/bash
# Time every tools/variants/*.so on one workload (run on the GPU box):
#   tools/sweep_variants.sh [config] [rounds]
cd "$(dirname "$0")/.."
CFG=${1:-2}
ROUNDS=${2:-1}
C=/tmp/sweep_cfg${CFG//:/_}.npz
python tools/run_matvec.py --config $CFG --iters 4 --cache $C > /dev/null 2>&1
for r in $(seq $ROUNDS); do
  for so in paper_2407_21637_b200/libhodlr_b200.so tools/variants/*.so; do
    HODLR_B200_LIB=$PWD/$so VARIANT=$(basename $so .so) timeout 120 python tools/run_matvec.py --config $CFG --iters 200 \
      --time --cache $C 2>&1 | grep -E "TIME|Error|error" | head -2
  done
done
