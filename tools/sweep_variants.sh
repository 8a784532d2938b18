#!/bin/bash
# Time every tools/variants/*.so on one workload (run on the GPU box).
cd "$(dirname "$0")/.."
CFG=${1:-2}
cp paper_2407_21637_b200/libhodlr_b200.so /tmp/libhodlr_b200.so.main
python tools/run_matvec.py --config $CFG --iters 4 --cache /tmp/cfg$CFG.npz > /dev/null 2>&1
for so in tools/variants/*.so; do
  cp $so paper_2407_21637_b200/libhodlr_b200.so
  VARIANT=$(basename $so .so) timeout 120 python tools/run_matvec.py --config $CFG --iters 60 --time --cache /tmp/cfg$CFG.npz 2>&1 | grep -E "TIME|Error|error" | head -2
done
cp /tmp/libhodlr_b200.so.main paper_2407_21637_b200/libhodlr_b200.so
