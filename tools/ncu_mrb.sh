#!/bin/bash
# ncu --set full (source-level) of the slab phase-A kernel on cfg4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/time_configs.py 4 > gpurun_out/mrb_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_mr2_b -s 3 -c 1 -o gpurun_out/prof_mrb_cfg4 -f \
  python tools/time_configs.py 4 > gpurun_out/mrb_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/mrb_ncu.log
