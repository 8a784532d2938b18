#!/bin/bash
# ncu --set full of the multi-RHS kernels on a reduced cfg (args: cfg n depth s kernel-regex)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python tools/time_configs.py $1 $2 $3 $4"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$5" -s 3 -c 2 -o gpurun_out/prof_$5_cfg$1 -f $CMD > gpurun_out/ncu_run.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_run.log
