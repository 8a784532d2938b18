#!/bin/bash
# ncu --set full (source-level) of one kernel on a synthetic config: ncu_synth.sh <cfg> <kernel-regex> [skip]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/synth_time.py $1 --iters 3 > gpurun_out/synth_plain_$1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${3:-4} -c 1 -o gpurun_out/prof_$2_synth$1 -f \
  python tools/synth_time.py $1 --iters 3 > gpurun_out/synth_ncu_$1.log 2>&1
echo "rc=$?" >> gpurun_out/synth_ncu_$1.log; tail -3 gpurun_out/synth_ncu_$1.log
