#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/f2; O=gpurun_out/f2
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q > $O/pytest_fused.log 2>&1; echo "rc=$?" >> $O/pytest_fused.log
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stream" -c 40 --csv --log-file $O/launches_cfg2.csv $CMD > $O/ncu_launch.log 2>&1
python tools/e2e_breakdown.py 2 > $O/e2e_breakdown.txt 2>&1
