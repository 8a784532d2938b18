#!/bin/bash
# Iteration check on one GPU: GPU tests, e2e breakdown, cfg2 + cfg4 bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/e2e_breakdown.py 2 > $O/e2e_breakdown.txt 2>&1
timeout 600 python bench.py --steps 500 --warmup 10 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --config 4 --steps 40 --warmup 3 --cpu-seconds 5 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
