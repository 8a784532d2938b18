#!/bin/bash
# One GPU round trip: tests, bench line (cfg2), config timings.  Logs -> gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench_cfg2.log 2>&1
for c in ${CONFIGS:-3 4}; do timeout 900 python tools/time_configs.py $c > gpurun_out/time_cfg$c.log 2>&1; done
