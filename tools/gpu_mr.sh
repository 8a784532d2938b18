#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mrhs.py -x -q > gpurun_out/pytest_mrhs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mrhs.log
for c in ${CONFIGS:-3 4}; do timeout 900 python tools/time_configs.py $c --prof > gpurun_out/time_cfg$c.log 2>&1; done
