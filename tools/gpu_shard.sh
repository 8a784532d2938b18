#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mrhs.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
timeout 600 python tools/shard_time.py 4 1 2 4 8 > gpurun_out/shard_time_cfg4.log 2>&1
