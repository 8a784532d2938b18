#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python tools/time_configs.py 4 --prof > $O/time_cfg4.log 2>&1
timeout 900 python bench.py --config 4 --steps 40 --warmup 3 --cpu-seconds 10 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
