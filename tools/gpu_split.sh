#!/bin/bash
# Split (A launch + PDL-dependent R/BC launch) vs single fused launch: tests and bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for sp in 1 0; do
  HODLR_SV_SPLIT=$sp timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > $O/bench_cfg2_split$sp.json 2> $O/bench_cfg2_split$sp.err
  for e in 1e-2 1e-10; do
    HODLR_SV_SPLIT=$sp timeout 600 python bench.py --config 5:$e --steps 50 --warmup 3 --no-cpu-baseline > $O/bench_cfg5_${e}_split$sp.json 2> $O/bench_cfg5_${e}_split$sp.err
  done
done
