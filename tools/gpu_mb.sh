#!/bin/bash
# MB ring/buffer variants on cfg4 (and cfg3): per-kernel times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mrhs.py -x -q > gpurun_out/pytest_mrhs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mrhs.log
for c in ${CONFIGS:-4 3}; do
  for v in "1 8" "1 6" "1 4" "2 4" "2 3"; do set -- $v
    echo "== cfg$c nbuf=$1 ns=$2" >> gpurun_out/mb_variants.log
    HODLR_B200_MB_NBUF=$1 HODLR_B200_MB_NS=$2 timeout 600 python tools/time_configs.py $c --prof 2>&1 | grep -E "matvec|k_mr2" >> gpurun_out/mb_variants.log
  done
done
