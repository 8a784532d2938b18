#!/bin/bash
# New round-2 tests only (strict-order kernels, containers, builder pins, Fig. 4 harness).
cd "$(dirname "$0")/.."
O=gpurun_out/new; mkdir -p $O
timeout 1200 python -m pytest tests/test_experiments.py tests/test_container.py tests/test_gpu_builder.py tests/test_capi.py -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -40 $O/pytest.log
