#!/bin/bash
# The paper's experiments on the GPU path: Fig. 4 matvec sweep (mat-1..4, n=2000, l=8,
# fp64/fp32/bf16 working, 10 trials) and the LU sweep; CSVs under gpurun_out/sweeps/.
cd "$(dirname "$0")/.."
O=gpurun_out/sweeps; mkdir -p $O
timeout 600 python -m pytest tests/test_lu.py tests/test_experiments.py -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 1500 python -m paper_2407_21637_b200.experiments matvec --out $O/fig4_matvec.csv > $O/fig4.log 2>&1; echo "rc=$?" >> $O/fig4.log
timeout 900 python -m paper_2407_21637_b200.experiments lu --out $O/lu_sweep.csv > $O/lu.log 2>&1; echo "rc=$?" >> $O/lu.log
tail -3 $O/pytest.log $O/fig4.log $O/lu.log
