#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/sweep_variants.sh 2 2 > gpurun_out/variants2_cfg2.txt 2>&1
bash tools/sweep_variants.sh 5:1e-4 1 > gpurun_out/variants2_cfg5.txt 2>&1
