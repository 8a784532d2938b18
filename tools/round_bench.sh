#!/bin/bash
# Round-end evidence on one GPU: cfg1 and cfg5 sweep bench lines, and the ncu
# launch list (per-kernel durations) of the multi-RHS cfg3 / cfg4 paths and the
# fused cfg2 kernel (only our kernels are profiled: -k filter).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --config 1 --steps 200 --warmup 5 > gpurun_out/b_cfg1.json 2> gpurun_out/b_cfg1.err
for e in 1e-2 1e-4 1e-6 1e-8 1e-10; do
  timeout 900 python bench.py --config 5:$e --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg5_$e.json 2> gpurun_out/b_cfg5_$e.err
done
for c in 2 3 4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tc_|k_mr|k_stream|k_gen|k_ext" -c 40 --csv \
    --log-file gpurun_out/launches_cfg$c.csv python tools/time_configs.py $c > gpurun_out/ncu_launch_cfg$c.log 2>&1
done
echo done
