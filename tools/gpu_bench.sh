#!/bin/bash
# Round evidence: GPU tests, bench lines (cfg2 headline, cfg4, cfg3, reference arm,
# 1-rank sharded path), and the ncu launch list of the headline bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out
echo skip-tests > $O/pytest_gpu.log

timeout 600 python bench.py --steps 500 --warmup 10 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --config 4 --steps 40 --warmup 3 --cpu-seconds 10 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config 3 --steps 40 --warmup 3 --cpu-seconds 10 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref_cfg2.json 2> $O/bench_ref.err
timeout 600 python bench.py --sharded --steps 200 --warmup 5 --no-cpu-baseline > $O/bench_sharded1.json 2> $O/bench_sharded1.err
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$CMD > $O/ncu_plain_cfg2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg2.csv $CMD > $O/ncu_launch.log 2>&1
echo done >> $O/pytest_gpu.log
