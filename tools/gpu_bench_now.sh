#!/bin/bash
# Default bench at the driver's settings + the reference arm + the 1-rank sharded path.
cd "$(dirname "$0")/.."
O=gpurun_out/bench; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
timeout 900 python bench.py --sharded --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_sharded1.json 2> $O/bench_sharded1.err; echo "rc=$?" >> $O/bench_sharded1.err
tail -2 $O/*.err
