#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/f4; O=gpurun_out/f4
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --config 1 --steps 500 --warmup 10 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
for e in 1e-2 1e-4 1e-6 1e-8 1e-10; do
  timeout 900 python bench.py --config 5:$e --steps 100 --warmup 5 --cpu-seconds 5 > $O/bench_cfg5_$e.json 2> $O/bench_cfg5_$e.err
done
timeout 600 python bench.py --sharded --steps 200 --warmup 5 --no-cpu-baseline > $O/bench_sharded1_cfg2.json 2> $O/bench_sharded1.err
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stream" -c 40 --csv --log-file $O/launches_cfg2.csv $CMD > $O/ncu_launch.log 2>&1
python tools/run_matvec.py --config 2 --iters 8 --cache /tmp/cfg2_cache.npz > $O/ncu_full_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 4 -c 1 -o $O/full_cfg2 -f \
  python tools/run_matvec.py --config 2 --iters 8 --cache /tmp/cfg2_cache.npz > $O/ncu_full_cfg2.log 2>&1
echo done > $O/DONE
