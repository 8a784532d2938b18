#!/bin/bash
# Round-end evidence on one GPU: GPU tests, smoke, every config's bench line,
# the reference arm, the 1-rank sharded path, ncu launch lists and one
# `ncu --set full` capture of the top kernels (cfg2 k_stream, cfg4 k_mr2_b).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; O=gpurun_out/re; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref_cfg2.json 2> $O/bench_ref.err
timeout 600 python bench.py --config 1 --steps 500 --warmup 10 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --config 4 --steps 40 --warmup 3 --cpu-seconds 10 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config 3 --steps 40 --warmup 3 --cpu-seconds 10 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for e in 1e-2 1e-4 1e-6 1e-8 1e-10; do
  timeout 900 python bench.py --config 5:$e --steps 100 --warmup 5 --cpu-seconds 5 > $O/bench_cfg5_$e.json 2> $O/bench_cfg5_$e.err
done
timeout 600 python bench.py --sharded --steps 200 --warmup 5 --no-cpu-baseline > $O/bench_sharded1_cfg2.json 2> $O/bench_sharded1.err
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$CMD > $O/ncu_plain_cfg2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stream|k_gen|k_ext|k_round|k_widen" -c 60 --csv --log-file $O/launches_cfg2.csv $CMD > $O/ncu_launch_cfg2.log 2>&1
for c in 3 4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tc_|k_mr|k_stream|k_gen|k_ext" -c 40 --csv \
    --log-file $O/launches_cfg$c.csv python tools/time_configs.py $c > $O/ncu_launch_cfg$c.log 2>&1
done
python tools/run_matvec.py --config 2 --iters 8 --cache /tmp/cfg2_cache.npz > $O/ncu_full_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 4 -c 1 -o $O/full_cfg2 -f \
  python tools/run_matvec.py --config 2 --iters 8 --cache /tmp/cfg2_cache.npz > $O/ncu_full_cfg2.log 2>&1
echo "rc=$?" >> $O/ncu_full_cfg2.log
echo done > $O/DONE
