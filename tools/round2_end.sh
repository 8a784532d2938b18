#!/bin/bash
# Round-2 evidence on one B200 -> gpurun_out/r2e/ (summaries are copied to profiles/ by hand):
# GPU tests, smoke, bench lines (cfg4 headline + cfg2 secondary, reference arm, cfg1/3/5),
# ncu launch list of the bench command, ncu --set full of the cfg4 kernels, emulated
# per-rank shard times.
cd "$(dirname "$0")/.."
O=gpurun_out/r2e; mkdir -p $O
rm -f gpurun_out/parity_full.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cp gpurun_out/parity_full.jsonl $O/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "rc=$?" >> $O/bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_cfg4.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
timeout 600 python bench.py --config 1 --steps 200 --warmup 10 --no-secondary > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 --cpu-seconds 10 --no-secondary > $O/bench_cfg3.json 2> $O/bench_cfg3.err
HODLR_B200_TC_SUMS=tmem timeout 900 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --no-secondary > $O/bench_cfg3_tmemsums.json 2> $O/bench_cfg3_tmemsums.err
for e in 1e-2 1e-4 1e-6 1e-8 1e-10; do
  timeout 900 python bench.py --config 5:$e --steps 50 --warmup 5 --cpu-seconds 5 --no-secondary > $O/bench_cfg5_$e.json 2> $O/bench_cfg5_$e.err
done
# ncu: launch list of the bench command (cold, serialised: shares, not absolutes)
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline"
$CMD > $O/ncu_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_mr|k_stream|k_gen|k_tc" -c 120 --csv --log-file $O/launches_bench.csv $CMD > $O/ncu_launch.log 2>&1
# ncu --set full of the cfg4 kernels (synthetic matrix of cfg4's shape: same kernels, same bytes)
for k in k_mr2_b k_mr4_a; do
  python tools/synth_time.py 4 --iters 3 > $O/full_plain_$k.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o $O/full_$k -f python tools/synth_time.py 4 --iters 3 > $O/full_$k.log 2>&1
  # (reports are 25 MB each and gpurun_out/ is capped at 64 MiB: keep the text summaries)
  python tools/ncu_summary.py $O/full_$k.ncu-rep > $O/ncu_full_$k.txt 2>&1; python tools/ncu_sass.py $O/full_$k.ncu-rep 25 >> $O/ncu_full_$k.txt 2>&1; rm -f $O/full_$k.ncu-rep
done
for k in k_tc_a k_tc_b; do
  python tools/synth_time.py 3 --iters 3 > $O/full_plain_$k.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/full_$k -f python tools/synth_time.py 3 --iters 3 > $O/full_$k.log 2>&1
  python tools/ncu_summary.py $O/full_$k.ncu-rep > $O/ncu_full_$k.txt 2>&1; python tools/ncu_sass.py $O/full_$k.ncu-rep 25 >> $O/ncu_full_$k.txt 2>&1; rm -f $O/full_$k.ncu-rep
done
timeout 300 python tools/synth_time.py 3 --prof > $O/synth_cfg3_kernels.txt 2>&1
python tools/synth_time.py 2 --iters 3 > $O/full_plain_sv.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 4 -c 1 -o $O/full_k_stream -f python tools/synth_time.py 2 --iters 3 > $O/full_k_stream.log 2>&1
python tools/ncu_summary.py $O/full_k_stream.ncu-rep > $O/ncu_full_k_stream.txt 2>&1; python tools/ncu_sass.py $O/full_k_stream.ncu-rep 25 >> $O/ncu_full_k_stream.txt 2>&1; rm -f $O/full_k_stream.ncu-rep
timeout 600 python tools/shard_time.py s4 1 2 4 8 2>&1 | grep -v -i warn > $O/shard_rank_times_cfg4.txt
echo done > $O/DONE
