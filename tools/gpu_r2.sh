#!/bin/bash
# Round-2 GPU check: full GPU suite (every BASELINE config at full size), smoke,
# the default bench (cfg4 headline + cfg2 secondary) at the driver's settings,
# and the reference arm.
cd "$(dirname "$0")/.."
O=gpurun_out/r2; mkdir -p $O
rm -f gpurun_out/parity_full.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cp gpurun_out/parity_full.jsonl $O/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
echo done > $O/DONE
