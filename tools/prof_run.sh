#!/bin/bash
# Run the instrumented (HODLR_PROFILE) build on cfg2 and print the per-CTA cycle accounting.
cd "$(dirname "$0")/.."
cp paper_2407_21637_b200/libhodlr_b200.so /tmp/libhodlr_b200.so.keep
cp tools/libhodlr_b200_prof.so paper_2407_21637_b200/libhodlr_b200.so
python tools/run_matvec.py --config ${1:-2} --iters 4 2>&1 | grep -E "PROF|ok" | tail -8
cp /tmp/libhodlr_b200.so.keep paper_2407_21637_b200/libhodlr_b200.so
