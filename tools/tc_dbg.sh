#!/bin/bash
# Time cfg3's tcgen05 kernels under HODLR_TC_DBG ablations (results are NOT valid under dbg != 0):
#   1 no A_lo pass, 2 no MMAs, 4 converters skip smem loads, 8 stagers skip global loads, 16 phase-A epilogue no flush
cd "$(dirname "$0")/.."
for d in ${DBGS:-0 1 2 4 8 14}; do
  echo "== dbg $d"
  HODLR_TC_DBG=$d timeout 300 python tools/time_configs.py 3 --prof 2>&1 | grep -E "k_tc_|matvec s="
done
