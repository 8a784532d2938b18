#!/bin/bash
# cfg2 fused-kernel time vs the queue position of the R pieces (HODLR_POS_R)
cd "$(dirname "$0")/.."
python tools/run_matvec.py --config 2 --cache /tmp/cfg2.npz --iters 3 > /dev/null 2>&1
for p in ${POSR:-64 128 192 256 384 512}; do
  echo "pos_r $p: $(HODLR_POS_R=$p python tools/run_matvec.py --config 2 --cache /tmp/cfg2.npz --time --iters 200 2>&1 | grep TIME)"
done
