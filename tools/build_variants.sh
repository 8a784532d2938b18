#!/bin/bash
# Build libhodlr_b200.so variants of the fast-path constants for a timing sweep:
#   tools/build_variants.sh "NS CTAS STAGE_KB CONSUMERS" ...
set -e
cd "$(dirname "$0")/../paper_2407_21637_b200/csrc"
for cfg in "$@"; do
  set -- $cfg
  tag="ns$1_c$2_s$3_w$4"
  sed -e "s/^constexpr int kNS = [0-9]*;/constexpr int kNS = $1;/" \
      -e "s/^constexpr int kCtasPerSm = [0-9]*;/constexpr int kCtasPerSm = $2;/" \
      -e "s/^constexpr int kStage = [0-9]* \* 1024;/constexpr int kStage = $3 * 1024;/" \
      -e "s/^constexpr int kConsumers = [0-9]*;/constexpr int kConsumers = $4;/" kernels_sv.cu > build/kv_$tag.cu
  cp *.cuh *.h build/ 2>/dev/null || true
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
       -I. -c build/kv_$tag.cu -o build/kv_$tag.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/libhodlr_b200_$tag.so \
       build/capi.o build/kernels_generic.o build/kv_$tag.o -cudart static
  echo built $tag
done
