#!/bin/bash
# Build libhodlr_b200.so variants of the fused kernel for a timing sweep:
#   tools/build_variants.sh "tag:-DHODLR_KNS=2 -DHODLR_KSTAGE=33280" "tag2:..." ...
# Outputs tools/variants/libhodlr_b200_<tag>.so (load with HODLR_B200_LIB=...).
set -e
cd "$(dirname "$0")/../paper_2407_21637_b200/csrc"
make -s
mkdir -p ../../tools/variants
for spec in "$@"; do
  tag=${spec%%:*}
  defs=${spec#*:}
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
       $defs -c kernels_sv.cu -o build/kv_$tag.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/libhodlr_b200_$tag.so \
       build/capi.o build/kernels_generic.o build/kernels_seq.o build/kernels_shard.o build/kernels_mrhs.o build/kernels_tc.o build/kernels_sv_g1.o build/kv_$tag.o -cudart static
  echo built $tag
done
