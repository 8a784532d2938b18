#!/bin/bash
# Build tools/variants/libhodlr_tctrace.so: the library with -DHODLR_TC_TRACE in kernels_tc.cu
# (per-item clock traces of CTA 0); run with HODLR_B200_LIB=$PWD/tools/variants/libhodlr_tctrace.so.
set -e
cd "$(dirname "$0")/../paper_2407_21637_b200/csrc"
make >/dev/null
mkdir -p ../../tools/variants
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
     ${TRACE_FLAGS:--DHODLR_TC_TRACE} -c kernels_tc.cu -o /tmp/kernels_tc_trace.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/libhodlr_tctrace.so \
     build/capi.o build/kernels_generic.o build/kernels_seq.o build/kernels_sv.o build/kernels_shard.o \
     build/kernels_mrhs.o build/kernels_sv_g1.o /tmp/kernels_tc_trace.o -cudart static
