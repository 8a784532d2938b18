#!/bin/bash
# Instrumented build (HODLR_TRACE): per-CTA %globaltimer stamps of the fused kernel.
set -e
cd "$(dirname "$0")/../paper_2407_21637_b200/csrc"
make -s
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
     -DHODLR_TRACE ${EXTRA:-} -c kernels_sv.cu -o build/kernels_sv_trace.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/libhodlr_b200_trace.so \
     build/capi.o build/kernels_generic.o build/kernels_shard.o build/kernels_mrhs.o build/kernels_tc.o build/kernels_sv_trace.o -cudart static
echo built tools/libhodlr_b200_trace.so
