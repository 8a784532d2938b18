// Kernel launchers (internal to the .so).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "plan.h"

namespace hodlr {

cudaError_t launch_quantize(int fmt, const double* src, void* dst, int64_t count, cudaStream_t st);
cudaError_t launch_dequantize(int fmt, const void* src, double* dst, int64_t count,
                              cudaStream_t st);
template <typename W>
cudaError_t launch_round_in(const double* x, W* xw, int64_t rows, int64_t s, int64_t ldin,
                            int64_t ldout, cudaStream_t st);
template <typename W>
cudaError_t launch_widen_out(const W* bw, double* b, int64_t rows, int64_t s, int64_t ldin,
                             int64_t ldout, cudaStream_t st);

// Generic path (any s / alignment).
template <typename W>
cudaError_t gen_begin(const PlanView& p, const W* x, int64_t ldx, int64_t s, W* partial, W* tbuf,
                      W* send, cudaStream_t st);
template <typename W>
cudaError_t gen_ext(const PlanView& p, int64_t s, const W* recv, W* tbuf, cudaStream_t st);
template <typename W>
cudaError_t gen_end(const PlanView& p, const W* x, int64_t ldx, const W* tbuf, W* b, int64_t ldb,
                    int64_t s, int max_chunk_rows, cudaStream_t st);

// Strict-order path (kernels_seq.cu): the reference's per-operation rounding in
// any working format, bit-identical to arithmetic.py; binary64 carriers.
cudaError_t seq_round(int fmt, const double* src, double* dst, int64_t rows, int64_t s, int64_t ldin, int64_t ldout,
                      cudaStream_t st);
cudaError_t seq_matvec(int fmt, const PlanView& p, const double* x, int64_t ldx, double* b, int64_t ldb, int64_t s,
                       double* tbuf, cudaStream_t st);

// Sharded path, external levels (kernels_shard.cu).
int ext_v_blocks(int64_t n_local);
template <typename W>
cudaError_t ext_begin(const PlanView& p, const W* x, int64_t ldx, int64_t s, W* scratch, unsigned* ticket,
                      W* send, cudaStream_t st);
template <typename W>
cudaError_t ext_finish(const PlanView& p, int64_t s, const W* recv, W* tbuf, W* b, int64_t ldb,
                       cudaStream_t st);

}  // namespace hodlr
