// Device helpers shared by the matvec kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "formats.cuh"
#include "plan.h"

namespace hodlr {

// One scalar product v*x accumulated into acc in the working type W.
// Narrow storage formats are exact in fp32, so for W=float they are decoded
// to float and fused; an fp64-stored factor under fp32 working is multiplied
// in binary64 and the product rounded once to fp32 (the operand "enters as-is,
// only results are rounded", arithmetic.py:14-21).
template <typename W>
__device__ __forceinline__ W mac(int fmt, const uint8_t* base, int64_t i, W x, W acc);

template <>
__device__ __forceinline__ double mac<double>(int fmt, const uint8_t* base, int64_t i, double x,
                                              double acc) {
    return fma(dec_any(fmt, base, i), x, acc);
}
template <>
__device__ __forceinline__ float mac<float>(int fmt, const uint8_t* base, int64_t i, float x,
                                            float acc) {
    if (fmt == HODLR_FMT_FP64)
        return acc + __double2float_rn(((const double*)base)[i] * (double)x);
    return fmaf((float)dec_any(fmt, base, i), x, acc);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace hodlr
