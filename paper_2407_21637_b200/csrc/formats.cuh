// Storage formats of the adaptive-precision HODLR (fpsim.py:110-114) and their
// exact conversions, compiled for both host and sm_100a.
//
// Encode (K0, store_factor -> round_matrix, lowrank.py:117-119, fpsim.py:160-185):
//   RNE from binary64 straight to the narrow format, one rounding, overflow -> inf,
//   subnormals kept.  On sm_100a these are single cvt.rn.{f16,bf16,f32}.f64 / the
//   e5m2 cvt; NOT via an fp32 intermediate (torch/ml_dtypes casts double-round).
// Decode: exact widening (every narrow value is a binary64 / binary32 value):
//   e5m2 byte b is the high byte of the binary16 with the same value (<< 8),
//   bf16 is the high half of the binary32 (<< 16), fp16 -> fp32 is exact.
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "../../include/hodlr_b200.h"

namespace hodlr {

constexpr int kNumFormats = 5;

__host__ __device__ inline int fmt_bytes(int fmt) {
    return fmt == HODLR_FMT_Q52 ? 1 : fmt == HODLR_FMT_FP32 ? 4 : fmt == HODLR_FMT_FP64 ? 8 : 2;
}

// ---- encode (binary64 -> narrow bits), bit-exact RNE ----
__host__ __device__ inline uint8_t enc_q52(double x) {
    return (uint8_t)__nv_cvt_double_to_fp8(x, __NV_NOSAT, __NV_E5M2);
}
__host__ __device__ inline uint16_t enc_bf16(double x) {
    __nv_bfloat16 h = __double2bfloat16(x);
    return *reinterpret_cast<uint16_t*>(&h);
}
__host__ __device__ inline uint16_t enc_fp16(double x) {
    __half h = __double2half(x);
    return *reinterpret_cast<uint16_t*>(&h);
}
__host__ __device__ inline float enc_fp32(double x) {
#ifdef __CUDA_ARCH__
    return __double2float_rn(x);
#else
    return (float)x;  // IEEE RNE on the host (default rounding mode)
#endif
}

// ---- decode (narrow bits -> float / double), exact ----
__host__ __device__ inline float dec_fp16_bits(uint16_t b) {
    __half_raw r; r.x = b;
    return __half2float(__half(r));
}
__host__ __device__ inline float dec_q52(uint8_t b) { return dec_fp16_bits((uint16_t)(b) << 8); }
__host__ __device__ inline float dec_bf16(uint16_t b) {
#ifdef __CUDA_ARCH__
    return __uint_as_float((uint32_t)b << 16);
#else
    uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f;
#endif
}
__host__ __device__ inline float dec_fp16(uint16_t b) { return dec_fp16_bits(b); }

// Decode element i of a narrow array as double.
__host__ __device__ inline double dec_any(int fmt, const void* p, int64_t i) {
    switch (fmt) {
        case HODLR_FMT_Q52: return (double)dec_q52(((const uint8_t*)p)[i]);
        case HODLR_FMT_BF16: return (double)dec_bf16(((const uint16_t*)p)[i]);
        case HODLR_FMT_FP16: return (double)dec_fp16(((const uint16_t*)p)[i]);
        case HODLR_FMT_FP32: return (double)((const float*)p)[i];
        default: return ((const double*)p)[i];
    }
}
__host__ __device__ inline void enc_any(int fmt, double x, void* p, int64_t i) {
    switch (fmt) {
        case HODLR_FMT_Q52: ((uint8_t*)p)[i] = enc_q52(x); break;
        case HODLR_FMT_BF16: ((uint16_t*)p)[i] = enc_bf16(x); break;
        case HODLR_FMT_FP16: ((uint16_t*)p)[i] = enc_fp16(x); break;
        case HODLR_FMT_FP32: ((float*)p)[i] = enc_fp32(x); break;
        default: ((double*)p)[i] = x; break;
    }
}

}  // namespace hodlr
