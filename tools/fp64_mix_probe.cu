// Does the FP64 tensor subpipe (DMMA) share hardware with the FP64 CUDA-core
// pipe (DFMA)?  Half the warps run DMMA chains, the other half DFMA chains;
// compare the combined rate with each alone.  Also: legacy int8 mma.sync
// (IMMA m16n8k32) throughput, the building block of an exact int8 slice
// (Ozaki-style) fp64 product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int K>
__device__ __forceinline__ void dmma_chains(double (&c)[K][2], double a, double b, int iters) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < K; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
}
template <int K>
__device__ __forceinline__ void dfma_chains(double (&c)[K], double a, double b, int iters) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < K; ++i) c[i] = fma(c[i], a, b);
    }
}

// mode 0: all DMMA, 1: all DFMA, 2: even warps DMMA / odd warps DFMA
__global__ void k_mix(double* out, int iters, int mode, int dfma_iters) {
    const int warp = threadIdx.x >> 5;
    double s = 0;
    const bool dm = mode == 0 || (mode == 2 && (warp & 1) == 0);
    if (dm) {
        double c[8][2];
        for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
        dmma_chains<8>(c, threadIdx.x * 1e-3, 1.0 + threadIdx.x * 1e-4, iters);
        for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    } else {
        double c[8];
        for (int i = 0; i < 8; ++i) c[i] = threadIdx.x;
        dfma_chains<8>(c, 1.0000001, 1e-9, dfma_iters);
        for (int i = 0; i < 8; ++i) s += c[i];
    }
    if (s == 12345.0) out[0] = s;
}

template <int K>
__global__ void k_imma(int* out, int iters) {
    int c[K][4];
    for (int i = 0; i < K; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
    uint32_t a = 0x01020304u + threadIdx.x, b = 0x05060708u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < K; ++i)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                         : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3]) : "r"(a), "r"(b));
    }
    int s = 0;
    for (int i = 0; i < K; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345) out[0] = s;
}
template <int K>
__global__ void k_imma_u8(int* out, int iters) {
    int c[K][4];
    for (int i = 0; i < K; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
    uint32_t a = 0x81828384u + threadIdx.x, b = 0x05060708u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < K; ++i)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                         : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3]) : "r"(a), "r"(b));
    }
    int s = 0;
    for (int i = 0; i < K; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345) out[0] = s;
}

int main() {
    void* out;
    cudaMalloc(&out, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    for (int w : {8, 16}) {
        dim3 grid(sms * 2), block(32 * w);
        for (int mode = 0; mode < 3; ++mode) {
            // DFMA warps: 8 chains x 2 flop x 32 lanes per iter = 512 flop/iter;
            // DMMA warps: 8 x 512 = 4096 flop/iter: give DFMA 4x the iterations
            // so both halves take similar time when the pipes are independent
            const int diters = mode == 1 ? iters : iters * 4;
            k_mix<<<grid, block>>>((double*)out, 100, mode, 400);
            cudaEventRecord(a);
            k_mix<<<grid, block>>>((double*)out, iters, mode, diters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double dm_w = mode == 0 ? w : mode == 2 ? w / 2 : 0;
            double df_w = mode == 1 ? w : mode == 2 ? w / 2 : 0;
            double flops = (double)grid.x * (dm_w * iters * 4096.0 + df_w * diters * 512.0);
            printf("%2d warps/blk mode %d (%s): %.1f TFLOP/s fp64 (%.2f ms) %s\n", w, mode,
                   mode == 0 ? "DMMA" : mode == 1 ? "DFMA" : "half DMMA + half DFMA", flops / ms / 1e9, ms,
                   cudaGetErrorString(cudaGetLastError()));
        }
        k_imma<8><<<grid, block>>>((int*)out, 100);
        cudaEventRecord(a);
        k_imma<8><<<grid, block>>>((int*)out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%2d warps/blk IMMA m16n8k32 s8: %.1f TOP/s (%.2f ms) %s\n", w,
               (double)grid.x * w * iters * 8 * 2.0 * 16 * 8 * 32 / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
        k_imma_u8<8><<<grid, block>>>((int*)out, 100);
        cudaEventRecord(a);
        k_imma_u8<8><<<grid, block>>>((int*)out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("%2d warps/blk IMMA m16n8k32 u8.s8: %.1f TOP/s (%.2f ms) %s\n", w,
               (double)grid.x * w * iters * 8 * 2.0 * 16 * 8 * 32 / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
