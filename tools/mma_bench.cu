// Throughput of the legacy warp-level MMA kinds on this GPU (DMMA f64,
// HMMA tf32, HMMA bf16) and plain DFMA/FFMA, per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

template <int K>
__global__ void k_dmma(double* out, int iters) {
    double c[K][2];
    for (int i = 0; i < K; ++i) c[i][0] = c[i][1] = 0;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < K; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < K; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}
template <int K>
__global__ void k_tf32(float* out, int iters) {
    float c[K][4];
    for (int i = 0; i < K; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
    uint32_t a = 0x3f800000u + threadIdx.x, b = 0x3f000000u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < K; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                         : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3]) : "r"(a), "r"(b));
    }
    float s = 0;
    for (int i = 0; i < K; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.0f) out[0] = s;
}
template <int K>
__global__ void k_bf16(float* out, int iters) {
    float c[K][4];
    for (int i = 0; i < K; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
    uint32_t a = 0x3f803f80u + threadIdx.x, b = 0x3f003f00u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < K; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                         : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3]) : "r"(a), "r"(b));
    }
    float s = 0;
    for (int i = 0; i < K; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.0f) out[0] = s;
}
template <int K>
__global__ void k_dfma(double* out, int iters) {
    double c[K];
    for (int i = 0; i < K; ++i) c[i] = threadIdx.x;
    double a = 1.0000001, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < K; ++i) c[i] = fma(c[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < K; ++i) s += c[i];
    if (s == 12345.0) out[0] = s;
}

template <typename T>
void run(const char* name, void (*kern)(T*, int), void* outv, double flop_per_warp_iter, int warps_per_block) {
    T* out = (T*)outv;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps_per_block);
    kern<<<grid, block>>>(out, 100);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, block>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = flop_per_warp_iter * iters * (double)grid.x * warps_per_block;
    printf("%-28s %8.1f TFLOP/s  (%.2f ms)  err=%s\n", name, flops / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    void* out; cudaMalloc(&out, 64);
    for (int w : {4, 8, 16}) {
        printf("-- %d warps/block, 2 blocks/SM\n", w);
        run("dmma m8n8k4 x8 chains", k_dmma<8>, out, 8 * 2.0 * 8 * 8 * 4, w);
        run("tf32 m16n8k8 x8 chains", k_tf32<8>, out, 8 * 2.0 * 16 * 8 * 8, w);
        run("bf16 m16n8k16 x8 chains", k_bf16<8>, out, 8 * 2.0 * 16 * 8 * 16, w);
        run("dfma x8 chains", k_dfma<8>, out, 8 * 2.0 * 32, w);
    }
    return 0;
}
