// Dependent-chain latency of DFMA, F2F.F64.F32 and LDS on sm_100a (one warp).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, float seed, int n) {
    __shared__ double sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x * 1e-3;
    __syncthreads();
    double acc = seed;
    float f = seed;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc = fma(acc, 1.0000001, 0.5);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) { acc = fma((double)f, 1.0000001, acc); f = (float)acc; }
    long long t2 = clock64();
    int idx = (int)seed;
    for (int i = 0; i < n; ++i) { double v = sm[idx & 63]; idx = (int)v + i; acc += v; }
    long long t3 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
    out[threadIdx.x] = acc + f;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 3 * 8);
    const int n = 4096;
    lat<<<1, 32>>>(out, cyc, 1.0f, n);
    long long h[3];
    cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
    printf("DFMA chain latency          %.1f cycles\n", (double)h[0] / n);
    printf("F2F.F64.F32 + DFMA + F2F.F32.F64 chain %.1f cycles\n", (double)h[1] / n);
    printf("LDS.64 + F2I + DADD chain   %.1f cycles\n", (double)h[2] / n);
    return 0;
}
