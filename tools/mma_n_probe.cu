// tcgen05 kind::tf32 M128 K8 (A in TMEM) chained issue cost for N = 64 / 128 / 256.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_n_probe tools/mma_n_probe.cu
#include <cstdio>
#include "../paper_2407_21637_b200/csrc/async.cuh"
#include "../paper_2407_21637_b200/csrc/tc.cuh"
using namespace hodlr;

template <int N>
__global__ void k(long long* out, int reps) {
    __shared__ __align__(1024) float sB[256 * 8];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) sB[i] = 0.5f;
    if (warp == 0) tc::tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) { tma::mbar_init(&bar, 1); tma::fence_mbar_init(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x == 0) {
        const uint64_t bd = tc::smem_desc(tc::smem_u32(sB), (N / 8) * 128, 128);
        constexpr uint32_t id = tc::idesc_tf32(128, N);
        const uint32_t d = tb + (N == 256 ? 256 : 0), a = tb + (N == 256 ? 0 : 256);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) tc::mma_tf32_ts(d, a, bd, id, 1);
        tc::commit(&bar);
        tma::mbar_wait(&bar, 0);
        out[0] = clock64() - t0;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tb);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    long long c;
    k<64><<<1, 128>>>(d, 2048); cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("N=64 : %.1f cyc/MMA (%s)\n", c / 2048.0, cudaGetErrorString(cudaGetLastError()));
    k<128><<<1, 128>>>(d, 2048); cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("N=128: %.1f cyc/MMA (%s)\n", c / 2048.0, cudaGetErrorString(cudaGetLastError()));
    k<256><<<1, 128>>>(d, 2048); cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("N=256: %.1f cyc/MMA (%s)\n", c / 2048.0, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
