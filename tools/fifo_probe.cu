// Does tcgen05.st (+ wait::st) from one warp wait behind tcgen05.mma queued by
// another warp?  Latency of STTM.x8 + wait::st alone vs. right after 64 MMAs
// (M128 N64 K8 tf32, A in TMEM) were issued by warp 0.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/fifo_probe tools/fifo_probe.cu
#include <cstdio>
#include "../paper_2407_21637_b200/csrc/async.cuh"
#include "../paper_2407_21637_b200/csrc/tc.cuh"
using namespace hodlr;

__global__ void k(long long* out, int nmma) {
    __shared__ __align__(1024) float sB[64 * 32];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    __shared__ volatile int go;
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) sB[i] = 0.5f;
    if (warp == 0) tc::tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) { tma::mbar_init(&bar, 1); tma::fence_mbar_init(); go = 0; }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t idesc = tc::idesc_tf32(128, 64);
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t bd = tc::smem_desc(tc::smem_u32(sB), 1024, 128);
            long long t0 = clock64();
            for (int r = 0; r < nmma; ++r) tc::mma_tf32_ts(tb, tb + 128, bd, idesc, 1);
            long long t1 = clock64();
            go = 1;
            tc::commit(&bar);
            tma::mbar_wait(&bar, 0);
            out[0] = t1 - t0;             // issue time of the MMAs
            out[1] = clock64() - t0;      // completion
        }
    } else if (warp == 4) {
        while (!go) {}
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) v[i] = i;
        long long t0 = clock64();
        tc::st_x8(tb + 256, v);          // lane quarter 0 (warp 4 % 4 == 0), columns unused by the MMAs
        tc::wait_st();
        long long t1 = clock64();
        if (lane == 0) out[2] = t1 - t0;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tb);
}

int main() {
    long long* d;
    cudaMalloc(&d, 24);
    for (int n : {0, 8, 64, 256}) {
        long long h[3] = {0, 0, 0};
        k<<<1, 256>>>(d, n);
        cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
        printf("MMAs queued %3d: issue %6lld cyc, complete %6lld cyc | STTM+wait::st after them: %6lld cyc (%s)\n", n,
               h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
