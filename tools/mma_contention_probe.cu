// tcgen05 kind::tf32 M128 N64 K8 (A in TMEM) issue rate alone vs. with 8 warps
// streaming tcgen05.st into other TMEM columns, and with 8 warps streaming
// shared-memory stores (B-operand-like traffic).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_contention_probe tools/mma_contention_probe.cu
#include <cstdio>
#include "../paper_2407_21637_b200/csrc/async.cuh"
#include "../paper_2407_21637_b200/csrc/tc.cuh"
using namespace hodlr;

__global__ void k(long long* out, int reps, int mode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    __shared__ volatile int done;
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    float* sB = (float*)sm;  // 64 x 32 K-major
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) sB[i] = 0.5f;
    if (warp == 0) tc::tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) { tma::mbar_init(&bar, 1); tma::fence_mbar_init(); done = 0; }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t idesc = tc::idesc_tf32(128, 64);
    if (warp == 0) {
        if (lane == 0) {
            uint64_t bd[4];
            for (int ks = 0; ks < 4; ++ks) bd[ks] = tc::smem_desc(tc::smem_u32(sB) + ks * 2 * 1024, 1024, 128);
            long long t0 = clock64();
            for (int r = 0; r < reps; ++r) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
#pragma unroll
                    for (int m = 0; m < 2; ++m) tc::mma_tf32_ts(tb + m * 64, tb + 128 + m * 64 + ks * 8, bd[ks], idesc, 1);
            }
            tc::commit(&bar);
            tma::mbar_wait(&bar, 0);
            out[0] = clock64() - t0;
            done = 1;
        }
    } else if (mode == 1 && warp >= 8) {
        // 8 warps: tcgen05.st into columns 256..511 (quarter = warp % 4)
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) v[i] = i;
        const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + 256 + ((warp >> 2) & 1) * 128;
        while (!done) {
            for (int c = 0; c < 128; c += 8) tc::st_x8(base + c, v);
            tc::wait_st();
        }
    } else if (mode == 2 && warp >= 8) {
        uint4* p = (uint4*)(sm + 16384);
        while (!done) {
            for (int i = 0; i < 16; ++i) p[(warp - 8) * 512 + i * 32 + lane] = make_uint4(i, 1, 2, 3);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tb);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 8 * 8192);
    const char* names[] = {"alone", "with 8 warps tcgen05.st", "with 8 warps st.shared"};
    for (int mode = 0; mode < 3; ++mode) {
        int reps = 1024;
        k<<<1, 16 * 32, 16384 + 8 * 8192>>>(d, reps, mode);
        long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %.1f cycles/MMA (%s)\n", names[mode], (double)c / (reps * 8), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
