// Throughput of tcgen05.st (registers -> TMEM) by shape, 4/8/16 warps storing
// disjoint columns, with a tcgen05.wait::st every `batch` stores.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/sttm_probe tools/sttm_probe.cu
#include <cstdio>
#include "../paper_2407_21637_b200/csrc/tc.cuh"
using namespace hodlr;

template <int X>
__device__ __forceinline__ void st_n(uint32_t taddr, const uint32_t* v);
template <>
__device__ __forceinline__ void st_n<8>(uint32_t a, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}
template <>
__device__ __forceinline__ void st_n<32>(uint32_t a, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

template <int X>
__global__ void k(long long* out, int iters, int batch) {
    __shared__ uint32_t tb;
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) tc::tmem_alloc<512>(&tb);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int nw = blockDim.x / 32;
    const int per_q = nw / 4;                  // warps per lane quarter
    const int cols = 512 / per_q;              // columns owned by this warp
    const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * cols;
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = lane * 32 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < cols; c += X) {
            st_n<X>(base + c, v);
        }
        if ((it + 1) % batch == 0) tc::wait_st();
    }
    tc::wait_st();
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tb);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    for (int nw : {4, 8, 16}) {
        for (int batch : {1, 4}) {
            long long c8, c32;
            int iters = 64;
            k<8><<<1, nw * 32>>>(d, iters, batch);
            cudaMemcpy(&c8, d, 8, cudaMemcpyDeviceToHost);
            k<32><<<1, nw * 32>>>(d, iters, batch);
            cudaMemcpy(&c32, d, 8, cudaMemcpyDeviceToHost);
            double bytes = 128.0 * 512 * 4 * iters;  // whole TMEM per iteration
            printf("warps %2d wait every %d sweeps: x8 %.1f B/cyc  x32 %.1f B/cyc  (%s)\n", nw, batch, bytes / c8,
                   bytes / c32, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
