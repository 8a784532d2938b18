// Isolated timing of the fused kernel's phase-A inner loop (a_rows) and the
// D-block loop (col_block) on shared-memory data, plus candidate rewrites.
#include "../paper_2407_21637_b200/csrc/kernels_sv.cu"

namespace hodlr {
namespace {
// candidate: rows processed 4 at a time, loads first, clamped lane address
// instead of a branch (inactive lanes read a valid address, result unused)
template <typename W>
__device__ __forceinline__ void a_rows_v1(const uint8_t* rows, int nrows, int vpad, const W* xs, int warp, int lane,
                                          W acc[2][4]) {
    const int nq = vpad >> 2;
    const int row_bytes = vpad * 4;
    const bool act0 = lane < nq, act1 = lane + 32 < nq;
    const int q0 = act0 ? lane : 0, q1 = act1 ? lane + 32 : 0;
    int j = warp;
    for (; j + 3 * kConsumers < nrows; j += 4 * kConsumers) {
        float4 v0[4], v1[4];
        W xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint8_t* row = rows + (size_t)(j + u * kConsumers) * row_bytes;
            xv[u] = xs[j + u * kConsumers];
            v0[u] = *reinterpret_cast<const float4*>(row + q0 * 16);
            if (act1) v1[u] = *reinterpret_cast<const float4*>(row + q1 * 16);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (act0) {
                acc[0][0] = fma((W)v0[u].x, xv[u], acc[0][0]);
                acc[0][1] = fma((W)v0[u].y, xv[u], acc[0][1]);
                acc[0][2] = fma((W)v0[u].z, xv[u], acc[0][2]);
                acc[0][3] = fma((W)v0[u].w, xv[u], acc[0][3]);
            }
            if (act1) {
                acc[1][0] = fma((W)v1[u].x, xv[u], acc[1][0]);
                acc[1][1] = fma((W)v1[u].y, xv[u], acc[1][1]);
                acc[1][2] = fma((W)v1[u].z, xv[u], acc[1][2]);
                acc[1][3] = fma((W)v1[u].w, xv[u], acc[1][3]);
            }
        }
    }
    for (; j < nrows; j += kConsumers) {
        const uint8_t* row = rows + (size_t)j * row_bytes;
        const W x1 = xs[j];
        if (act0) {
            const float4 t = *reinterpret_cast<const float4*>(row + q0 * 16);
            acc[0][0] = fma((W)t.x, x1, acc[0][0]); acc[0][1] = fma((W)t.y, x1, acc[0][1]);
            acc[0][2] = fma((W)t.z, x1, acc[0][2]); acc[0][3] = fma((W)t.w, x1, acc[0][3]);
        }
        if (act1) {
            const float4 t = *reinterpret_cast<const float4*>(row + q1 * 16);
            acc[1][0] = fma((W)t.x, x1, acc[1][0]); acc[1][1] = fma((W)t.y, x1, acc[1][1]);
            acc[1][2] = fma((W)t.z, x1, acc[1][2]); acc[1][3] = fma((W)t.w, x1, acc[1][3]);
        }
    }
}

__global__ void bench_a(long long* cyc, double* out, int reps) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 33280 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1e-3f * (i & 255);
    __syncthreads();
    double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
        a_rows<HODLR_FMT_FP32, double>(sm + 2048, 64, 112, reinterpret_cast<const double*>(sm), warp, lane, acc);
    long long t1 = clock64();
    double bacc[4][kRPL] = {};
    const double* xs = reinterpret_cast<const double*>(sm);
    auto mul = [&](int c) { return xs[c]; };
    for (int r = 0; r < reps; ++r) col_block<HODLR_FMT_FP64, double>(sm + 512, 64, warp, lane, mul, bacc);
    long long t2 = clock64();
    for (int r = 0; r < reps; ++r)
        a_rows_v1<double>(sm + 2048, 64, 112, reinterpret_cast<const double*>(sm), warp, lane, acc);
    long long t3 = clock64();
    // U-like: 104 fp32 columns, multiplier via a column -> coefficient slot table
    __shared__ int16_t ci_tab[128];
    if (threadIdx.x < 128) ci_tab[threadIdx.x] = (int16_t)((threadIdx.x * 7) & 127);
    __syncthreads();
    const double* coef = reinterpret_cast<const double*>(sm + 30000);
    auto mulu = [&](int c) { return coef[ci_tab[c]]; };
    long long t4 = clock64();
    for (int r = 0; r < reps; ++r) col_block<HODLR_FMT_FP32, double>(sm + 1024, 104, warp, lane, mulu, bacc);
    long long t5 = clock64();
    auto mulx = [&](int c) { return xs[c]; };
    for (int r = 0; r < reps; ++r) col_block<HODLR_FMT_FP32, double>(sm + 1024, 104, warp, lane, mulx, bacc);
    long long t6 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t5 - t4; cyc[4] = t6 - t5; }
    double s = 0;
    for (int i = 0; i < 2; ++i) for (int e = 0; e < 4; ++e) s += acc[i][e];
    for (int i = 0; i < 4; ++i) for (int e = 0; e < kRPL; ++e) s += bacc[i][e];
    out[threadIdx.x] = s;
}
}  // namespace
}  // namespace hodlr

int main() {
    long long* cyc; double* out;
    cudaMalloc(&cyc, 40); cudaMalloc(&out, 4096 * 8);
    cudaFuncSetAttribute(hodlr::bench_a, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    const int reps = 100;
    for (int w : {8, 16}) {
        hodlr::bench_a<<<1, 32 * w, 40000>>>(cyc, out, reps);
        long long h[5];
        cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
        printf("%2d warps: a_rows %.0f | a_rows_v1 %.0f | D col_block(64 fp64) %.0f | U col_block(104 fp32, cidx) %.0f | "
               "(104 fp32, direct) %.0f  cycles/call\n",
               w, (double)h[0] / reps, (double)h[2] / reps, (double)h[1] / reps, (double)h[3] / reps, (double)h[4] / reps);
    }
    return 0;
}
