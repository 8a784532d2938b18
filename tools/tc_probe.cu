// Probe of the tcgen05 kind::tf32 conventions used by the tensor-core
// multi-RHS kernels (tc.cuh): A in TMEM (TS) and in shared memory (SS),
// K-major no-swizzle B descriptors, operand rounding mode, and MMA throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2407_21637_b200/csrc/async.cuh"
#include "../paper_2407_21637_b200/csrc/tc.cuh"

using namespace hodlr;

constexpr int M = 128, N = 64, K = 32;  // 4 k-steps of 8

// B (N x K) element (n, k) in the K-major no-swizzle layout [kc][ng][8][4]
__host__ __device__ inline int b_off(int n, int k) { return (k / 4) * (N / 8) * 32 + (n / 8) * 32 + (n % 8) * 4 + k % 4; }
// A (M x K) element (m, k), same layout with M rows
__host__ __device__ inline int a_off(int m, int k) { return (k / 4) * (M / 8) * 32 + (m / 8) * 32 + (m % 8) * 4 + k % 4; }

template <int mode>
__global__ void k_probe(const float* A, const float* B, float* D_ts, float* D_ss, long long* cyc,
                        int reps) {
    __shared__ __align__(1024) float sB[N * K];
    __shared__ __align__(1024) float sA[M * K];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < N * K; i += blockDim.x) {
        int n = i / K, k = i % K;
        sB[b_off(n, k)] = B[i];
    }
    for (int i = tid; i < M * K; i += blockDim.x) {
        int m = i / K, k = i % K;
        sA[a_off(m, k)] = A[i];
    }
    if (warp == 0) tc::tmem_alloc<512>(&tbase);
    if (tid == 0) {
        tma::mbar_init(&bar, 1);
        tma::fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    uint32_t tb = tbase;
    // A -> TMEM columns [128, 128 + K): warp w writes lanes 32w..32w+31 (row = lane)
    {
        int row = warp * 32 + lane;
        for (int c = 0; c < K; c += 8) {
            uint32_t v[8];
            for (int j = 0; j < 8; ++j) v[j] = __float_as_uint(A[row * K + c + j]);
            tc::st_x8(tb + ((uint32_t)(warp * 32) << 16) + 128 + c, v);
        }
        tc::wait_st();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t idesc = tc::idesc_tf32(M, N);
    if (tid == 0) {
        uint64_t bd[4], ad[4];
        for (int ks = 0; ks < 4; ++ks) {
            bd[ks] = tc::smem_desc(tc::smem_u32(sB) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
            ad[ks] = tc::smem_desc(tc::smem_u32(sA) + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
        }
        constexpr int NN = mode == 3 ? 128 : mode == 4 ? 256 : mode == 5 ? 32 : 64;
        constexpr uint32_t id = tc::idesc_tf32(M, NN);
        long long t0 = clock64();
        tc::mma_tf32_ts(tb + 0, tb + 128, bd[0], id, 0);
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                if (mode == 1)
                    tc::mma_tf32_ss(tb + 0, ad[ks], bd[ks], id, 1);
                else if (mode == 2)
                    tc::mma_tf32_ts(tb + (ks & 1) * 64, tb + 128 + ks * 8, bd[ks], id, 1);
                else if (mode == 5)
                    tc::mma_tf32_ts(tb + (ks & 3) * 32, tb + 128 + ks * 8, bd[ks], id, 1);
                else
                    tc::mma_tf32_ts(tb + (mode == 4 ? 256 : 0), tb + 128 + ks * 8, bd[ks], id, 1);
            }
        }
        tc::commit(&bar);
        tma::mbar_wait(&bar, 0);
        long long t1 = clock64();
        *cyc = t1 - t0;
    }
    __syncthreads();
    tc::fence_after();
    {
        int row = warp * 32 + lane;
        float* D = mode == 0 ? D_ts : D_ss;
        for (int c = 0; c < N; c += 16) {
            uint32_t v[16];
            tc::ld_x16(tb + ((uint32_t)(warp * 32) << 16) + c, v);
            tc::wait_ld();
            for (int j = 0; j < 16; ++j) D[row * N + c + j] = __uint_as_float(v[j]);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tb);
}

static float trunc_tf32(float a) {
    uint32_t u;
    memcpy(&u, &a, 4);
    u &= 0xFFFFE000u;
    memcpy(&a, &u, 4);
    return a;
}
static float rn_tf32(float a) {
    uint32_t u;
    memcpy(&u, &a, 4);
    uint32_t lsb = (u >> 13) & 1;
    u = (u + 0xFFF + lsb) & 0xFFFFE000u;
    memcpy(&a, &u, 4);
    return a;
}
static float rna_tf32(float a) {
    uint32_t u;
    memcpy(&u, &a, 4);
    u = (u + 0x1000) & 0xFFFFE000u;
    memcpy(&a, &u, 4);
    return a;
}

int main() {
    std::vector<float> A(M * K), B(N * K), Dts(M * N), Dss(M * N);
    srand(1);
    auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
    for (auto& a : A) a = rnd();
    for (auto& b : B) b = rnd();
    float *dA, *dB, *dD1, *dD2;
    long long* dc;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD1, Dts.size() * 4);
    cudaMalloc(&dD2, Dss.size() * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
        if (mode == 0) k_probe<0><<<1, 128>>>(dA, dB, dD1, dD2, dc, 1); else k_probe<1><<<1, 128>>>(dA, dB, dD1, dD2, dc, 1);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("mode %d error %s\n", mode, cudaGetErrorString(e));
            return 1;
        }
    }
    cudaMemcpy(Dts.data(), dD1, Dts.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(Dss.data(), dD2, Dss.size() * 4, cudaMemcpyDeviceToHost);
    double e_tr[2] = {0, 0}, e_rn[2] = {0, 0}, e_rna[2] = {0, 0}, e_ex[2] = {0, 0}, mx = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s_tr = 0, s_rn = 0, s_rna = 0, s_ex = 0;
            for (int k = 0; k < K; ++k) {
                s_tr += (double)trunc_tf32(A[m * K + k]) * trunc_tf32(B[n * K + k]);
                s_rn += (double)rn_tf32(A[m * K + k]) * rn_tf32(B[n * K + k]);
                s_rna += (double)rna_tf32(A[m * K + k]) * rna_tf32(B[n * K + k]);
                s_ex += (double)A[m * K + k] * B[n * K + k];
            }
            for (int md = 0; md < 2; ++md) {
                double d = md == 0 ? Dts[m * N + n] : Dss[m * N + n];
                e_tr[md] = fmax(e_tr[md], fabs(d - s_tr));
                e_rn[md] = fmax(e_rn[md], fabs(d - s_rn));
                e_rna[md] = fmax(e_rna[md], fabs(d - s_rna));
                e_ex[md] = fmax(e_ex[md], fabs(d - s_ex));
            }
            mx = fmax(mx, fabs(s_ex));
        }
    for (int md = 0; md < 2; ++md)
        printf("%s: max|D - ref| trunc %.3e  rn %.3e  rna %.3e  exact-fp32 %.3e  (max|D| %.2f)\n",
               md == 0 ? "TS" : "SS", e_tr[md], e_rn[md], e_rna[md], e_ex[md], mx);
    // throughput: reps x 4 MMAs of 128x64x8
    const char* names[] = {"TS N64 chained", "SS N64 chained", "TS N64 2 accs", "TS N128", "TS N256", "TS N32 4 accs"};
    const int ns[] = {64, 64, 64, 128, 256, 32};
    for (int mode = 0; mode < 6; ++mode) {
        int reps = 2048;
        switch (mode) {
            case 0: k_probe<0><<<1, 128>>>(dA, dB, dD1, dD2, dc, reps); break;
            case 1: k_probe<1><<<1, 128>>>(dA, dB, dD1, dD2, dc, reps); break;
            case 2: k_probe<2><<<1, 128>>>(dA, dB, dD1, dD2, dc, reps); break;
            case 3: k_probe<3><<<1, 128>>>(dA, dB, dD1, dD2, dc, reps); break;
            case 4: k_probe<4><<<1, 128>>>(dA, dB, dD1, dD2, dc, reps); break;
            default: k_probe<5><<<1, 128>>>(dA, dB, dD1, dD2, dc, reps); break;
        }
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("%s: %d MMAs (M128 K8 tf32) in %lld cycles: %.1f cycles/MMA, %.0f flop/cycle/SM\n",
               names[mode], reps * 4, c, (double)c / (reps * 4), 2.0 * M * ns[mode] * 8 * reps * 4 / c);
    }
    return 0;
}
