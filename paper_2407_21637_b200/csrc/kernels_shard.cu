// External-level kernels of the sharded matvec.
//
// With nranks = 2^L, rank g owns level-L node g: levels L+1..l (its subtree)
// and its leaves need nothing from other ranks; levels 1..L ("external") need
// the V'^T x coefficients of the sibling subtrees, which live on other ranks.
// Per matvec:
//   k_ext_v   send[slot_k + c] = V'_k[own rows, c]^T x_own      (before the all-gather)
//   (all-gather of send over NVLink by the caller, overlapped with the subtree)
//   k_gen_reduce_ext  t_k = sum over the sibling ranks of recv, in rank order
//   k_ext_u   b_own += U_k[own rows] t_k, k = 1..L                (after the all-gather)
// Only the external factors' row slices are read here (a few MB); the subtree
// runs in the single-vector fused kernel or the generic kernels.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace hodlr {

namespace {

constexpr int kExtThreads = 256;
constexpr int kExtRowsV = 1024;  // rows per block of k_ext_v
constexpr int kExtWarps = kExtThreads / 32;

// Partial V'^T x of every external level over this block's rows, then the
// last block to finish sums the per-block partials in block order
// (deterministic) into send.  Slot padding (columns rv..rmax of a level) is 0.
template <typename W, int SB>
__global__ void __launch_bounds__(kExtThreads)
    k_ext_v(PlanView p, const W* __restrict__ x, int64_t ldx, int64_t s, W* __restrict__ scratch,
            unsigned* __restrict__ ticket, W* __restrict__ send) {
    __shared__ W red[kExtWarps][SB];
    __shared__ bool is_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t cnt = p.ext_count * s;
    const int r0 = blockIdx.x * kExtRowsV;
    const int r1 = min(p.n_local, r0 + kExtRowsV);
    W* mine = scratch + (int64_t)blockIdx.x * cnt;
    for (int64_t i = threadIdx.x; i < cnt; i += kExtThreads) mine[i] = W(0);
    __syncthreads();
    for (int e = 0; e < p.next; ++e) {  // external nodes are node ids 0..L-1 (levels 1..L)
        const NodeDesc nd = p.nodes[e];
        const int fb = fmt_bytes(nd.v_fmt);
        for (int c = 0; c < nd.rv; ++c) {
            const uint8_t* col = p.arena + nd.v_off + (int64_t)c * nd.v_ld * fb;
            for (int64_t q0 = 0; q0 < s; q0 += SB) {
                const int nq = (int)min((int64_t)SB, s - q0);
                W acc[SB];
#pragma unroll
                for (int q = 0; q < SB; ++q) acc[q] = W(0);
                for (int r = r0 + threadIdx.x; r < r1; r += kExtThreads) {
                    const W* xr = x + (int64_t)r * ldx + q0;
#pragma unroll
                    for (int q = 0; q < SB; ++q)
                        if (q < nq) acc[q] = mac<W>(nd.v_fmt, col, r - nd.row0, xr[q], acc[q]);
                }
#pragma unroll
                for (int q = 0; q < SB; ++q) {
                    const W v = warp_sum(acc[q]);
                    if (lane == 0) red[warp][q] = v;
                }
                __syncthreads();
                if (threadIdx.x < nq) {
                    W t = red[0][threadIdx.x];
#pragma unroll
                    for (int w = 1; w < kExtWarps; ++w) t += red[w][threadIdx.x];
                    mine[((int64_t)nd.ext_slot + c) * s + q0 + threadIdx.x] = t;
                }
                __syncthreads();
            }
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    for (int64_t i = threadIdx.x; i < cnt; i += kExtThreads) {
        W t = __ldcg(scratch + i);
        for (unsigned blk = 1; blk < gridDim.x; ++blk) t += __ldcg(scratch + (int64_t)blk * cnt + i);
        send[i] = t;
    }
    if (threadIdx.x == 0) *ticket = 0u;  // ready for the next call (stream-ordered)
}

// b_own += U_k t_k for the external levels k = 1..L, in level order, each
// level's U t formed separately and then added (Alg. 3).
template <typename W, int SB>
__global__ void __launch_bounds__(kExtThreads)
    k_ext_u(PlanView p, const W* __restrict__ tbuf, W* __restrict__ b, int64_t ldb, int64_t s) {
    const int r = blockIdx.x * kExtThreads + threadIdx.x;
    if (r >= p.n_local) return;
    for (int64_t q0 = 0; q0 < s; q0 += SB) {
        const int nq = (int)min((int64_t)SB, s - q0);
        W acc[SB];
#pragma unroll
        for (int q = 0; q < SB; ++q)
            if (q < nq) acc[q] = b[(int64_t)r * ldb + q0 + q];
        for (int e = 0; e < p.next; ++e) {
            const NodeDesc nd = p.nodes[e];
            const W* t = tbuf + nd.tsrc_off * s + q0;
            const int fb = fmt_bytes(nd.u_fmt);
            W ut[SB];
#pragma unroll
            for (int q = 0; q < SB; ++q) ut[q] = W(0);
            for (int c = 0; c < nd.ru; ++c) {
                const uint8_t* col = p.arena + nd.u_off + (int64_t)c * nd.u_ld * fb;
#pragma unroll
                for (int q = 0; q < SB; ++q)
                    if (q < nq) ut[q] = mac<W>(nd.u_fmt, col, r - nd.row0, t[(int64_t)c * s + q], ut[q]);
            }
#pragma unroll
            for (int q = 0; q < SB; ++q) acc[q] += ut[q];
        }
#pragma unroll
        for (int q = 0; q < SB; ++q)
            if (q < nq) b[(int64_t)r * ldb + q0 + q] = acc[q];
    }
}

}  // namespace

int ext_v_blocks(int64_t n_local) { return (int)((n_local + kExtRowsV - 1) / kExtRowsV); }

template <typename W>
cudaError_t ext_begin(const PlanView& p, const W* x, int64_t ldx, int64_t s, W* scratch, unsigned* ticket,
                      W* send, cudaStream_t st) {
    if (p.next == 0 || p.n_local == 0) return cudaSuccess;
    const int grid = ext_v_blocks(p.n_local);
    if (s == 1)
        k_ext_v<W, 1><<<grid, kExtThreads, 0, st>>>(p, x, ldx, s, scratch, ticket, send);
    else
        k_ext_v<W, 8><<<grid, kExtThreads, 0, st>>>(p, x, ldx, s, scratch, ticket, send);
    return cudaGetLastError();
}

template <typename W>
cudaError_t ext_finish(const PlanView& p, int64_t s, const W* recv, W* tbuf, W* b, int64_t ldb,
                       cudaStream_t st) {
    if (p.next == 0 || p.n_local == 0) return cudaSuccess;
    cudaError_t e = gen_ext<W>(p, s, recv, tbuf, st);
    if (e != cudaSuccess) return e;
    const int grid = (p.n_local + kExtThreads - 1) / kExtThreads;
    if (s == 1)
        k_ext_u<W, 1><<<grid, kExtThreads, 0, st>>>(p, tbuf, b, ldb, s);
    else
        k_ext_u<W, 8><<<grid, kExtThreads, 0, st>>>(p, tbuf, b, ldb, s);
    return cudaGetLastError();
}

template cudaError_t ext_begin<double>(const PlanView&, const double*, int64_t, int64_t, double*, unsigned*,
                                       double*, cudaStream_t);
template cudaError_t ext_begin<float>(const PlanView&, const float*, int64_t, int64_t, float*, unsigned*, float*,
                                      cudaStream_t);
template cudaError_t ext_finish<double>(const PlanView&, int64_t, const double*, double*, double*, int64_t,
                                        cudaStream_t);
template cudaError_t ext_finish<float>(const PlanView&, int64_t, const float*, float*, float*, int64_t,
                                       cudaStream_t);

}  // namespace hodlr
