// Generic (any s, any alignment, any leaf size) matvec kernels and the K0
// quantiser.  These are the layout-agnostic path: three stream-ordered launches
//   A  partial V'^T x per (node, chunk)         -- PAPER.md:524-525 inner products
//   R  fixed-order reduction of partials -> t
//   B  b = sum_k U_k t_k (level order) + D x    -- PAPER.md:524-531
// The single-vector fast path lives in kernels_sv.cu.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace hodlr {

// ------------------------------------------------------------------ K0
__global__ void k_quantize(int fmt, const double* __restrict__ src, void* __restrict__ dst,
                           int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        enc_any(fmt, src[i], dst, i);
}

__global__ void k_dequantize(int fmt, const void* __restrict__ src, double* __restrict__ dst,
                             int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = dec_any(fmt, src, i);
}

// Round x (binary64) into the working type (RNE, like round_matrix to fp32) /
// widen b back to binary64, with leading dimensions.
template <typename W>
__global__ void k_round_in(const double* __restrict__ x, W* __restrict__ xw, int64_t rows,
                           int64_t s, int64_t ldin, int64_t ldout) {
    int64_t total = rows * s;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / s, q = i % s;
        xw[r * ldout + q] = (W)x[r * ldin + q];
    }
}
template <typename W>
__global__ void k_widen_out(const W* __restrict__ bw, double* __restrict__ b, int64_t rows,
                            int64_t s, int64_t ldin, int64_t ldout) {
    int64_t total = rows * s;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / s, q = i % s;
        b[r * ldout + q] = (double)bw[r * ldin + q];
    }
}

// ------------------------------------------------------------------ A
// grid (nchunks, ceil(s/SB)); warp per V' column; lanes stride the chunk rows.
template <typename W, int SB>
__global__ void __launch_bounds__(256) k_gen_phaseA(PlanView p, const W* __restrict__ x,
                                                   int64_t ldx, int64_t s,
                                                   W* __restrict__ partial) {
    const int chunk = blockIdx.x;
    const int q0 = blockIdx.y * SB;
    const int nq = min((int64_t)SB, s - q0);
    const ChunkDesc ch = p.chunks[chunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int lv = 0; lv < p.nlev; ++lv) {
        const NodeDesc nd = p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
        const int off = ch.row0 - nd.row0;
        const int ci = chunk - nd.chunk0;
        for (int c = warp; c < nd.rv; c += nwarp) {
            const uint8_t* col = p.arena + nd.v_off + (int64_t)c * nd.v_ld * fmt_bytes(nd.v_fmt);
            W acc[SB];
#pragma unroll
            for (int q = 0; q < SB; ++q) acc[q] = W(0);
            for (int r = lane; r < ch.nrows; r += 32) {
                const W* xr = x + (int64_t)(ch.row0 + r) * ldx + q0;
#pragma unroll
                for (int q = 0; q < SB; ++q)
                    if (q < nq) acc[q] = mac<W>(nd.v_fmt, col, off + r, xr[q], acc[q]);
            }
#pragma unroll
            for (int q = 0; q < SB; ++q) {
                W v = warp_sum(acc[q]);
                if (lane == 0 && q < nq)
                    partial[nd.part_off * s + ((int64_t)c * s + q0 + q) * nd.nchunk + ci] = v;
            }
        }
    }
}

// ------------------------------------------------------------------ R
// One block per node: coefficient (c, q) = sum over the node's chunks in
// chunk order (deterministic).  External-level nodes write this rank's
// partial into the send buffer instead.
template <typename W>
__global__ void k_gen_reduce(PlanView p, int64_t s, const W* __restrict__ partial,
                             W* __restrict__ tbuf, W* __restrict__ send) {
    const NodeDesc nd = p.nodes[blockIdx.x];
    const int64_t cnt = (int64_t)nd.rv * s;
    W* dst = nd.ext_slot >= 0 ? send + (int64_t)nd.ext_slot * s : tbuf + nd.t_off * s;
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        const W* src = partial + nd.part_off * s + i * nd.nchunk;
        W acc = src[0];
        for (int j = 1; j < nd.nchunk; ++j) acc += src[j];
        dst[i] = acc;
    }
}

// External levels: sum the gathered per-rank partials of the sibling subtree
// in rank order.
template <typename W>
__global__ void k_gen_reduce_ext(PlanView p, int64_t s, const W* __restrict__ recv,
                                 W* __restrict__ tbuf) {
    const ExtDesc e = p.ext[blockIdx.x];
    const int64_t cnt = (int64_t)e.rank * s;
    const int64_t stride = p.ext_count * s;
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        W acc = recv[(int64_t)e.g0 * stride + e.slot * s + i];
        for (int g = e.g0 + 1; g < e.g1; ++g) acc += recv[(int64_t)g * stride + e.slot * s + i];
        tbuf[e.tdst * s + i] = acc;
    }
}

// ------------------------------------------------------------------ B
// grid (nchunks, ceil(s/SB)).  Leaf product first into shared memory (warp per
// row), then per (row, q): levels 1..l in order, each level's U t formed
// separately and added (b <- b + U t), the leaf term added last (Alg. 3 order).
template <typename W, int SB>
__global__ void __launch_bounds__(256) k_gen_phaseB(PlanView p, const W* __restrict__ x,
                                                   int64_t ldx, const W* __restrict__ tbuf,
                                                   W* __restrict__ b, int64_t ldb, int64_t s) {
    extern __shared__ unsigned char smem_raw[];
    W* y = reinterpret_cast<W*>(smem_raw);  // [nrows][SB]
    const int chunk = blockIdx.x;
    const int q0 = blockIdx.y * SB;
    const int nq = min((int64_t)SB, s - q0);
    const ChunkDesc ch = p.chunks[chunk];
    const LeafDesc lf = p.leaves[ch.leaf];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int wb = fmt_bytes(lf.fmt);
    for (int rr = warp; rr < ch.nrows; rr += nwarp) {
        const int lr = ch.row0 + rr - lf.row0;
        const uint8_t* drow = p.arena + lf.off + (int64_t)lr * lf.ld * wb;
        W acc[SB];
#pragma unroll
        for (int q = 0; q < SB; ++q) acc[q] = W(0);
        for (int j = lane; j < lf.m; j += 32) {
            const W* xr = x + (int64_t)(lf.row0 + j) * ldx + q0;
#pragma unroll
            for (int q = 0; q < SB; ++q)
                if (q < nq) acc[q] = mac<W>(lf.fmt, drow, j, xr[q], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < SB; ++q) {
            W v = warp_sum(acc[q]);
            if (lane == 0) y[rr * SB + q] = v;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ch.nrows * nq; i += blockDim.x) {
        const int rr = i / nq, q = i % nq;
        const int row = ch.row0 + rr;
        W bacc = W(0);
        for (int lv = 0; lv < p.nlev; ++lv) {
            const NodeDesc nd = p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
            const uint8_t* ucol = p.arena + nd.u_off;
            const int64_t cstride = (int64_t)nd.u_ld * fmt_bytes(nd.u_fmt);
            const W* t = tbuf + nd.tsrc_off * s + q0 + q;
            W lacc = W(0);
            for (int c = 0; c < nd.ru; ++c)
                lacc = mac<W>(nd.u_fmt, ucol + c * cstride, row - nd.row0, t[(int64_t)c * s], lacc);
            bacc += lacc;
        }
        b[(int64_t)row * ldb + q0 + q] = bacc + y[rr * SB + q];
    }
}

// ------------------------------------------------------------------ launchers
static inline int grid_for(int64_t count) {
    int64_t g = (count + 255) / 256;
    return (int)(g < 148 * 8 ? (g < 1 ? 1 : g) : 148 * 8);
}

cudaError_t launch_quantize(int fmt, const double* src, void* dst, int64_t count, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    k_quantize<<<grid_for(count), 256, 0, st>>>(fmt, src, dst, count);
    return cudaGetLastError();
}
cudaError_t launch_dequantize(int fmt, const void* src, double* dst, int64_t count,
                              cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    k_dequantize<<<grid_for(count), 256, 0, st>>>(fmt, src, dst, count);
    return cudaGetLastError();
}

template <typename W>
cudaError_t launch_round_in(const double* x, W* xw, int64_t rows, int64_t s, int64_t ldin,
                            int64_t ldout, cudaStream_t st) {
    if (rows * s <= 0) return cudaSuccess;
    k_round_in<W><<<grid_for(rows * s), 256, 0, st>>>(x, xw, rows, s, ldin, ldout);
    return cudaGetLastError();
}
template <typename W>
cudaError_t launch_widen_out(const W* bw, double* b, int64_t rows, int64_t s, int64_t ldin,
                             int64_t ldout, cudaStream_t st) {
    if (rows * s <= 0) return cudaSuccess;
    k_widen_out<W><<<grid_for(rows * s), 256, 0, st>>>(bw, b, rows, s, ldin, ldout);
    return cudaGetLastError();
}
template cudaError_t launch_round_in<double>(const double*, double*, int64_t, int64_t, int64_t,
                                             int64_t, cudaStream_t);
template cudaError_t launch_round_in<float>(const double*, float*, int64_t, int64_t, int64_t,
                                            int64_t, cudaStream_t);
template cudaError_t launch_widen_out<double>(const double*, double*, int64_t, int64_t, int64_t,
                                              int64_t, cudaStream_t);
template cudaError_t launch_widen_out<float>(const float*, double*, int64_t, int64_t, int64_t,
                                             int64_t, cudaStream_t);

template <typename W, int SB>
static cudaError_t gen_begin_sb(const PlanView& p, const W* x, int64_t ldx, int64_t s, W* partial,
                                W* tbuf, W* send, cudaStream_t st) {
    dim3 ga(p.nchunks, (unsigned)((s + SB - 1) / SB));
    k_gen_phaseA<W, SB><<<ga, 256, 0, st>>>(p, x, ldx, s, partial);
    k_gen_reduce<W><<<p.nnodes, 256, 0, st>>>(p, s, partial, tbuf, send);
    return cudaGetLastError();
}

template <typename W>
cudaError_t gen_begin(const PlanView& p, const W* x, int64_t ldx, int64_t s, W* partial, W* tbuf,
                      W* send, cudaStream_t st) {
    if (p.nchunks == 0) return cudaSuccess;
    if (p.nnodes == 0) return cudaSuccess;
    if (s == 1) return gen_begin_sb<W, 1>(p, x, ldx, s, partial, tbuf, send, st);
    if (s <= 4) return gen_begin_sb<W, 4>(p, x, ldx, s, partial, tbuf, send, st);
    return gen_begin_sb<W, 16>(p, x, ldx, s, partial, tbuf, send, st);
}

template <typename W>
cudaError_t gen_ext(const PlanView& p, int64_t s, const W* recv, W* tbuf, cudaStream_t st) {
    if (p.next == 0) return cudaSuccess;
    k_gen_reduce_ext<W><<<p.next, 256, 0, st>>>(p, s, recv, tbuf);
    return cudaGetLastError();
}

template <typename W, int SB>
static cudaError_t gen_end_sb(const PlanView& p, const W* x, int64_t ldx, const W* tbuf, W* b,
                              int64_t ldb, int64_t s, int max_chunk_rows, cudaStream_t st) {
    dim3 gb(p.nchunks, (unsigned)((s + SB - 1) / SB));
    size_t smem = (size_t)max_chunk_rows * SB * sizeof(W);
    k_gen_phaseB<W, SB><<<gb, 256, smem, st>>>(p, x, ldx, tbuf, b, ldb, s);
    return cudaGetLastError();
}

template <typename W>
cudaError_t gen_end(const PlanView& p, const W* x, int64_t ldx, const W* tbuf, W* b, int64_t ldb,
                    int64_t s, int max_chunk_rows, cudaStream_t st) {
    if (p.nchunks == 0) return cudaSuccess;
    if (s == 1) return gen_end_sb<W, 1>(p, x, ldx, tbuf, b, ldb, s, max_chunk_rows, st);
    if (s <= 4) return gen_end_sb<W, 4>(p, x, ldx, tbuf, b, ldb, s, max_chunk_rows, st);
    return gen_end_sb<W, 16>(p, x, ldx, tbuf, b, ldb, s, max_chunk_rows, st);
}

template cudaError_t gen_begin<double>(const PlanView&, const double*, int64_t, int64_t, double*,
                                       double*, double*, cudaStream_t);
template cudaError_t gen_begin<float>(const PlanView&, const float*, int64_t, int64_t, float*,
                                      float*, float*, cudaStream_t);
template cudaError_t gen_ext<double>(const PlanView&, int64_t, const double*, double*,
                                     cudaStream_t);
template cudaError_t gen_ext<float>(const PlanView&, int64_t, const float*, float*, cudaStream_t);
template cudaError_t gen_end<double>(const PlanView&, const double*, int64_t, const double*,
                                     double*, int64_t, int64_t, int, cudaStream_t);
template cudaError_t gen_end<float>(const PlanView&, const float*, int64_t, const float*, float*,
                                    int64_t, int64_t, int, cudaStream_t);

}  // namespace hodlr
