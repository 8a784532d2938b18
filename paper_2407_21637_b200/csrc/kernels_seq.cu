// Simulated narrow working precisions (bf16 / fp16 / q52 working): Alg. 3 with
// the reference's "full-arithmetic" rounding model (arithmetic.py:14-67,
// SPEC.md:337,400), used by the paper's matvec experiment (PAPER.md:1264-1279,
// working in {fp64, fp32, bf16}).
//
// The model: operands enter as stored (binary64 view of the narrow factor),
// every scalar product and every partial sum is formed in binary64 and rounded
// at once to the working format, and contractions run strictly left to right
//     acc = rnd(a_0 b_0);  acc = rnd(acc + rnd(a_j b_j)),  j = 1, 2, ...
// (arithmetic.py:59-67).  The per-op rounding makes the result depend on the
// summation order, so these kernels keep the reference's order and give every
// output chain to ONE thread: the result is bit-identical to the reference
// arithmetic, and the parallelism is across chains only
//     phase A: one thread per (node, V' column, rhs)   -- chain over the node's rows
//     phase B: one thread per (row, rhs)               -- levels 1..l in order, each
//              level's U t chain over its rank, b = rnd(b + y); the leaf chain last
// x, t and b travel as binary64 holding working-format values (the reference's
// own representation, fpsim.py:160-185).  No tensor cores, no reordering: this
// is the fidelity path of the sweep harness, not the throughput path.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace hodlr {

namespace {

// binary64 -> nearest value of the working format, as binary64 (round_matrix:
// one RNE rounding, overflow -> inf, subnormals kept)
template <int FMT>
__device__ __forceinline__ double rnd(double v) {
    if (FMT == HODLR_FMT_Q52) return (double)dec_q52(enc_q52(v));
    if (FMT == HODLR_FMT_BF16) return (double)dec_bf16(enc_bf16(v));
    if (FMT == HODLR_FMT_FP16) return (double)dec_fp16(enc_fp16(v));
    if (FMT == HODLR_FMT_FP32) return (double)enc_fp32(v);
    return v;
}

// acc <- rnd(acc + rnd(a*b)), or rnd(a*b) for the first term; no contraction
template <int FMT>
__device__ __forceinline__ double step(double acc, double a, double b, bool first) {
    const double p = rnd<FMT>(__dmul_rn(a, b));
    return first ? p : rnd<FMT>(__dadd_rn(acc, p));
}

template <int FMT>
__global__ void k_seq_round(const double* __restrict__ src, double* __restrict__ dst, int64_t rows, int64_t s,
                            int64_t ldin, int64_t ldout) {
    const int64_t total = rows * s;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / s, q = i - r * s;
        dst[r * ldout + q] = rnd<FMT>(src[r * ldin + q]);
    }
}

// t_{k,j}[c, q] = V'_{k,j}[:, c]^T x[I_j, q], strictly in row order
template <int FMT>
__global__ void __launch_bounds__(128) k_seq_a(PlanView p, const double* __restrict__ x, int64_t ldx, int64_t s,
                                               double* __restrict__ tbuf) {
    const NodeDesc nd = p.nodes[blockIdx.x];
    const int64_t cnt = (int64_t)nd.rv * s;
    const int vb = fmt_bytes(nd.v_fmt);
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        const int64_t c = i / s, q = i - c * s;
        const uint8_t* col = p.arena + nd.v_off + c * nd.v_ld * vb;
        const double* xr = x + (int64_t)nd.row0 * ldx + q;
        double acc = 0.0;
        for (int r = 0; r < nd.nrows; ++r) acc = step<FMT>(acc, dec_any(nd.v_fmt, col, r), xr[(int64_t)r * ldx], r == 0);
        tbuf[nd.t_off * s + i] = acc;
    }
}

// b[row, q] = (((0 + U_1 t_1) + U_2 t_2) + ... + U_l t_l) + D x, each "+" rounded
template <int FMT>
__global__ void __launch_bounds__(128) k_seq_b(PlanView p, const double* __restrict__ x, int64_t ldx,
                                               const double* __restrict__ tbuf, double* __restrict__ b, int64_t ldb,
                                               int64_t s) {
    const int chunk = blockIdx.x;
    const ChunkDesc ch = p.chunks[chunk];
    const LeafDesc lf = p.leaves[ch.leaf];
    const int64_t cnt = (int64_t)ch.nrows * s;
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        const int rr = (int)(i / s);
        const int64_t q = i - (int64_t)rr * s;
        const int row = ch.row0 + rr;
        double bacc = 0.0;
        for (int lv = 0; lv < p.nlev; ++lv) {
            const NodeDesc nd = p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
            const uint8_t* ucol = p.arena + nd.u_off;
            const int64_t cstride = (int64_t)nd.u_ld * fmt_bytes(nd.u_fmt);
            const double* t = tbuf + nd.tsrc_off * s + q;
            double y = 0.0;
            for (int c = 0; c < nd.ru; ++c)
                y = step<FMT>(y, dec_any(nd.u_fmt, ucol + c * cstride, row - nd.row0), t[(int64_t)c * s], c == 0);
            bacc = rnd<FMT>(__dadd_rn(bacc, y));
        }
        const uint8_t* drow = p.arena + lf.off + (int64_t)(row - lf.row0) * lf.ld * fmt_bytes(lf.fmt);
        const double* xr = x + (int64_t)lf.row0 * ldx + q;
        double y = 0.0;
        for (int j = 0; j < lf.m; ++j) y = step<FMT>(y, dec_any(lf.fmt, drow, j), xr[(int64_t)j * ldx], j == 0);
        b[(int64_t)row * ldb + q] = rnd<FMT>(__dadd_rn(bacc, y));
    }
}

template <int FMT>
cudaError_t seq_run(const PlanView& p, const double* x, int64_t ldx, double* b, int64_t ldb, int64_t s, double* tbuf,
                    cudaStream_t st) {
    if (p.nchunks == 0) return cudaSuccess;
    if (p.nnodes > 0) k_seq_a<FMT><<<p.nnodes, 128, 0, st>>>(p, x, ldx, s, tbuf);
    k_seq_b<FMT><<<p.nchunks, 128, 0, st>>>(p, x, ldx, tbuf, b, ldb, s);
    return cudaGetLastError();
}

}  // namespace

cudaError_t seq_round(int fmt, const double* src, double* dst, int64_t rows, int64_t s, int64_t ldin, int64_t ldout,
                      cudaStream_t st) {
    if (rows * s <= 0) return cudaSuccess;
    const int64_t g64 = (rows * s + 255) / 256;
    const int g = (int)(g64 < 148 * 8 ? g64 : 148 * 8);
    switch (fmt) {
        case HODLR_FMT_Q52: k_seq_round<HODLR_FMT_Q52><<<g, 256, 0, st>>>(src, dst, rows, s, ldin, ldout); break;
        case HODLR_FMT_BF16: k_seq_round<HODLR_FMT_BF16><<<g, 256, 0, st>>>(src, dst, rows, s, ldin, ldout); break;
        case HODLR_FMT_FP16: k_seq_round<HODLR_FMT_FP16><<<g, 256, 0, st>>>(src, dst, rows, s, ldin, ldout); break;
        case HODLR_FMT_FP32: k_seq_round<HODLR_FMT_FP32><<<g, 256, 0, st>>>(src, dst, rows, s, ldin, ldout); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t seq_matvec(int fmt, const PlanView& p, const double* x, int64_t ldx, double* b, int64_t ldb, int64_t s,
                       double* tbuf, cudaStream_t st) {
    switch (fmt) {
        case HODLR_FMT_Q52: return seq_run<HODLR_FMT_Q52>(p, x, ldx, b, ldb, s, tbuf, st);
        case HODLR_FMT_BF16: return seq_run<HODLR_FMT_BF16>(p, x, ldx, b, ldb, s, tbuf, st);
        case HODLR_FMT_FP16: return seq_run<HODLR_FMT_FP16>(p, x, ldx, b, ldb, s, tbuf, st);
        case HODLR_FMT_FP32: return seq_run<HODLR_FMT_FP32>(p, x, ldx, b, ldb, s, tbuf, st);
        case HODLR_FMT_FP64: return seq_run<HODLR_FMT_FP64>(p, x, ldx, b, ldb, s, tbuf, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hodlr
