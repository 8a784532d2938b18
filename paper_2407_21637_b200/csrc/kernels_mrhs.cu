// Multi-right-hand-side kernels (see mrhs.h for the schedule).
//
// Operand staging.  X (and the coefficients T) are staged in shared memory in
// MMA-fragment order, so a lane fetches its whole B fragment with 16-byte
// loads and no bank conflicts.  The reduction index of every MMA is permuted
// so that a lane's four k positions of a 16-wide k step are four CONSECUTIVE
// rows (4*tig .. 4*tig+3): factor columns (V', contiguous over rows) and leaf
// rows (contiguous over columns) are then read with one 4-element vector load
// per lane whatever the storage format (q52 4 B, bf16/fp16 8 B, fp32 16 B,
// fp64 2x16 B), up-converted in registers, never re-packed in memory.  Any
// bijection of the k index leaves the contraction unchanged as long as A and
// B use the same one.
//
// MMA kinds:
//   fp64 working: mma.sync.m8n8k4.f64 (SASS DMMA, the FP64 tensor pipe);
//   fp32 working: mma.sync.m16n8k8.tf32, every operand split a = hi + lo
//                 (hi = rna_tf32(a), lo = rna_tf32(a - hi)) and
//                 acc += hi*lo' + lo*hi' + hi*hi'  (fp32-level accuracy).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "mrhs.h"

namespace hodlr {

namespace {

constexpr int kMrThreads = 256;
constexpr int kMrWarps = kMrThreads / 32;
constexpr int kChunk = 256;            // rows per chunk (plan.h chunks are <= 256 rows)
constexpr size_t kMrSmemTarget = 110 * 1024;  // keep two CTAs per SM

// ------------------------------------------------------------------ operand loads
template <typename W>
__device__ __forceinline__ void cvt4(float a, float b, float c, float d, W (&v)[4]) {
    v[0] = (W)a; v[1] = (W)b; v[2] = (W)c; v[3] = (W)d;
}

// Four consecutive elements i..i+3 (i a multiple of 4) of a narrow array.
template <typename W>
__device__ __forceinline__ void load4(int fmt, const uint8_t* base, int64_t i, W (&v)[4]) {
    switch (fmt) {
        case HODLR_FMT_FP64: {
            const double2* p = reinterpret_cast<const double2*>(base + i * 8);
            double2 a = __ldg(p), b = __ldg(p + 1);
            v[0] = (W)a.x; v[1] = (W)a.y; v[2] = (W)b.x; v[3] = (W)b.y;
            break;
        }
        case HODLR_FMT_FP32: {
            float4 a = __ldg(reinterpret_cast<const float4*>(base + i * 4));
            cvt4<W>(a.x, a.y, a.z, a.w, v);
            break;
        }
        case HODLR_FMT_FP16: {
            uint2 a = __ldg(reinterpret_cast<const uint2*>(base + i * 2));
            cvt4<W>(dec_fp16((uint16_t)a.x), dec_fp16((uint16_t)(a.x >> 16)), dec_fp16((uint16_t)a.y),
                    dec_fp16((uint16_t)(a.y >> 16)), v);
            break;
        }
        case HODLR_FMT_BF16: {
            uint2 a = __ldg(reinterpret_cast<const uint2*>(base + i * 2));
            cvt4<W>(__uint_as_float(a.x << 16), __uint_as_float(a.x & 0xffff0000u),
                    __uint_as_float(a.y << 16), __uint_as_float(a.y & 0xffff0000u), v);
            break;
        }
        default: {  // q52: the E5M2 byte is the high byte of the binary16 of the same value
            uint32_t a = __ldg(reinterpret_cast<const unsigned int*>(base + i));
            cvt4<W>(dec_q52((uint8_t)a), dec_q52((uint8_t)(a >> 8)), dec_q52((uint8_t)(a >> 16)),
                    dec_q52((uint8_t)(a >> 24)), v);
            break;
        }
    }
}

template <typename W>
__device__ __forceinline__ W load1(int fmt, const uint8_t* base, int64_t i) {
    return (W)dec_any(fmt, base, i);
}

// ------------------------------------------------------------------ MMA kinds
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = tf32_rna(x);
    lo = tf32_rna(x - __uint_as_float(hi));
}
__device__ __forceinline__ void tmma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// MR rows per m-tile, AR A-rows per lane (g, g+8), CR accumulators per lane,
// KU / UV: k width of one U-part step and coefficient values per lane.
// C element i of a lane: row g + 8*(i/2), column 2*tig + (i%2).
struct PolF64 {
    using W = double;
    static constexpr int MR = 8, AR = 1, CR = 2, KU = 4, UV = 1;
    // 16-wide k step, lane k positions = rows 4*tig + j
    __device__ static __forceinline__ void mma16(W (&c)[CR], const W (&a)[AR][4], const W (&b)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(c, a[0][j], b[j]);
    }
    // U step: lane k position tig = column 4*step + tig
    __device__ static __forceinline__ void mmau(W (&c)[CR], const W (&a)[AR][UV], const W (&b)[UV]) {
        dmma884(c, a[0][0], b[0]);
    }
};

struct PolTF32 {
    using W = float;
    static constexpr int MR = 16, AR = 2, CR = 4, KU = 8, UV = 2;
    // two m16n8k8 per 16-wide step: MMA p, k position tig -> row 4*tig+2p,
    // k position tig+4 -> row 4*tig+2p+1
    __device__ static __forceinline__ void mma16(W (&c)[CR], const W (&a)[AR][4], const W (&b)[4]) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t ah[4], al[4], bh[2], bl[2];
            split_tf32(a[0][2 * p], ah[0], al[0]);
            split_tf32(a[1][2 * p], ah[1], al[1]);
            split_tf32(a[0][2 * p + 1], ah[2], al[2]);
            split_tf32(a[1][2 * p + 1], ah[3], al[3]);
            split_tf32(b[2 * p], bh[0], bl[0]);
            split_tf32(b[2 * p + 1], bh[1], bl[1]);
            tmma(c, ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
            tmma(c, al[0], al[1], al[2], al[3], bh[0], bh[1]);
            tmma(c, ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
        }
    }
    // U step (k = 8): k position tig -> column 8*step + 2*tig, tig+4 -> 2*tig+1
    __device__ static __forceinline__ void mmau(W (&c)[CR], const W (&a)[AR][UV], const W (&b)[UV]) {
        uint32_t ah[4], al[4], bh[2], bl[2];
        split_tf32(a[0][0], ah[0], al[0]);
        split_tf32(a[1][0], ah[1], al[1]);
        split_tf32(a[0][1], ah[2], al[2]);
        split_tf32(a[1][1], ah[3], al[3]);
        split_tf32(b[0], bh[0], bl[0]);
        split_tf32(b[1], bh[1], bl[1]);
        tmma(c, ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
        tmma(c, al[0], al[1], al[2], al[3], bh[0], bh[1]);
        tmma(c, ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
    }
};

// Fragment-order index of X element (row r < 256, column q < ncol) for a
// CTA holding nct n-tiles: [r/16][q/8][lane = 4*(q%8) + (r/4)%4][r%4].
__device__ __forceinline__ int xfrag(int r, int q, int nct) {
    return ((((r >> 4) * nct + (q >> 3)) * 32 + (((q & 7) << 2) | ((r >> 2) & 3))) << 2) | (r & 3);
}

// Stage rows [r0, r0 + nrows) (zero beyond) and columns [q0, q0 + ncol) (zero
// beyond s) of a row-major matrix into fragment order.
template <typename W>
__device__ __forceinline__ void stage_x(W* xs, const W* __restrict__ x, int64_t ldx, int64_t r0,
                                        int nrows, int64_t q0, int ncol, int64_t s) {
    const int nct = ncol >> 3;
    for (int i = threadIdx.x; i < kChunk * ncol; i += blockDim.x) {
        const int r = i / ncol, q = i - r * ncol;
        W v = W(0);
        if (r < nrows && q0 + q < s) v = x[(r0 + r) * ldx + q0 + q];
        xs[xfrag(r, q, nct)] = v;
    }
}

// Map a task id of the phase-A list to (level, m-tile, n-tile).  Levels
// lev_lo.. contribute ceil(rv_max / MR) m-tiles x nct n-tiles each.
template <class Pol>
__device__ __forceinline__ void decode_task(const MrView& m, int lev_lo, int nct, int t, int& lv, int& mt,
                                            int& nt) {
    lv = lev_lo;
    for (;; ++lv) {
        const int cnt = ((m.lev[lv].rv_max + Pol::MR - 1) / Pol::MR) * nct;
        if (t < cnt) break;
        t -= cnt;
    }
    mt = t / nct;
    nt = t - mt * nct;
}

template <class Pol>
__device__ __forceinline__ int count_tasks(const MrView& m, int lev_lo, int nct) {
    int n = 0;
    for (int lv = lev_lo; lv < m.nlev; ++lv) n += ((m.lev[lv].rv_max + Pol::MR - 1) / Pol::MR) * nct;
    return n;
}

// ------------------------------------------------------------------ MA
// grid (nb, ceil(spad / ncol)), kMrThreads.  Shared memory: X chunk in
// fragment order (256 x ncol) + one accumulator tile per task, each element
// owned by one lane of one warp for the whole kernel (no shared-memory races,
// no block barrier besides the X restaging).
template <class Pol>
__global__ void __launch_bounds__(kMrThreads) k_mr_a(PlanView p, const __grid_constant__ MrView m, int lev_lo,
                                                     const typename Pol::W* __restrict__ x, int64_t ldx,
                                                     int64_t s, int spad, int ncol,
                                                     typename Pol::W* __restrict__ partial) {
    using W = typename Pol::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* xs = reinterpret_cast<W*>(smem_raw);
    W* accs = xs + kChunk * ncol;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int nct = ncol >> 3;
    const int64_t q0 = (int64_t)blockIdx.y * ncol;
    const int ntasks = count_tasks<Pol>(m, lev_lo, nct);
    const int c_beg = (int)((int64_t)blockIdx.x * p.nchunks / gridDim.x);
    const int c_end = (int)((int64_t)(blockIdx.x + 1) * p.nchunks / gridDim.x);

    for (int t = warp; t < ntasks; t += kMrWarps)
#pragma unroll
        for (int i = 0; i < Pol::CR; ++i) accs[((size_t)t * 32 + lane) * Pol::CR + i] = W(0);

    for (int ci = c_beg; ci < c_end; ++ci) {
        const ChunkDesc ch = p.chunks[ci];
        stage_x<W>(xs, x, ldx, ch.row0, ch.nrows, q0, ncol, s);
        __syncthreads();
        const int nk = (ch.nrows + 15) >> 4;
        for (int t = warp; t < ntasks; t += kMrWarps) {
            int lv, mt, nt;
            decode_task<Pol>(m, lev_lo, nct, t, lv, mt, nt);
            const int node = p.chunk_nodes[ci * p.nlev + lv];
            const NodeDesc nd = p.nodes[node];
            const int off = ch.row0 - nd.row0;
            const int fb = fmt_bytes(nd.v_fmt);
            const uint8_t* col[Pol::AR];
#pragma unroll
            for (int a = 0; a < Pol::AR; ++a) {
                const int c = mt * Pol::MR + g + 8 * a;
                col[a] = c < nd.rv ? p.arena + nd.v_off + (int64_t)c * nd.v_ld * fb : nullptr;
            }
            W acc[Pol::CR];
#pragma unroll
            for (int i = 0; i < Pol::CR; ++i) acc[i] = W(0);
#pragma unroll 4
            for (int kb = 0; kb < nk; ++kb) {
                const int r = kb * 16 + 4 * tig;
                W av[Pol::AR][4];
#pragma unroll
                for (int a = 0; a < Pol::AR; ++a) {
                    if (col[a]) {
                        load4<W>(nd.v_fmt, col[a], off + r, av[a]);
                        if (r + 4 > ch.nrows) {  // ragged chunk end: rows past it are another chunk's
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (r + j >= ch.nrows) av[a][j] = W(0);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) av[a][j] = W(0);
                    }
                }
                const float4* bp = reinterpret_cast<const float4*>(xs + ((kb * nct + nt) * 32 + lane) * 4);
                W bv[4];
                if constexpr (sizeof(W) == 8) {
                    const float4 u0 = bp[0], u1 = bp[1];
                    const double2 d0 = *reinterpret_cast<const double2*>(&u0);
                    const double2 d1 = *reinterpret_cast<const double2*>(&u1);
                    bv[0] = d0.x; bv[1] = d0.y; bv[2] = d1.x; bv[3] = d1.y;
                } else {
                    const float4 u0 = bp[0];
                    bv[0] = u0.x; bv[1] = u0.y; bv[2] = u0.z; bv[3] = u0.w;
                }
                Pol::mma16(acc, av, bv);
            }
            W* my = accs + ((size_t)t * 32 + lane) * Pol::CR;
#pragma unroll
            for (int i = 0; i < Pol::CR; ++i) my[i] += acc[i];
            const bool more = ci + 1 < c_end && p.chunk_nodes[(ci + 1) * p.nlev + lv] == node;
            if (!more) {
                const MrLevel L = m.lev[lv];
                const int64_t slot = (int64_t)blockIdx.x + m.slots[node].jrel;
#pragma unroll
                for (int i = 0; i < Pol::CR; ++i) {
                    const int c = mt * Pol::MR + g + 8 * (i >> 1);
                    const int q = nt * 8 + 2 * tig + (i & 1);
                    if (c < L.rv_max)
                        partial[(L.part_rows + slot * L.rv_pad + c) * spad + q0 + q] = my[i];
                    my[i] = W(0);
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ MR
// One CTA per node: T[c][q] = sum over the node's slots in CTA order.
template <typename W>
__global__ void __launch_bounds__(256) k_mr_reduce(PlanView p, const __grid_constant__ MrView m, int node_lo,
                                                   int64_t s, int spad, const W* __restrict__ partial,
                                                   W* __restrict__ tbuf) {
    const int node = node_lo + blockIdx.x;
    const NodeDesc nd = p.nodes[node];
    const MrSlot sl = m.slots[node];
    const MrLevel L = m.lev[sl.lv];
    const int64_t cnt = (int64_t)nd.rv * s;
    W* dst = tbuf + nd.t_off * s;
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        const int64_t c = i / s, q = i - c * s;
        const W* src = partial + (L.part_rows + (int64_t)(sl.b0 + sl.jrel) * L.rv_pad + c) * spad + q;
        const int64_t stride = (int64_t)L.rv_pad * spad;
        W acc = src[0];
        for (int b = sl.b0 + 1; b <= sl.b1; ++b) acc += src[(int64_t)(b - sl.b0) * stride];
        dst[i] = acc;
    }
}

// ------------------------------------------------------------------ MB
// grid (nchunks, ceil(spad / ncol)), kMrThreads; warp w owns chunk rows
// [32w, 32w + 32) (MT m-tiles) x all NT n-tiles of the CTA's columns.
template <class Pol, int NT>
__global__ void __launch_bounds__(kMrThreads) k_mr_b(PlanView p, const __grid_constant__ MrView m, int lev_lo,
                                                     const typename Pol::W* __restrict__ x, int64_t ldx,
                                                     const typename Pol::W* __restrict__ tbuf,
                                                     typename Pol::W* __restrict__ b, int64_t ldb,
                                                     int64_t s) {
    using W = typename Pol::W;
    constexpr int MT = 32 / Pol::MR;
    constexpr int ncol = NT * 8;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* xs = reinterpret_cast<W*>(smem_raw);
    W* ts = xs + kChunk * ncol;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int chunk = blockIdx.x;
    const int64_t q0 = (int64_t)blockIdx.y * ncol;
    const ChunkDesc ch = p.chunks[chunk];
    const LeafDesc lf = p.leaves[ch.leaf];

    // coefficients of every level, fragment order [step][nt][lane][UV]
    {
        int base = 0;
        for (int lv = lev_lo; lv < m.nlev; ++lv) {
            const int steps = (m.lev[lv].ru_max + Pol::KU - 1) / Pol::KU;
            const NodeDesc nd = p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
            const W* t = tbuf + nd.tsrc_off * s;
            for (int i = threadIdx.x; i < steps * Pol::KU * ncol; i += blockDim.x) {
                const int c = i / ncol, q = i - c * ncol;
                W v = W(0);
                if (c < nd.ru && q0 + q < s) v = t[(int64_t)c * s + q0 + q];
                const int step = c / Pol::KU, w = c - step * Pol::KU;
                const int tg = w / Pol::UV, u = w - tg * Pol::UV;
                const int ln = (q & 7) * 4 + tg;
                ts[base + ((step * NT + (q >> 3)) * 32 + ln) * Pol::UV + u] = v;
            }
            base += steps * NT * 32 * Pol::UV;
        }
    }

    W acc[MT][NT][Pol::CR];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < Pol::CR; ++i) acc[mt][nt][i] = W(0);

    const int wb = fmt_bytes(lf.fmt);
    const int lr0 = ch.row0 - lf.row0;  // first leaf row of the chunk
    // leaf product D[chunk rows, :] X[leaf rows]
    for (int kblk = 0; kblk < lf.m; kblk += kChunk) {
        const int kn = min(kChunk, lf.m - kblk);
        __syncthreads();  // previous X block (and, first time, the T staging) consumed/complete
        stage_x<W>(xs, x, ldx, lf.row0 + kblk, kn, q0, ncol, s);
        __syncthreads();
        const int nk = (kn + 15) >> 4;
        const uint8_t* drow[MT][Pol::AR];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int a = 0; a < Pol::AR; ++a) {
                const int row = warp * 32 + mt * Pol::MR + g + 8 * a;
                drow[mt][a] = row < ch.nrows
                                  ? p.arena + lf.off + ((int64_t)(lr0 + row) * lf.ld + kblk) * wb
                                  : nullptr;
            }
#pragma unroll 2
        for (int kb = 0; kb < nk; ++kb) {
            const int k = kb * 16 + 4 * tig;
            W av[MT][Pol::AR][4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int a = 0; a < Pol::AR; ++a) {
                    if (drow[mt][a]) {
                        load4<W>(lf.fmt, drow[mt][a], k, av[mt][a]);
                        if (k + 4 > kn) {
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (k + j >= kn) av[mt][a][j] = W(0);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) av[mt][a][j] = W(0);
                    }
                }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const float4* bp = reinterpret_cast<const float4*>(xs + ((kb * NT + nt) * 32 + lane) * 4);
                W bv[4];
                if constexpr (sizeof(W) == 8) {
                    const float4 u0 = bp[0], u1 = bp[1];
                    const double2 d0 = *reinterpret_cast<const double2*>(&u0);
                    const double2 d1 = *reinterpret_cast<const double2*>(&u1);
                    bv[0] = d0.x; bv[1] = d0.y; bv[2] = d1.x; bv[3] = d1.y;
                } else {
                    const float4 u0 = bp[0];
                    bv[0] = u0.x; bv[1] = u0.y; bv[2] = u0.z; bv[3] = u0.w;
                }
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) Pol::mma16(acc[mt][nt], av[mt], bv);
            }
        }
    }

    // sum_k U_k[chunk rows] T_k
    int base = 0;
    for (int lv = lev_lo; lv < m.nlev; ++lv) {
        const int steps = (m.lev[lv].ru_max + Pol::KU - 1) / Pol::KU;
        const NodeDesc nd = p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
        const int fb = fmt_bytes(nd.u_fmt);
        const uint8_t* ucol = p.arena + nd.u_off;
        const int64_t cstride = (int64_t)nd.u_ld * fb;
        const int off = ch.row0 - nd.row0;
        const int nsteps = (nd.ru + Pol::KU - 1) / Pol::KU;
        for (int step = 0; step < nsteps; ++step) {
            W av[MT][Pol::AR][Pol::UV];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int a = 0; a < Pol::AR; ++a) {
                    const int row = warp * 32 + mt * Pol::MR + g + 8 * a;
#pragma unroll
                    for (int u = 0; u < Pol::UV; ++u) {
                        const int c = step * Pol::KU + Pol::UV * tig + u;
                        av[mt][a][u] = (c < nd.ru && row < ch.nrows)
                                           ? load1<W>(nd.u_fmt, ucol + c * cstride, off + row)
                                           : W(0);
                    }
                }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                W bv[Pol::UV];
#pragma unroll
                for (int u = 0; u < Pol::UV; ++u)
                    bv[u] = ts[base + ((step * NT + nt) * 32 + lane) * Pol::UV + u];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) Pol::mmau(acc[mt][nt], av[mt], bv);
            }
        }
        base += steps * NT * 32 * Pol::UV;
    }

    // epilogue: rows disjoint per chunk, written once
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < Pol::CR; ++i) {
                const int row = warp * 32 + mt * Pol::MR + g + 8 * (i >> 1);
                const int64_t q = q0 + nt * 8 + 2 * tig + (i & 1);
                if (row < ch.nrows && q < s) b[(int64_t)(ch.row0 + row) * ldb + q] = acc[mt][nt][i];
            }
}

// ------------------------------------------------------------------ host helpers
template <class Pol>
size_t ma_smem(const MrView& m, int lev_lo, int ncol) {
    size_t tiles = 0;
    for (int lv = lev_lo; lv < m.nlev; ++lv) tiles += (m.lev[lv].rv_max + Pol::MR - 1) / Pol::MR;
    tiles *= ncol / 8;
    return (size_t)kChunk * ncol * sizeof(typename Pol::W) + tiles * 32 * Pol::CR * sizeof(typename Pol::W);
}
template <class Pol>
size_t mb_smem(const MrView& m, int lev_lo, int ncol) {
    size_t rows = 0;
    for (int lv = lev_lo; lv < m.nlev; ++lv)
        rows += (size_t)((m.lev[lv].ru_max + Pol::KU - 1) / Pol::KU) * Pol::KU;
    return ((size_t)kChunk + rows) * ncol * sizeof(typename Pol::W);
}

template <class Pol>
cudaError_t launch_mb(int nt, dim3 grid, size_t smem, cudaStream_t st, const PlanView& p, const MrView& m,
                      int lev_lo, const typename Pol::W* x, int64_t ldx, const typename Pol::W* tbuf,
                      typename Pol::W* b, int64_t ldb, int64_t s) {
#define HODLR_MB_CASE(NTV)                                                                        \
    case NTV: {                                                                                   \
        auto k = k_mr_b<Pol, NTV>;                                                                \
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                             (int)smem);                                          \
        if (e != cudaSuccess) return e;                                                           \
        k<<<grid, kMrThreads, smem, st>>>(p, m, lev_lo, x, ldx, tbuf, b, ldb, s);                 \
        return cudaGetLastError();                                                                \
    }
    switch (nt) {
        HODLR_MB_CASE(1)
        HODLR_MB_CASE(2)
        HODLR_MB_CASE(4)
        default: return cudaErrorInvalidValue;
    }
#undef HODLR_MB_CASE
}

template <class Pol>
cudaError_t mr_run(const PlanView& p, const MrPlan& mr, int lev_lo, const typename Pol::W* x, int64_t ldx,
                   typename Pol::W* b, int64_t ldb, int64_t s, typename Pol::W* partial,
                   typename Pol::W* tbuf, cudaStream_t st) {
    using W = typename Pol::W;
    const MrView& m = mr.view;
    const int spad = (int)mr_spad(s);
    if (p.nchunks == 0) return cudaSuccess;
    const bool any_level = lev_lo < m.nlev;
    if (any_level) {
        // MA: widest column group whose shared memory keeps two CTAs per SM
        int ncol = spad;
        while (ncol > 8 && ma_smem<Pol>(m, lev_lo, ncol) > kMrSmemTarget) ncol = (ncol / 2 + 7) / 8 * 8;
        size_t sm_a = ma_smem<Pol>(m, lev_lo, ncol);
        if (sm_a > 227 * 1024) return cudaErrorInvalidConfiguration;
        auto ka = k_mr_a<Pol>;
        cudaError_t e = cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_a);
        if (e != cudaSuccess) return e;
        dim3 ga(m.nb, (spad + ncol - 1) / ncol);
        ka<<<ga, kMrThreads, sm_a, st>>>(p, m, lev_lo, x, ldx, s, spad, ncol, partial);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        const int node_lo = m.lev[lev_lo].node0;
        const int nred = p.nnodes - node_lo;
        if (nred > 0) {
            k_mr_reduce<W><<<nred, 256, 0, st>>>(p, m, node_lo, s, spad, partial, tbuf);
            e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
    }
    // MB: n-tiles per warp (1, 2 or 4), shared memory within the target
    int nt = spad >= 32 ? 4 : spad >= 16 ? 2 : 1;
    while (nt > 1 && mb_smem<Pol>(m, lev_lo, nt * 8) > kMrSmemTarget) nt /= 2;
    size_t sm_b = mb_smem<Pol>(m, lev_lo, nt * 8);
    if (sm_b > 227 * 1024) return cudaErrorInvalidConfiguration;
    dim3 gb(p.nchunks, (spad + nt * 8 - 1) / (nt * 8));
    return launch_mb<Pol>(nt, gb, sm_b, st, p, m, lev_lo, x, ldx, tbuf, b, ldb, s);
}

}  // namespace

// ------------------------------------------------------------------ plan
hodlr_status mr_prepare(const MrInput& in, MrPlan& mr) {
    mr = MrPlan{};
    const auto& nodes = *in.nodes;
    const auto& chunks = *in.chunks;
    const auto& cn = *in.chunk_nodes;
    const int nlev = in.nlev;
    mr.leaf_fmt = in.leaf_fmt;
    if (nlev > kMrMaxLevels || chunks.empty()) return HODLR_OK;  // not eligible: generic path
    for (const LeafDesc& l : *in.leaves) mr.max_leaf_m = std::max(mr.max_leaf_m, l.m);
    // 4-element vector loads need 16-row aligned chunk offsets inside nodes
    for (size_t ci = 0; ci < chunks.size(); ++ci)
        for (int lv = 0; lv < nlev; ++lv) {
            const NodeDesc& nd = nodes[cn[ci * nlev + lv]];
            if ((chunks[ci].row0 - nd.row0) % 16 != 0) return HODLR_OK;
        }
    for (const ChunkDesc& c : chunks) {
        const LeafDesc& l = (*in.leaves)[c.leaf];
        if ((c.row0 - l.row0) % 16 != 0) return HODLR_OK;
    }
    MrView& v = mr.view;
    v.nlev = nlev;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, in.device);
    const int nch = (int)chunks.size();
    v.nb = std::max(1, std::min(nch, 2 * sms));
    for (int lv = 0; lv < nlev; ++lv) v.lev[lv] = MrLevel{-1, 0, 0, 0, 0, 0, 0};
    for (size_t id = 0; id < nodes.size(); ++id) {
        const NodeDesc& nd = nodes[id];
        const int lv = nd.level - 1;
        if (lv < 0 || lv >= nlev) return HODLR_OK;
        MrLevel& L = v.lev[lv];
        if (L.node0 < 0) L.node0 = (int)id;
        if ((int)id != L.node0 + L.nnodes) return HODLR_OK;  // levels must be contiguous id ranges
        L.nnodes++;
        L.rv_max = std::max(L.rv_max, nd.rv);
        L.ru_max = std::max(L.ru_max, nd.ru);
        if (nd.u_fmt == HODLR_FMT_FP64 || nd.v_fmt == HODLR_FMT_FP64) mr.has_fp64_operand = true;
    }
    if (in.leaf_fmt == HODLR_FMT_FP64) mr.has_fp64_operand = true;
    int64_t rows = 0;
    for (int lv = 0; lv < nlev; ++lv) {
        MrLevel& L = v.lev[lv];
        if (L.node0 < 0) return HODLR_OK;
        L.rv_pad = (L.rv_max + 7) / 8 * 8;
        L.part_rows = rows;
        rows += (int64_t)(v.nb + L.nnodes) * L.rv_pad;
    }
    v.part_rows = rows;
    // node -> CTA range of the phase-A grid
    std::vector<MrSlot> slots(nodes.size(), MrSlot{-1, -1, 0, 0});
    for (int b = 0; b < v.nb; ++b) {
        const int c0 = (int)((int64_t)b * nch / v.nb), c1 = (int)((int64_t)(b + 1) * nch / v.nb);
        for (int ci = c0; ci < c1; ++ci)
            for (int lv = 0; lv < nlev; ++lv) {
                MrSlot& s = slots[cn[(size_t)ci * nlev + lv]];
                if (s.b0 < 0) s.b0 = b;
                s.b1 = b;
            }
    }
    for (size_t id = 0; id < nodes.size(); ++id) {
        const int lv = nodes[id].level - 1;
        slots[id].lv = lv;
        slots[id].jrel = (int)id - v.lev[lv].node0;
        if (slots[id].b0 < 0) return HODLR_OK;  // node without rows: generic path
    }
    cudaError_t e = cudaMalloc(&mr.dev, slots.size() * sizeof(MrSlot));
    if (e == cudaSuccess)
        e = cudaMemcpy(mr.dev, slots.data(), slots.size() * sizeof(MrSlot), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        mr_release(mr);
        return HODLR_ERR_CUDA;
    }
    v.slots = (const MrSlot*)mr.dev;
    mr.ok = true;
    return HODLR_OK;
}

void mr_release(MrPlan& mr) {
    if (mr.dev) cudaFree(mr.dev);
    mr.dev = nullptr;
    mr.ok = false;
}

bool mr_usable(const MrPlan& mr, int working_fmt) {
    if (!mr.ok) return false;
    if (working_fmt == HODLR_FMT_FP64) return true;
    // TF32 kind: every operand must be exact in fp32 (fp64-stored factors under
    // fp32 working are multiplied in binary64 by the generic kernels)
    return working_fmt == HODLR_FMT_FP32 && !mr.has_fp64_operand;
}

int mr_launches() { return 3; }

template <>
cudaError_t mr_matvec<double>(const PlanView& p, const MrPlan& mr, int lev_lo, const double* x, int64_t ldx,
                              double* b, int64_t ldb, int64_t s, double* partial, double* tbuf,
                              cudaStream_t st) {
    return mr_run<PolF64>(p, mr, lev_lo, x, ldx, b, ldb, s, partial, tbuf, st);
}
template <>
cudaError_t mr_matvec<float>(const PlanView& p, const MrPlan& mr, int lev_lo, const float* x, int64_t ldx,
                             float* b, int64_t ldb, int64_t s, float* partial, float* tbuf, cudaStream_t st) {
    return mr_run<PolTF32>(p, mr, lev_lo, x, ldx, b, ldb, s, partial, tbuf, st);
}

}  // namespace hodlr
