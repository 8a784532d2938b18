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
#include <cuda.h>  // CUtensorMap types only (the encoder is fetched through the runtime's driver entry point)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "async.cuh"
#include "mrhs.h"

namespace hodlr {

namespace {

constexpr int kMrThreads = 256;
constexpr int kMrWarps = kMrThreads / 32;
constexpr int kChunk = 256;            // rows per chunk (plan.h chunks are <= 256 rows)
constexpr size_t kMrSmemTarget = 110 * 1024;  // keep two CTAs per SM
constexpr int kBWarps = 16;                  // slab phase-B CTA: 16 warps ...
constexpr int kBRows = kChunk / kBWarps;     // ... of 16 chunk rows each
constexpr int kAWarps = 16;                  // slab phase-A CTA warps (one task list each)

// ------------------------------------------------------------------ operand loads
// values the integer widening does not cover
__host__ __device__ __forceinline__ bool f32_special(uint32_t bits) {
    const uint32_t t = bits & 0x7fffffffu;
    return t != 0 && (t - 0x00800000u) >= 0x7f000000u;
}
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
// x = hi + lo (+ O(2^-22 |x|)).  Non-finite x: lo = 0, so inf propagates as
// inf instead of turning into inf - inf = NaN.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = tf32_rna(x);
    const float r = x - __uint_as_float(hi);
    lo = tf32_rna(fabsf(x) <= 3.402823466e38f ? r : 0.0f);
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
    // operand fragments as the MMA consumes them (fp64: as loaded)
    struct AF { W v[AR][4]; };
    struct BF { W v[4]; };
    struct AUF { W v[AR][UV]; };
    struct BUF { W v[UV]; };
    __device__ static __forceinline__ void prep_a(AF& f, const W (&a)[AR][4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) f.v[0][j] = a[0][j];
    }
    __device__ static __forceinline__ void prep_b(BF& f, const W (&b)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) f.v[j] = b[j];
    }
    __device__ static __forceinline__ void prep_au(AUF& f, const W (&a)[AR][UV]) { f.v[0][0] = a[0][0]; }
    __device__ static __forceinline__ void prep_bu(BUF& f, const W (&b)[UV]) { f.v[0] = b[0]; }
    // 16-wide k step, lane k positions = rows 4*tig + j
    __device__ static __forceinline__ void mma16(W (&c)[CR], const AF& a, const BF& b) {
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(c, a.v[0][j], b.v[j]);
    }
    // U step: lane k position tig = column 4*step + tig
    __device__ static __forceinline__ void mmau(W (&c)[CR], const AUF& a, const BUF& b) {
        dmma884(c, a.v[0][0], b.v[0]);
    }
    // whole warp tile, independent accumulators interleaved between dependent MMAs
    template <int MT, int NT>
    __device__ static __forceinline__ void mma16_tile(W (&c)[MT][NT][CR], const AF (&a)[MT], const BF (&b)[NT]) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) dmma884(c[mt][nt], a[mt].v[0][j], b[nt].v[j]);
    }
    template <int MT, int NT>
    __device__ static __forceinline__ void mmau_tile(W (&c)[MT][NT][CR], const AUF (&a)[MT], const BUF (&b)[NT]) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) dmma884(c[mt][nt], a[mt].v[0][0], b[nt].v[0]);
    }
    // the first MT of MTA tiles: MT * NT independent accumulators between dependent MMAs
    template <int MT, int NT, int MTA>
    __device__ static __forceinline__ void mma16_group(W (&c)[MTA][NT][CR], const AF (&a)[MTA], const BF (&b)[NT]) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) dmma884(c[mt][nt], a[mt].v[0][j], b[nt].v[j]);
    }
};

struct PolTF32 {
    using W = float;
    static constexpr int MR = 16, AR = 2, CR = 4, KU = 8, UV = 2;
    // operands split once into tf32 hi/lo pairs, reused across tiles
    struct AF { uint32_t h[AR][4], l[AR][4]; };
    struct BF { uint32_t h[4], l[4]; };
    struct AUF { uint32_t h[AR][UV], l[AR][UV]; };
    struct BUF { uint32_t h[UV], l[UV]; };
    __device__ static __forceinline__ void prep_a(AF& f, const W (&a)[AR][4]) {
#pragma unroll
        for (int r = 0; r < AR; ++r)
#pragma unroll
            for (int j = 0; j < 4; ++j) split_tf32(a[r][j], f.h[r][j], f.l[r][j]);
    }
    __device__ static __forceinline__ void prep_b(BF& f, const W (&b)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) split_tf32(b[j], f.h[j], f.l[j]);
    }
    __device__ static __forceinline__ void prep_au(AUF& f, const W (&a)[AR][UV]) {
#pragma unroll
        for (int r = 0; r < AR; ++r)
#pragma unroll
            for (int u = 0; u < UV; ++u) split_tf32(a[r][u], f.h[r][u], f.l[r][u]);
    }
    __device__ static __forceinline__ void prep_bu(BUF& f, const W (&b)[UV]) {
#pragma unroll
        for (int u = 0; u < UV; ++u) split_tf32(b[u], f.h[u], f.l[u]);
    }
    // two m16n8k8 per 16-wide step: MMA p, k position tig -> row 4*tig+2p,
    // k position tig+4 -> row 4*tig+2p+1; acc += hi*lo' + lo*hi' + hi*hi'
    __device__ static __forceinline__ void mma16(W (&c)[CR], const AF& a, const BF& b) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int j0 = 2 * p, j1 = 2 * p + 1;
            tmma(c, a.h[0][j0], a.h[1][j0], a.h[0][j1], a.h[1][j1], b.l[j0], b.l[j1]);
            tmma(c, a.l[0][j0], a.l[1][j0], a.l[0][j1], a.l[1][j1], b.h[j0], b.h[j1]);
            tmma(c, a.h[0][j0], a.h[1][j0], a.h[0][j1], a.h[1][j1], b.h[j0], b.h[j1]);
        }
    }
    // U step (k = 8): k position tig -> column 8*step + 2*tig, tig+4 -> 2*tig+1
    __device__ static __forceinline__ void mmau(W (&c)[CR], const AUF& a, const BUF& b) {
        tmma(c, a.h[0][0], a.h[1][0], a.h[0][1], a.h[1][1], b.l[0], b.l[1]);
        tmma(c, a.l[0][0], a.l[1][0], a.l[0][1], a.l[1][1], b.h[0], b.h[1]);
        tmma(c, a.h[0][0], a.h[1][0], a.h[0][1], a.h[1][1], b.h[0], b.h[1]);
    }
    // whole warp tile, independent accumulators interleaved between dependent MMAs
    template <int MT, int NT>
    __device__ static __forceinline__ void mma16_tile(W (&c)[MT][NT][CR], const AF (&a)[MT], const BF (&b)[NT]) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int j0 = 2 * p, j1 = 2 * p + 1;
#pragma unroll
            for (int pass = 0; pass < 3; ++pass)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const auto& A = a[mt];
                        const auto& B = b[nt];
                        if (pass == 0)
                            tmma(c[mt][nt], A.h[0][j0], A.h[1][j0], A.h[0][j1], A.h[1][j1], B.l[j0], B.l[j1]);
                        else if (pass == 1)
                            tmma(c[mt][nt], A.l[0][j0], A.l[1][j0], A.l[0][j1], A.l[1][j1], B.h[j0], B.h[j1]);
                        else
                            tmma(c[mt][nt], A.h[0][j0], A.h[1][j0], A.h[0][j1], A.h[1][j1], B.h[j0], B.h[j1]);
                    }
        }
    }
    template <int MT, int NT, int MTA>
    __device__ static __forceinline__ void mma16_group(W (&c)[MTA][NT][CR], const AF (&a)[MTA], const BF (&b)[NT]) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int j0 = 2 * p, j1 = 2 * p + 1;
#pragma unroll
            for (int pass = 0; pass < 3; ++pass)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const auto& A = a[mt];
                        const auto& B = b[nt];
                        if (pass == 0)
                            tmma(c[mt][nt], A.h[0][j0], A.h[1][j0], A.h[0][j1], A.h[1][j1], B.l[j0], B.l[j1]);
                        else if (pass == 1)
                            tmma(c[mt][nt], A.l[0][j0], A.l[1][j0], A.l[0][j1], A.l[1][j1], B.h[j0], B.h[j1]);
                        else
                            tmma(c[mt][nt], A.h[0][j0], A.h[1][j0], A.h[0][j1], A.h[1][j1], B.h[j0], B.h[j1]);
                    }
        }
    }
    template <int MT, int NT>
    __device__ static __forceinline__ void mmau_tile(W (&c)[MT][NT][CR], const AUF (&a)[MT], const BUF (&b)[NT]) {
#pragma unroll
        for (int pass = 0; pass < 3; ++pass)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const auto& A = a[mt];
                    const auto& B = b[nt];
                    if (pass == 0)
                        tmma(c[mt][nt], A.h[0][0], A.h[1][0], A.h[0][1], A.h[1][1], B.l[0], B.l[1]);
                    else if (pass == 1)
                        tmma(c[mt][nt], A.l[0][0], A.l[1][0], A.l[0][1], A.l[1][1], B.h[0], B.h[1]);
                    else
                        tmma(c[mt][nt], A.h[0][0], A.h[1][0], A.h[0][1], A.h[1][1], B.h[0], B.h[1]);
                }
    }
};

// Byte offset of element e (of n per lane, fb bytes each) of `lane` inside a
// 32-lane fragment block.  A lane holding <= 16 B keeps them contiguous (lanes
// consecutive); wider lanes are split into 16-byte units stored unit-major
// ([unit][lane][16 B]).  Either way every warp-wide vector load of a block is
// one contiguous, bank-conflict-free sweep.
__host__ __device__ __forceinline__ int frag_byte(int lane, int e, int fb, int n) {
    const int lb = n * fb;
    if (lb <= 16) return lane * lb + e * fb;
    const int byte = e * fb;
    return (byte >> 4) * 512 + lane * 16 + (byte & 15);
}

// Fragment-order index (elements) of X element (row r < 256, column q < ncol)
// for a CTA holding nct n-tiles: block [r/16][q/8] of 32 lanes x 4 values,
// lane = 4*(q%8) + (r/4)%4, value r%4.
template <typename W>
__device__ __forceinline__ int xfrag(int r, int q, int nct) {
    const int lane = ((q & 7) << 2) | ((r >> 2) & 3);
    return ((r >> 4) * nct + (q >> 3)) * 128 + frag_byte(lane, r & 3, (int)sizeof(W), 4) / (int)sizeof(W);
}

// Fragment slabs use their own bijection of a 16-wide k-block (any bijection
// works as long as both operands share it): the lane at k position tig holds,
// as its j-th value, row kperm_row(tig, j) = 2 tig + (j & 1) + 8 (j >> 1).  For a
// fixed j the four tig lanes then sit on rows with distinct (row & 7) / 2, which
// makes the B-fragment loads from a 128-byte-swizzled X tile (k_mr4_a)
// bank-conflict free.  Phase A only (A slab, k_mr2_a / k_mr3_a / k_mr4_a); phase B
// and the arena kernels keep rows 4 tig + j (measured: the bijection slows the
// phase-B stagers' fragment-order stores, 428 -> 446 us on cfg4).
__host__ __device__ __forceinline__ int kperm_row(int tig, int j) { return 2 * tig + (j & 1) + 8 * (j >> 1); }
__host__ __device__ __forceinline__ int kperm_tig(int r) { return (r & 7) >> 1; }
__host__ __device__ __forceinline__ int kperm_j(int r) { return (r & 1) | (((r >> 3) & 1) << 1); }
// xfrag with the slab bijection (row r of a 16-row block -> lane k position, value index)
template <typename W>
__device__ __forceinline__ int xfrag2(int r, int q, int nct) {
    const int lane = ((q & 7) << 2) | kperm_tig(r);
    return ((r >> 4) * nct + (q >> 3)) * 128 + frag_byte(lane, kperm_j(r), (int)sizeof(W), 4) / (int)sizeof(W);
}

// A lane's B fragment (4 values) of block `blk` (128 elements).
template <typename W>
__device__ __forceinline__ void load_bfrag(const W* blk, int lane, W (&bv)[4]) {
    if constexpr (sizeof(W) == 8) {
        const double2 d0 = reinterpret_cast<const double2*>(blk)[lane];
        const double2 d1 = reinterpret_cast<const double2*>(blk)[32 + lane];
        bv[0] = d0.x; bv[1] = d0.y; bv[2] = d1.x; bv[3] = d1.y;
    } else {
        const float4 u0 = reinterpret_cast<const float4*>(blk)[lane];
        bv[0] = u0.x; bv[1] = u0.y; bv[2] = u0.z; bv[3] = u0.w;
    }
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
        xs[xfrag<W>(r, q, nct)] = v;
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
                W bv[4];
                load_bfrag<W>(xs + (kb * nct + nt) * 128, lane, bv);
                typename Pol::AF af;
                typename Pol::BF bf;
                Pol::prep_a(af, av);
                Pol::prep_b(bf, bv);
                Pol::mma16(acc, af, bf);
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
                    if (c < L.rv_max && q0 + q < spad)  // the last column group may overhang spad
                        partial[(L.part_rows + slot * L.rv_pad + c) * spad + q0 + q] = my[i];
                    my[i] = W(0);
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ MR
// grid.x = nodes, grid.y = tiles of 256 (c, q) coefficients: T[c][q] = sum
// over the node's slots in CTA order (fixed order: deterministic).
// nodes with more slots than this are summed by 8 warps per coefficient tile (k_mr_reduce)
constexpr int kMrBigSlots = 32;
template <typename W>
__global__ void __launch_bounds__(256) k_mr_reduce(PlanView p, const __grid_constant__ MrView m, int node_lo,
                                                   int64_t s, int spad, const W* __restrict__ partial,
                                                   W* __restrict__ tbuf, W* __restrict__ send,
                                                   const int32_t* __restrict__ list, int nbig = 0, int ty_big = 0,
                                                   int ty_small = 0) {
    // ty_big > 0: ONE 1-D launch over the listed nodes, the first nbig (many
    // slots) with ty_big tiles each, the others with ty_small (no idle CTAs, one
    // launch instead of two); else grid (nodes, tiles)
    int bx = blockIdx.x, by = blockIdx.y, gy = gridDim.y;
    if (ty_big > 0) {
        if (bx < nbig * ty_big) {
            by = bx % ty_big;
            bx /= ty_big;
            gy = ty_big;
        } else {
            bx -= nbig * ty_big;
            by = bx % ty_small;
            bx = nbig + bx / ty_small;
            gy = ty_small;
        }
    }
    const int node = list ? list[bx] : node_lo + bx;
    const NodeDesc nd = p.nodes[node];
    const MrSlot sl = m.slots[node];
    const MrLevel L = m.lev[sl.lv];
    const int64_t cnt = (int64_t)nd.rv * s;
    // external level of a sharded handle: this rank's partial goes to the send
    // buffer, zero-padded to the level's slot width
    const bool ext = nd.ext_slot >= 0;
    W* dst = ext ? send + (int64_t)nd.ext_slot * s : tbuf + nd.t_off * s;
    const int64_t cnt_out = ext ? (int64_t)L.ext_w * s : cnt;
    const int64_t stride = (int64_t)L.rv_pad * spad;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nb = sl.b1 - sl.b0 + 1;
    const int64_t i0 = (int64_t)by * 256;
    if (nb <= kMrBigSlots) {
        if (i0 >= cnt_out) return;
        // few slots: one thread per coefficient, slots in order
        for (int64_t i = i0 + threadIdx.x; i < cnt_out; i += (int64_t)gy * 256) {
            W acc = W(0);
            if (i < cnt) {
                const int64_t c = i / s, q = i - c * s;
                const W* src = partial + (L.part_rows + (int64_t)(sl.b0 + sl.jrel) * L.rv_pad + c) * spad + q;
                int b = 0;
                for (; b + 8 <= nb; b += 8) {  // 8 loads in flight, additions in slot order
                    W v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = src[(int64_t)(b + u) * stride];
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc += v[u];
                }
                for (; b < nb; ++b) acc += src[(int64_t)b * stride];
            }
            dst[i] = acc;
        }
        return;
    }
    // many slots (upper levels): a CTA owns 32 consecutive coefficients per step (one 128/256-byte
    // row segment of every slot: coalesced).  Warp w sums slots w, w + 8, ... in order, four loads
    // in flight; the 8 warp sums are combined in warp order through shared memory (deterministic).
    __shared__ W red[8][33];
    for (int64_t base = (int64_t)by * 32; base < cnt_out; base += (int64_t)gy * 32) {
        const int64_t i = base + lane;
        W acc = W(0);
        if (i < cnt) {
            const int64_t c = i / s, q = i - c * s;
            const W* src = partial + (L.part_rows + (int64_t)(sl.b0 + sl.jrel) * L.rv_pad + c) * spad + q;
            int bb = warp;
            for (; bb + 24 < nb; bb += 32) {
                const W v0 = src[(int64_t)bb * stride], v1 = src[(int64_t)(bb + 8) * stride];
                const W v2 = src[(int64_t)(bb + 16) * stride], v3 = src[(int64_t)(bb + 24) * stride];
                acc += v0;
                acc += v1;
                acc += v2;
                acc += v3;
            }
            for (; bb < nb; bb += 8) acc += src[(int64_t)bb * stride];
        }
        red[warp][lane] = acc;
        __syncthreads();
        if (warp == 0 && i < cnt_out) {
            W t = red[0][lane];
#pragma unroll
            for (int w = 1; w < 8; ++w) t += red[w][lane];
            dst[i] = t;
        }
        __syncthreads();
    }
}

inline dim3 reduce_grid(const MrView& m, int node_lo, int nnodes_total, int64_t s) {
    int rmax = 0;
    for (int lv = 0; lv < m.nlev; ++lv) {
        rmax = rmax > m.lev[lv].rv_max ? rmax : m.lev[lv].rv_max;
        rmax = rmax > m.lev[lv].ext_w ? rmax : m.lev[lv].ext_w;
    }
    // y tiles of 8 coefficients (one per warp) for many-slot nodes; the
    // one-thread-per-coefficient nodes use tiles of 256 (extra CTAs exit)
    const int64_t tiles = ((int64_t)rmax * s + 7) / 8;
    return dim3(nnodes_total - node_lo, (unsigned)(tiles < 1 ? 1 : tiles > 2048 ? 2048 : tiles));
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
            typename Pol::AF af[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) Pol::prep_a(af[mt], av[mt]);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                W bv[4];
                load_bfrag<W>(xs + (kb * NT + nt) * 128, lane, bv);
                typename Pol::BF bf;
                Pol::prep_b(bf, bv);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) Pol::mma16(acc[mt][nt], af[mt], bf);
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
            typename Pol::AUF af[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) Pol::prep_au(af[mt], av[mt]);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                W bv[Pol::UV];
#pragma unroll
                for (int u = 0; u < Pol::UV; ++u)
                    bv[u] = ts[base + ((step * NT + nt) * 32 + lane) * Pol::UV + u];
                typename Pol::BUF bf;
                Pol::prep_bu(bf, bv);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) Pol::mmau(acc[mt][nt], af[mt], bf);
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

// ================================================================== slab path
// Relayout kernels (create time): arena -> fragment slabs.  Pure byte moves of
// already-quantised values (no rounding), zero fill for padding.
template <class Pol>
__global__ void k_slab_a(PlanView p, const __grid_constant__ Mr2View v, uint8_t* __restrict__ slab, int* __restrict__ special) {
    // one thread per (chunk, task, k-block, lane, a): 4 consecutive rows of one V' column
    const int64_t per_chunk = (int64_t)v.ntasks * 16 * 32 * Pol::AR;
    const int64_t total = per_chunk * p.nchunks;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int chunk = (int)(i / per_chunk);
        int64_t r = i - (int64_t)chunk * per_chunk;
        const int a = (int)(r % Pol::AR);
        r /= Pol::AR;
        const int lane = (int)(r % 32);
        r /= 32;
        const int kb = (int)(r % 16);
        const int t = (int)(r / 16);
        const int fb = fmt_bytes(v.task_fmt[t]);
        uint8_t* blk = slab + (int64_t)chunk * v.a_chunk_bytes + (int64_t)kb * v.arow + v.task_off[t];
        const int m = t * Pol::MR + (lane >> 2) + 8 * a;  // stacked row
        const int lv = v.row_lv[m], c = v.row_c[m];
        const ChunkDesc ch = p.chunks[chunk];
        const NodeDesc* nd = lv >= 0 ? &p.nodes[p.chunk_nodes[chunk * p.nlev + lv]] : nullptr;
        for (int j = 0; j < 4; ++j) {
            const int row = kb * 16 + kperm_row(lane & 3, j);
            uint8_t* dst = blk + frag_byte(lane, a * 4 + j, fb, Pol::AR * 4);
            if (nd && c < nd->rv) {
                const uint8_t* src = p.arena + nd->v_off + ((int64_t)c * nd->v_ld + (ch.row0 - nd->row0) + row) * fb;
                for (int b = 0; b < fb; ++b) dst[b] = src[b];
                if (fb < 8 && f32_special(__float_as_uint((float)dec_any(v.task_fmt[t], src, 0)))) *special = 1;
            } else {
                for (int b = 0; b < fb; ++b) dst[b] = 0;
            }
        }
    }
}

template <class Pol>
__global__ void k_slab_b(PlanView p, const __grid_constant__ Mr2View v, uint8_t* __restrict__ slab, int* __restrict__ special) {
    constexpr int MT = kBRows / Pol::MR;
    // D part: one thread per (chunk, warp, kb, mt, lane, a): 4 consecutive leaf columns
    const int64_t dper = (int64_t)kBWarps * 16 * MT * 32 * Pol::AR;
    const int64_t dtotal = dper * p.nchunks;
    const int lfb = fmt_bytes(v.leaf_fmt);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dtotal; i += (int64_t)gridDim.x * blockDim.x) {
        const int chunk = (int)(i / dper);
        int64_t r = i - (int64_t)chunk * dper;
        const int a = (int)(r % Pol::AR); r /= Pol::AR;
        const int lane = (int)(r % 32); r /= 32;
        const int mt = (int)(r % MT); r /= MT;
        const int kb = (int)(r % 16);
        const int w = (int)(r / 16);
        const ChunkDesc ch = p.chunks[chunk];
        const LeafDesc lf = p.leaves[ch.leaf];
        const int row = (ch.row0 - lf.row0) + kBRows * w + mt * Pol::MR + (lane >> 2) + 8 * a;
        uint8_t* blk = slab + (int64_t)chunk * v.b_chunk_bytes + ((int64_t)kb * kBWarps + w) * v.d_item +
                       (int64_t)mt * 32 * Pol::AR * 4 * lfb;
        for (int j = 0; j < 4; ++j) {
            const int col = kb * 16 + 4 * (lane & 3) + j;  // (phase B keeps rows 4 tig + j: its X / T staging stores are faster that way)
            const uint8_t* src = p.arena + lf.off + ((int64_t)row * lf.ld + col) * lfb;
            uint8_t* dst = blk + frag_byte(lane, a * 4 + j, lfb, Pol::AR * 4);
            for (int b = 0; b < lfb; ++b) dst[b] = src[b];
            if (lfb < 8 && f32_special(__float_as_uint((float)dec_any(v.leaf_fmt, src, 0)))) *special = 1;
        }
    }
    if (v.ustack) {
        // stacked U: one thread per (chunk, warp, k-block, mt, lane, a): 4 consecutive stacked columns
        const int fb = fmt_bytes(v.ufmt_all);
        const int64_t uper = (int64_t)kBWarps * v.nku * MT * 32 * Pol::AR;
        const int64_t utotal = uper * p.nchunks;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < utotal; i += (int64_t)gridDim.x * blockDim.x) {
            const int chunk = (int)(i / uper);
            int64_t r = i - (int64_t)chunk * uper;
            const int a = (int)(r % Pol::AR); r /= Pol::AR;
            const int lane = (int)(r % 32); r /= 32;
            const int mt = (int)(r % MT); r /= MT;
            const int kb = (int)(r % v.nku);
            const int w = (int)(r / v.nku);
            const ChunkDesc ch = p.chunks[chunk];
            uint8_t* blk = slab + (int64_t)chunk * v.b_chunk_bytes + 16LL * kBWarps * v.d_item +
                           ((int64_t)kb * kBWarps + w) * v.u_item + (int64_t)mt * 32 * Pol::AR * 4 * fb;
            for (int j = 0; j < 4; ++j) {
                const int sc = kb * 16 + 4 * (lane & 3) + j;
                const int lv = v.urow_lv[sc], c = v.urow_c[sc];
                uint8_t* dst = blk + frag_byte(lane, a * 4 + j, fb, Pol::AR * 4);
                bool put = false;
                if (lv >= 0) {
                    const NodeDesc nd = p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
                    if (c < nd.ru) {
                        const int row = (ch.row0 - nd.row0) + kBRows * w + mt * Pol::MR + (lane >> 2) + 8 * a;
                        const uint8_t* src = p.arena + nd.u_off + ((int64_t)c * nd.u_ld + row) * fb;
                        for (int b = 0; b < fb; ++b) dst[b] = src[b];
                        if (fb < 8 && f32_special(__float_as_uint((float)dec_any(v.ufmt_all, src, 0)))) *special = 1;
                        put = true;
                    }
                }
                if (!put)
                    for (int b = 0; b < fb; ++b) dst[b] = 0;
            }
        }
        return;
    }
    // U part: one thread per (chunk, warp, level, step, mt, lane, a, u): one element
    int64_t uper = 0;
    for (int lv = v.lev_lo; lv < v.nlev; ++lv) uper += (int64_t)v.lev[lv].steps * MT * 32 * Pol::AR * Pol::UV;
    const int64_t utotal = uper * kBWarps * p.nchunks;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < utotal; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cw = i / uper;
        int64_t r = i - cw * uper;
        const int chunk = (int)(cw / kBWarps), w = (int)(cw % kBWarps);
        int lv = v.lev_lo;
        for (;; ++lv) {
            const int64_t c = (int64_t)v.lev[lv].steps * MT * 32 * Pol::AR * Pol::UV;
            if (r < c) break;
            r -= c;
        }
        const int u = (int)(r % Pol::UV); r /= Pol::UV;
        const int a = (int)(r % Pol::AR); r /= Pol::AR;
        const int lane = (int)(r % 32); r /= 32;
        const int mt = (int)(r % MT);
        const int step = (int)(r / MT);
        const Mr2Level L = v.lev[lv];
        const int fb = fmt_bytes(L.ufmt);
        const ChunkDesc ch = p.chunks[chunk];
        const NodeDesc nd = p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
        const int row = (ch.row0 - nd.row0) + kBRows * w + mt * Pol::MR + (lane >> 2) + 8 * a;
        const int c = step * Pol::KU + Pol::UV * (lane & 3) + u;
        uint8_t* dst = slab + (int64_t)chunk * v.b_chunk_bytes + 16LL * kBWarps * v.d_item + L.uoff +
                       ((int64_t)step * kBWarps + w) * L.usz + (int64_t)mt * 32 * Pol::AR * Pol::UV * fb +
                       frag_byte(lane, a * Pol::UV + u, fb, Pol::AR * Pol::UV);
        if (c < nd.ru) {
            const uint8_t* src = p.arena + nd.u_off + ((int64_t)c * nd.u_ld + row) * fb;
            for (int b = 0; b < fb; ++b) dst[b] = src[b];
            if (fb < 8 && f32_special(__float_as_uint((float)dec_any(L.ufmt, src, 0)))) *special = 1;
        } else {
            for (int b = 0; b < fb; ++b) dst[b] = 0;
        }
    }
}

// float -> W.  FW: binary64 widening with integer ops instead of F2F.F64.F32
// (exponent re-biased by 896, mantissa shifted by 29, zero kept zero; exact when
// the slabs hold no fp32 subnormal / inf / nan, which is checked when they are
// built).  An experiment (HODLR_B200_FASTWIDEN=1): measured slightly SLOWER than
// the conversion instruction on cfg4 (the extra integer instructions cost more
// issue slots than F2F costs pipe time), so it is off by default.
template <typename W, bool FW>
__device__ __forceinline__ W widen(float f) {
    if constexpr (sizeof(W) == 8 && FW) {
        const uint32_t u = __float_as_uint(f), t = u & 0x7fffffffu;
        uint32_t h = __umulhi(t, 0x20000000u) + 0x38000000u;  // (t >> 3) + (896 << 20)
        h = t ? h : 0u;
        return (W)__hiloint2double((int)(h | (u & 0x80000000u)), (int)(u << 29));
    } else {
        return (W)f;
    }
}

// A lane's N values of a fragment block (layout of frag_byte), decoded to W.
template <typename W, int N, bool FW = false>
__device__ __forceinline__ void frag_load(int fmt, const uint8_t* blk, int lane, W (&v)[N]) {
    switch (fmt) {
        case HODLR_FMT_FP64:
            if constexpr (N == 1) {
                v[0] = (W) reinterpret_cast<const double*>(blk)[lane];
            } else {
#pragma unroll
                for (int u = 0; u < N / 2; ++u) {
                    const double2 d = reinterpret_cast<const double2*>(blk + u * 512)[lane];
                    v[2 * u] = (W)d.x;
                    v[2 * u + 1] = (W)d.y;
                }
            }
            break;
        case HODLR_FMT_FP32:
            if constexpr (N == 1) {
                v[0] = widen<W, FW>(reinterpret_cast<const float*>(blk)[lane]);
            } else if constexpr (N == 2) {
                const float2 f = reinterpret_cast<const float2*>(blk)[lane];
                v[0] = widen<W, FW>(f.x); v[1] = widen<W, FW>(f.y);
            } else {
#pragma unroll
                for (int u = 0; u < N / 4; ++u) {
                    const float4 f = reinterpret_cast<const float4*>(blk + u * 512)[lane];
                    v[4 * u] = widen<W, FW>(f.x); v[4 * u + 1] = widen<W, FW>(f.y); v[4 * u + 2] = widen<W, FW>(f.z); v[4 * u + 3] = widen<W, FW>(f.w);
                }
            }
            break;
        case HODLR_FMT_FP16:
        case HODLR_FMT_BF16: {
            uint32_t w[(N + 1) / 2];
            if constexpr (N == 1) {
                w[0] = reinterpret_cast<const uint16_t*>(blk)[lane];
            } else if constexpr (N == 2) {
                w[0] = reinterpret_cast<const uint32_t*>(blk)[lane];
            } else if constexpr (N == 4) {
                const uint2 t = reinterpret_cast<const uint2*>(blk)[lane];
                w[0] = t.x; w[1] = t.y;
            } else {
#pragma unroll
                for (int u = 0; u < N / 8; ++u) {
                    const uint4 t = reinterpret_cast<const uint4*>(blk + u * 512)[lane];
                    w[4 * u] = t.x; w[4 * u + 1] = t.y; w[4 * u + 2] = t.z; w[4 * u + 3] = t.w;
                }
            }
            const bool bf = fmt == HODLR_FMT_BF16;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const uint16_t h = (uint16_t)(w[i / 2] >> (16 * (i & 1)));
                v[i] = widen<W, FW>(bf ? __uint_as_float((uint32_t)h << 16) : dec_fp16(h));
            }
            break;
        }
        default: {  // q52
            uint32_t w[(N + 3) / 4];
            if constexpr (N == 1) {
                w[0] = blk[lane];
            } else if constexpr (N == 2) {
                w[0] = reinterpret_cast<const uint16_t*>(blk)[lane];
            } else if constexpr (N == 4) {
                w[0] = reinterpret_cast<const uint32_t*>(blk)[lane];
            } else if constexpr (N == 8) {
                const uint2 t = reinterpret_cast<const uint2*>(blk)[lane];
                w[0] = t.x; w[1] = t.y;
            } else {
#pragma unroll
                for (int u = 0; u < N / 16; ++u) {
                    const uint4 t = reinterpret_cast<const uint4*>(blk + u * 512)[lane];
                    w[4 * u] = t.x; w[4 * u + 1] = t.y; w[4 * u + 2] = t.z; w[4 * u + 3] = t.w;
                }
            }
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = widen<W, FW>(dec_q52((uint8_t)(w[i / 4] >> (8 * (i & 3)))));
            break;
        }
    }
}

constexpr int kRingMax = 8;  // max slots per warp ring (runtime depth ns <= kRingMax)

// ------------------------------------------------------------------ per-warp ring
// A warp-private ring of `ns` slots of `slot` bytes, filled by lane 0 with
// cp.async.bulk (complete_tx on the slot's mbarrier).  Items are consumed in
// order; the consumer state (slot, phase parity) advances by one per item.  An
// item is released -- its slot refilled with the producer's next item -- right
// after the warp has READ its last sub-block into registers, before the math,
// so ns items stay in flight.
struct WarpRing {
    uint64_t* bar;
    uint8_t* buf;
    int ns, slot;
    int cs = 0;
    unsigned cph = 0;
    __device__ __forceinline__ const uint8_t* wait() const {
        tma::mbar_wait(&bar[cs], cph);
        return buf + cs * slot;
    }
    __device__ __forceinline__ int advance() {
        const int k = cs;
        if (++cs == ns) {
            cs = 0;
            cph ^= 1u;
        }
        return k;
    }
    __device__ __forceinline__ void fill(int k, const void* src, unsigned bytes, uint64_t pol) const {
        tma::mbar_arrive_tx(&bar[k], bytes);
        tma::bulk_g2s(buf + k * slot, src, bytes, &bar[k], pol);
    }
};

__device__ __forceinline__ void cp_async(void* dst, const void* src, int bytes) {
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(tma::smem_u32(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tma::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Asynchronous stage_x (cp.async, element copies into fragment order); zero
// padding is stored directly.  Complete after cp_async_wait_all + a barrier.
template <typename W>
__device__ __forceinline__ void stage_x_async(W* xs, const W* __restrict__ x, int64_t ldx, int64_t r0, int nrows,
                                              int64_t q0, int ncol, int64_t s) {
    const int nct = ncol >> 3;
    for (int i = threadIdx.x; i < kChunk * ncol; i += blockDim.x) {
        const int r = i / ncol, q = i - r * ncol;
        W* dst = xs + xfrag<W>(r, q, nct);
        if (r < nrows && q0 + q < s)
            cp_async(dst, x + (r0 + r) * ldx + q0 + q, (int)sizeof(W));
        else
            *dst = W(0);
    }
}

// ------------------------------------------------------------------ MA2
// Persistent-range phase A over the A slab (CTA b: chunks [c_beg, c_end)).
//   warps 0..15  compute: warp w owns tasks t = w, w+16, ... (m-tiles of all
//                levels, <= MAXTW each), accumulators in registers per chunk,
//                then in a shared-memory tile per task across the chunks of one
//                node, flushed to the node's partial slot at its last chunk;
//   warp 16      producer: the run's A bytes are ONE contiguous range, streamed
//                in stages of G k-steps (all tasks) through a CTA-wide ring;
//   warp 17      stager: X of the next chunk (cp.async, fragment order).
constexpr int kAStagers = 4;  // X staging warps of the phase-A CTA
// Split-K factor of phase A: with few tasks (stacked m-tiles), KS warps share a
// task, warp w taking the k-steps kb = kp (mod KS); their accumulator tiles are
// summed in kp order at a row's flush (deterministic).  KS * ntasks <= kAWarps.
__host__ __device__ __forceinline__ int ma2_ks(int ntasks) {
    int ks = 1;
    while (ks < 16 && ntasks * ks * 2 <= kAWarps) ks *= 2;
    return ks;
}
constexpr int kAThreads = (kAWarps + 1 + kAStagers) * 32;

template <class Pol, int NCT, int MAXTW>
__global__ void __launch_bounds__(kAThreads) k_mr2_a(PlanView p, const __grid_constant__ MrView m,
                                                    const __grid_constant__ Mr2View v,
                                                    const typename Pol::W* __restrict__ x, int64_t ldx,
                                                    int64_t s, int spad, int G, int ns,
                                                    typename Pol::W* __restrict__ partial,
                                                    typename Pol::W* __restrict__ tbuf) {
    using W = typename Pol::W;
    constexpr int ncol = NCT * 8;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [kRingMax]
    uint64_t* empty = full + kRingMax;
    uint64_t* xfull = empty + kRingMax;                      // [2]
    uint64_t* xempty = xfull + 2;
    uint64_t* rawfull = xempty + 2;                          // [1]
    const int stage_bytes = G * v.arow;
    uint8_t* ring = smem_raw + 256;
    W* xsb = reinterpret_cast<W*>(ring + (size_t)ns * stage_bytes);  // [2][256 x ncol]
    W* accs = xsb + 2 * kChunk * ncol;                              // [task][NCT][32][CR]
    W* xraw = accs + (size_t)v.ntasks * ma2_ks(v.ntasks) * NCT * 32 * Pol::CR;  // [256 x ncol] row-major
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q0 = (int64_t)blockIdx.y * ncol;
    const int c_beg = (int)((int64_t)blockIdx.x * p.nchunks / gridDim.x);
    const int c_end = (int)((int64_t)(blockIdx.x + 1) * p.nchunks / gridDim.x);
    const int nst = 16 / G;  // stages per chunk

    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) {
            tma::mbar_init(&full[i], 1);
            tma::mbar_init(&empty[i], kAWarps);
        }
        for (int i = 0; i < 2; ++i) {
            tma::mbar_init(&xfull[i], 32 * kAStagers);
            tma::mbar_init(&xempty[i], kAWarps);
        }
        tma::mbar_init(rawfull, 1);
        tma::fence_mbar_init();
    }
    __syncthreads();

    if (warp == kAWarps) {
        // ---------------- producer
        if (lane == 0) {
            const uint64_t pol = tma::policy_evict_first();
            int slot = 0;
            unsigned ph = 0;
            int64_t n = 0;
            const uint8_t* src = v.slab_a + (int64_t)c_beg * v.a_chunk_bytes;
            const int64_t total = (int64_t)(c_end - c_beg) * nst;
            for (int64_t i = 0; i < total; ++i, ++n, src += stage_bytes) {
                if (n >= ns) tma::mbar_wait(&empty[slot], ph ^ 1u);
                tma::mbar_arrive_tx(&full[slot], (unsigned)stage_bytes);
                tma::bulk_g2s(ring + (size_t)slot * stage_bytes, src, (unsigned)stage_bytes, &full[slot], pol);
                if (++slot == ns) {
                    slot = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    if (warp > kAWarps) {
        // ---------------- stagers
        const int sl = threadIdx.x - (kAWarps + 1) * 32;
        // Contiguous X chunks (all columns of a row-major X with ldx = ncol): one
        // bulk copy of the chunk into a raw row-major buffer, then a shared-memory
        // permutation into fragment order (destination-ordered: conflict-free
        // stores), instead of ncol x 256 element cp.async requests through L1/L2.
        const bool raw_ok = q0 == 0 && ldx == ncol && s >= ncol && (((uintptr_t)x) & 15) == 0;
        if (raw_ok) {
            auto issue = [&](int ci) {
                if (sl == 0) {
                    const ChunkDesc ch = p.chunks[ci];
                    const unsigned bytes = (unsigned)(ch.nrows * ncol * sizeof(W));
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // raw reads done (barrier) before the refill
                    tma::mbar_arrive_tx(rawfull, bytes);
                    tma::bulk_g2s_plain(xraw, x + ch.row0 * ldx, bytes, rawfull);
                }
            };
            if (c_beg < c_end) issue(c_beg);
            for (int ci = c_beg; ci < c_end; ++ci) {
                const int k = ci - c_beg, buf = k & 1, use = k >> 1;
                if (use > 0) tma::mbar_wait(&xempty[buf], (unsigned)((use - 1) & 1));
                tma::mbar_wait(rawfull, (unsigned)(k & 1));
                const int nrows = p.chunks[ci].nrows;
                W* xs = xsb + buf * kChunk * ncol;
                for (int d = sl; d < kChunk * ncol; d += 32 * kAStagers) {
                    // inverse of xfrag: element d of fragment order -> (r, q)
                    const int blk = d >> 7, o = d & 127;
                    int ln, e;
                    if constexpr (sizeof(W) == 8) {
                        ln = (o & 63) >> 1;
                        e = ((o >> 6) << 1) | (o & 1);
                    } else {
                        ln = o >> 2;
                        e = o & 3;
                    }
                    const int r = 16 * (blk / NCT) + kperm_row(ln & 3, e);
                    const int q = 8 * (blk % NCT) + (ln >> 2);
                    xs[d] = r < nrows ? xraw[r * ncol + q] : W(0);
                }
                asm volatile("bar.sync 15, %0;" ::"r"(32 * kAStagers) : "memory");  // raw fully read
                if (ci + 1 < c_end) issue(ci + 1);
                asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tma::smem_u32(&xfull[buf]))
                             : "memory");
            }
            return;
        }
        for (int ci = c_beg; ci < c_end; ++ci) {
            const int k = ci - c_beg, buf = k & 1, use = k >> 1;
            if (use > 0) tma::mbar_wait(&xempty[buf], (unsigned)((use - 1) & 1));
            const ChunkDesc ch = p.chunks[ci];
            W* xs = xsb + buf * kChunk * ncol;
            for (int i = sl; i < kChunk * ncol; i += 32 * kAStagers) {
                const int r = i / ncol, q = i - r * ncol;
                W* dst = xs + xfrag2<W>(r, q, NCT);
                if (r < ch.nrows && q0 + q < s)
                    cp_async(dst, x + (ch.row0 + r) * ldx + q0 + q, (int)sizeof(W));
                else
                    *dst = W(0);
            }
            cp_async_wait_all();
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tma::smem_u32(&xfull[buf]))
                         : "memory");
        }
        return;
    }

    // ---------------- compute warps
    const int g = lane >> 2, tig = lane & 3;
    // KS > 1 only with MAXTW == 1: warp = task * KS + kp, tile index = warp
    const int KS = MAXTW == 1 ? ma2_ks(v.ntasks) : 1;
    const int kp = warp & (KS - 1), wtask = KS > 1 ? warp / KS : warp;
    int toff[MAXTW], tfmt[MAXTW];
    int ntw = 0;
#pragma unroll
    for (int i = 0; i < MAXTW; ++i) {
        const int t = wtask + i * kAWarps;
        toff[i] = 0;
        tfmt[i] = HODLR_FMT_FP32;
        if (t < v.ntasks) {
            toff[i] = v.task_off[t];
            tfmt[i] = v.task_fmt[t];
            ntw = i + 1;
        }
    }
#pragma unroll
    for (int i = 0; i < MAXTW; ++i)
        if (i < ntw)
#pragma unroll
            for (int nt = 0; nt < NCT; ++nt)
#pragma unroll
                for (int e = 0; e < Pol::CR; ++e)
                    accs[((((size_t)(warp + i * kAWarps)) * NCT + nt) * 32 + lane) * Pol::CR + e] = W(0);
    int slot = 0;
    unsigned ph = 0;
    for (int ci = c_beg; ci < c_end; ++ci) {
        const int k = ci - c_beg, buf = k & 1;
        tma::mbar_wait(&xfull[buf], (unsigned)((k >> 1) & 1));
        const W* xs = xsb + buf * kChunk * ncol;
        W acc[MAXTW][1][NCT][Pol::CR];
#pragma unroll
        for (int i = 0; i < MAXTW; ++i)
#pragma unroll
            for (int nt = 0; nt < NCT; ++nt)
#pragma unroll
                for (int e = 0; e < Pol::CR; ++e) acc[i][0][nt][e] = W(0);
        for (int gi = 0; gi < nst; ++gi) {
            tma::mbar_wait(&full[slot], ph);
            const uint8_t* base = ring + (size_t)slot * stage_bytes;
            // this warp's k-steps of the stage: kb = gi * G + kk with kb = kp (mod KS)
            const int kk0 = ((kp - gi * G) % KS + KS) % KS;
            for (int kk = ntw > 0 ? kk0 : G; kk < G; kk += KS) {
                const int kb = gi * G + kk;
                W tmp[MAXTW][Pol::AR * 4];
#pragma unroll
                for (int i = 0; i < MAXTW; ++i)
                    if (i < ntw) frag_load<W, Pol::AR * 4>(tfmt[i], base + kk * v.arow + toff[i], lane, tmp[i]);
                typename Pol::BF bf[NCT];
#pragma unroll
                for (int nt = 0; nt < NCT; ++nt) {
                    W bv[4];
                    load_bfrag<W>(xs + (kb * NCT + nt) * 128, lane, bv);
                    Pol::prep_b(bf[nt], bv);
                }
#pragma unroll
                for (int i = 0; i < MAXTW; ++i)
                    if (i < ntw) {
                        W av[Pol::AR][4];
#pragma unroll
                        for (int a = 0; a < Pol::AR; ++a)
#pragma unroll
                            for (int j = 0; j < 4; ++j) av[a][j] = tmp[i][a * 4 + j];
                        typename Pol::AF af[1];
                        Pol::prep_a(af[0], av);
                        Pol::template mma16_tile<1, NCT>(acc[i], af, bf);
                    }
            }
            // stage read (the A fragments are in registers): release it
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&empty[slot]);
            if (++slot == ns) {
                slot = 0;
                ph ^= 1u;
            }
        }
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&xempty[buf]);
        // accumulate into the task tiles; flush a row at its level node's last chunk of this run
#pragma unroll
        for (int i = 0; i < MAXTW; ++i) {
            if (i >= ntw) continue;
            const int t = wtask + i * kAWarps;
            const int tile = KS > 1 ? warp : t;
            bool more_a[Pol::AR], direct_a[Pol::AR];
            int64_t dst_a[Pol::AR];  // element offset of column q0 in tbuf / partial
            bool anyflush = false;
#pragma unroll
            for (int a = 0; a < Pol::AR; ++a) {
                // accumulator elements e with (e >> 1) == a belong to stacked row m
                const int srow = t * Pol::MR + g + 8 * a;
                const int lv = v.row_lv[srow], c = v.row_c[srow];
                bool more = true, direct = false;
                int64_t dst = -1;
                if (lv >= 0) {
                    const int node = p.chunk_nodes[ci * p.nlev + lv];
                    more = ci + 1 < c_end && p.chunk_nodes[(ci + 1) * p.nlev + lv] == node;
                    if (!more) {
                        const MrSlot sl = m.slots[node];
                        const NodeDesc nd = p.nodes[node];
                        // a node inside this CTA's run has one slot: its sum IS the coefficient
                        if (sl.b0 == sl.b1 && nd.ext_slot < 0) {
                            direct = true;
                            if (c < nd.rv) dst = nd.t_off * s + (int64_t)c * s + q0;
                        } else {
                            const MrLevel L = m.lev[lv];
                            if (c < L.rv_max) dst = (L.part_rows + ((int64_t)blockIdx.x + sl.jrel) * L.rv_pad + c) * spad + q0;
                        }
                    }
                }
                more_a[a] = more;
                direct_a[a] = direct;
                dst_a[a] = dst;
                anyflush |= !more;
            }
            auto store = [&](int a, int nt, int e, W val) {
                const int q = nt * 8 + 2 * tig + (e & 1);
                if (dst_a[a] >= 0) {
                    if (direct_a[a]) {
                        if (q0 + q < s) tbuf[dst_a[a] + q] = val;
                    } else if (q0 + q < spad) {
                        partial[dst_a[a] + q] = val;
                    }
                }
            };
            if (KS == 1) {
#pragma unroll
                for (int a = 0; a < Pol::AR; ++a)
#pragma unroll
                    for (int nt = 0; nt < NCT; ++nt) {
                        W* my = accs + (((size_t)tile * NCT + nt) * 32 + lane) * Pol::CR;
#pragma unroll
                        for (int e = 0; e < Pol::CR; ++e) {
                            if ((e >> 1) != a) continue;
                            const W val = my[e] + acc[i][0][nt][e];
                            if (more_a[a]) {
                                my[e] = val;
                            } else {
                                store(a, nt, e, val);
                                my[e] = W(0);
                            }
                        }
                    }
                continue;
            }
            // split-K: every warp of the task adds its chunk sums to its own tile;
            // at a flush the kp = 0 warp sums the KS tiles in kp order
#pragma unroll
            for (int nt = 0; nt < NCT; ++nt) {
                W* my = accs + (((size_t)tile * NCT + nt) * 32 + lane) * Pol::CR;
#pragma unroll
                for (int e = 0; e < Pol::CR; ++e) my[e] += acc[i][0][nt][e];
            }
            // same rows and chunk for the KS warps of a task: a uniform decision
            if (__any_sync(0xffffffffu, anyflush)) {
                asm volatile("bar.sync %0, %1;" ::"r"(1 + wtask), "r"(32 * KS) : "memory");
                if (kp == 0) {
#pragma unroll
                    for (int a = 0; a < Pol::AR; ++a) {
                        if (more_a[a]) continue;
#pragma unroll
                        for (int nt = 0; nt < NCT; ++nt)
#pragma unroll
                            for (int e = 0; e < Pol::CR; ++e) {
                                if ((e >> 1) != a) continue;
                                W val = W(0);
                                for (int k = 0; k < KS; ++k)
                                    val += accs[((((size_t)(tile + k)) * NCT + nt) * 32 + lane) * Pol::CR + e];
                                store(a, nt, e, val);
                            }
                    }
                }
                asm volatile("bar.sync %0, %1;" ::"r"(1 + wtask), "r"(32 * KS) : "memory");
#pragma unroll
                for (int a = 0; a < Pol::AR; ++a) {
                    if (more_a[a]) continue;
#pragma unroll
                    for (int nt = 0; nt < NCT; ++nt) {
                        W* my = accs + (((size_t)tile * NCT + nt) * 32 + lane) * Pol::CR;
#pragma unroll
                        for (int e = 0; e < Pol::CR; ++e)
                            if ((e >> 1) == a) my[e] = W(0);
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------ MA3
// Phase A with the reduction index split across the warps (contiguous X, i.e.
// s = ncol = ldx: the BASELINE multi-RHS shape).  Same A slab, same run
// partition and partial slots as k_mr2_a, different work split:
//   warps 0..7   compute: warp w owns k-blocks 2w, 2w+1 (chunk rows 32w..32w+31)
//                of EVERY task (m-tile) of every chunk, so it reads each A
//                fragment and its own 32 rows of X exactly once -- X needs no
//                fragment-order staging (the warp reads its B fragments straight
//                from the row-major bytes the bulk copy delivered) -- and keeps
//                one accumulator tile per task in registers ACROSS chunks.  The
//                raw operands of a chunk are pulled into registers first and the
//                ring stage released before the conversions and MMAs start;
//   warp 8       producer: per chunk, H = 16/KH stages of [KH k-steps of the A
//                slab | the matching 16*KH rows of X], two bulk copies per stage;
//   warp 9       reducer: when a node of some level ends (or the CTA's run does),
//                the compute warps park the affected accumulator tile in shared
//                memory (a few buffers, mbarrier hand-off, no CTA-wide barrier)
//                and carry on; the reducer sums the tiles in warp order
//                (deterministic) and stores the finished rows to the coefficient
//                buffer or the node's partial slot.
// A CTA takes R consecutive runs of the plan's partition (slots are per run).
// Which levels end at which chunk, and where their rows go, is resolved once
// per CTA into a shared-memory table before the first chunk (no dependent
// global loads on the per-chunk path).  AFMT >= 0: every task is stored in that
// format (no per-task format dispatch in the inner loop).
constexpr int kA3Kpw = 1;                      // k-blocks per compute warp
constexpr int kA3Warps = 16 / kA3Kpw;
constexpr int kA3Red = 2;                      // reducer warps (parked tiles round-robin; 1: 112 us, 2: 102, 3: 106 on cfg4)
constexpr int kA3Threads = (kA3Warps + 1 + kA3Red) * 32;
constexpr int kA3ParkMax = 8;                  // parking buffers (runtime depth npark <= kA3ParkMax)
constexpr bool kA3Prefetch = kA3Kpw > 1;       // raw operands of a chunk to registers, stage released before the MMAs
constexpr int kA3G = 1;                        // tiles whose MMAs are interleaved (independent accumulators)

template <class Pol, int NCT>
__host__ __device__ constexpr int ma3_red_elems() { return NCT * 32 * Pol::CR; }  // one tile, one warp

struct A3Dst {           // destination of a level's rows at a chunk where its node ends
    int64_t base;        // element offset of (column 0, rhs 0) in tbuf (direct) or partial
    int32_t clim;        // stored columns: c < clim
    int32_t direct;      // 1: the sum is the coefficient (tbuf, stride s); 0: partial slot (stride spad)
};

// raw (stored-format) A fragment of one k-block: AR * 4 values per lane
template <int AFMT, int N>
struct A3Raw {
    static constexpr int kWords = AFMT == HODLR_FMT_FP64 ? 2 * N : AFMT == HODLR_FMT_FP32 ? N : AFMT == HODLR_FMT_Q52 ? (N + 3) / 4 : (N + 1) / 2;
    uint32_t w[kWords];
};
template <int AFMT, int N>
__device__ __forceinline__ void a3_load_raw(const uint8_t* blk, int lane, A3Raw<AFMT, N>& r) {
    constexpr int bytes = A3Raw<AFMT, N>::kWords * 4;  // per lane
    if constexpr (bytes <= 16) {
        if constexpr (bytes == 16) {
            const uint4 t = reinterpret_cast<const uint4*>(blk)[lane];
            r.w[0] = t.x; r.w[1] = t.y; r.w[2] = t.z; r.w[3] = t.w;
        } else if constexpr (bytes == 8) {
            const uint2 t = reinterpret_cast<const uint2*>(blk)[lane];
            r.w[0] = t.x; r.w[1] = t.y;
        } else {
            r.w[0] = reinterpret_cast<const uint32_t*>(blk)[lane];
        }
    } else {
#pragma unroll
        for (int u = 0; u < bytes / 16; ++u) {
            const uint4 t = reinterpret_cast<const uint4*>(blk + u * 512)[lane];
            r.w[4 * u] = t.x; r.w[4 * u + 1] = t.y; r.w[4 * u + 2] = t.z; r.w[4 * u + 3] = t.w;
        }
    }
}
template <typename W, int AFMT, int N, bool FW>
__device__ __forceinline__ void a3_decode(const A3Raw<AFMT, N>& r, W (&v)[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if constexpr (AFMT == HODLR_FMT_FP64) {
            v[i] = (W)__hiloint2double((int)r.w[2 * i + 1], (int)r.w[2 * i]);
        } else if constexpr (AFMT == HODLR_FMT_FP32) {
            v[i] = widen<W, FW>(__uint_as_float(r.w[i]));
        } else if constexpr (AFMT == HODLR_FMT_BF16) {
            v[i] = widen<W, FW>(__uint_as_float((r.w[i / 2] >> (16 * (i & 1))) << 16));
        } else if constexpr (AFMT == HODLR_FMT_FP16) {
            v[i] = widen<W, FW>(dec_fp16((uint16_t)(r.w[i / 2] >> (16 * (i & 1)))));
        } else {
            v[i] = widen<W, FW>(dec_q52((uint8_t)(r.w[i / 4] >> (8 * (i & 3)))));
        }
    }
}

template <class Pol, int NCT, int MAXT, int AFMT, bool FW>
__global__ void __launch_bounds__(kA3Threads, 1) k_mr3_a(PlanView p, const __grid_constant__ MrView m,
                                                        const __grid_constant__ Mr2View v,
                                                        const typename Pol::W* __restrict__ x, int64_t s, int spad,
                                                        int KH, int ns, int R, int nloc_max, int npark, int dbg,
                                                        typename Pol::W* __restrict__ partial,
                                                        typename Pol::W* __restrict__ tbuf) {
    using W = typename Pol::W;
    constexpr int ncol = NCT * 8;
    constexpr int RE = ma3_red_elems<Pol, NCT>();
    constexpr int NA = Pol::AR * 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [kRingMax]
    uint64_t* empty = full + kRingMax;                       // [kRingMax]
    uint64_t* rfull = empty + kRingMax;                      // [kA3ParkMax]
    uint64_t* rfree = rfull + kA3ParkMax;                    // [kA3ParkMax]
    unsigned* s_tmask = reinterpret_cast<unsigned*>(rfree + kA3ParkMax);      // [MAXT] levels present in a task's rows
    int8_t* s_rowlv = reinterpret_cast<int8_t*>(s_tmask + MAXT);           // [MAXT * MR] level of a stacked row
    const int a_bytes = KH * v.arow, x_bytes = KH * 16 * ncol * (int)sizeof(W);
    const int stage_bytes = a_bytes + x_bytes;
    uint8_t* ring = smem_raw + 640;  // barriers + tables: 128 + 128 + 32 + 128 bytes
    W* red = reinterpret_cast<W*>(ring + (size_t)ns * stage_bytes);       // [npark][kA3Warps][RE]
    A3Dst* s_dst = reinterpret_cast<A3Dst*>(red + (size_t)npark * kA3Warps * RE);  // [nloc][nlev]
    unsigned* s_mask = reinterpret_cast<unsigned*>(s_dst + (size_t)nloc_max * p.nlev);  // [nloc] levels ending
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = 16 / KH;
    const int nch = p.nchunks, nb = m.nb;
    const int vb0 = blockIdx.x * R, vb1 = min(vb0 + R, nb);
    if (vb0 >= nb) return;
    const int C0 = (int)((int64_t)vb0 * nch / nb), C1 = (int)((int64_t)vb1 * nch / nb);

    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) {
            tma::mbar_init(&full[i], 1);
            tma::mbar_init(&empty[i], KH / kA3Kpw);
        }
        for (int i = 0; i < npark; ++i) {
            tma::mbar_init(&rfull[i], kA3Warps);
            tma::mbar_init(&rfree[i], 1);
        }
        tma::fence_mbar_init();
    }
    if (threadIdx.x < MAXT * Pol::MR) {
        const int t = threadIdx.x / Pol::MR;
        s_rowlv[threadIdx.x] = (int8_t)(t < v.ntasks ? v.row_lv[threadIdx.x] : -1);
    }
    if (threadIdx.x < MAXT) {
        unsigned tm = 0;
        if ((int)threadIdx.x < v.ntasks)
            for (int r = 0; r < Pol::MR; ++r) {
                const int lv = v.row_lv[threadIdx.x * Pol::MR + r];
                if (lv >= 0) tm |= 1u << lv;
            }
        s_tmask[threadIdx.x] = tm;
    }
    __syncthreads();

    if (warp == kA3Warps) {
        // ---------------- producer
        if (lane == 0 && !(dbg & 32)) {
            const uint64_t pol = tma::policy_evict_first();
            int slot = 0;
            unsigned ph = 0;
            int64_t n = 0;
            for (int ci = C0; ci < C1; ++ci) {
                const uint8_t* asrc = v.slab_a + (int64_t)ci * v.a_chunk_bytes;
                const W* xsrc = x + (int64_t)ci * kChunk * ncol;
                for (int h = 0; h < H; ++h, ++n) {
                    if (n >= ns) tma::mbar_wait(&empty[slot], ph ^ 1u);
                    uint8_t* dst = ring + (size_t)slot * stage_bytes;
                    tma::mbar_arrive_tx(&full[slot], (unsigned)stage_bytes);
                    tma::bulk_g2s(dst, asrc + (int64_t)h * a_bytes, (unsigned)a_bytes, &full[slot], pol);
                    tma::bulk_g2s_plain(dst + a_bytes, xsrc + (int64_t)h * KH * 16 * ncol, (unsigned)x_bytes, &full[slot]);
                    if (++slot == ns) {
                        slot = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ---------------- flush table of this CTA's chunks -> shared memory (all but the producer)
    {
        const int nthr = (kA3Warps + kA3Red) * 32;
        const int tid = warp > kA3Warps ? (int)threadIdx.x - 32 : (int)threadIdx.x;
        for (int i = tid; i < (C1 - C0) * p.nlev; i += nthr) {
            const MrFlush f = m.flush[(size_t)C0 * p.nlev + i];
            A3Dst d;
            d.base = f.row * (f.direct ? s : (int64_t)spad);
            d.clim = f.clim;
            d.direct = f.direct;
            s_dst[i] = d;
        }
        for (int k = tid; k < C1 - C0; k += nthr) s_mask[k] = m.flush_mask[C0 + k];
        asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    }
    unsigned fl = 0;  // parked tiles so far (same sequence in every warp)

    if (warp > kA3Warps) {
        // ---------------- reducers: reducer ri takes parked tiles it = ri (mod kA3Red)
        const int ri = warp - (kA3Warps + 1);
        for (int ci = C0; ci < C1; ++ci) {
            const unsigned mask = (dbg & 2) ? (ci + 1 == C1 ? s_mask[ci - C0] : 0u) : s_mask[ci - C0];
            if (!mask) continue;
            const A3Dst* dk = s_dst + (size_t)(ci - C0) * p.nlev;
#pragma unroll
            for (int t = 0; t < MAXT; ++t) {
                if (!(s_tmask[t] & mask)) continue;
                // rows of the task whose level ends here
                unsigned rows = 0;
#pragma unroll
                for (int r = 0; r < Pol::MR; ++r) {
                    const int lv = s_rowlv[t * Pol::MR + r];
                    if (lv >= 0 && ((mask >> lv) & 1u)) rows |= 1u << r;
                }
                const unsigned it = fl++;
                if ((int)(it % kA3Red) != ri) continue;
                const int buf = it % npark;
                tma::mbar_wait(&rfull[buf], (it / npark) & 1u);
                const W* rb = red + (size_t)buf * kA3Warps * RE;
                // 32 / ncol rows per sweep, one (row, rhs) per lane
                const int sub = lane / ncol, col = lane % ncol;
                if (dbg & 16) rows = 0;
                while (rows) {
                    unsigned rr = rows;
                    for (int i = 0; i < sub && rr; ++i) rr &= rr - 1;
                    if (rr) {
                        const int row = __ffs(rr) - 1;
                        const int srow = t * Pol::MR + row;
                        const int lv = s_rowlv[srow], c = v.row_c[srow];
                        const A3Dst d = dk[lv];
                        const int e = ((row >> 3) << 1) | (col & 1);
                        const int e0 = (((col >> 3) * 32) + (row & 7) * 4 + ((col & 7) >> 1)) * Pol::CR + e;
                        // fixed pairwise tree over the warps (deterministic; short dependent
                        // chains: the adds queue behind the compute warps' DMMAs on the FP64 pipe)
                        W part[kA3Warps];
#pragma unroll
                        for (int w = 0; w < kA3Warps; ++w) part[w] = rb[(size_t)w * RE + e0];
#pragma unroll
                        for (int st = 1; st < kA3Warps; st *= 2)
#pragma unroll
                            for (int w = 0; w + st < kA3Warps; w += 2 * st) part[w] += part[w + st];
                        const W sum = part[0];
                        if (c < d.clim) {
                            if (d.direct) {
                                if (col < s) tbuf[d.base + (int64_t)c * s + col] = sum;
                            } else if (col < spad) {
                                partial[d.base + (int64_t)c * spad + col] = sum;
                            }
                        }
                    }
                    for (int i = 0; i < 32 / ncol && rows; ++i) rows &= rows - 1;
                }
                __syncwarp();
                if (lane == 0) tma::mbar_arrive(&rfree[buf]);
            }
        }
        return;
    }

    // ---------------- compute warps
    const int g = lane >> 2, tig = lane & 3;
    const int kb0 = kA3Kpw * warp;               // first k-block of this warp
    const int wl = kb0 % KH, h = kb0 / KH;       // position inside its stage, stage of the chunk
    constexpr int GT = kA3G, NG = MAXT / kA3G;   // tiles per group, groups
    W acc[NG][GT][NCT][Pol::CR];
#pragma unroll
    for (int gi = 0; gi < NG; ++gi)
#pragma unroll
        for (int t = 0; t < GT; ++t)
#pragma unroll
            for (int nt = 0; nt < NCT; ++nt)
#pragma unroll
                for (int e = 0; e < Pol::CR; ++e) acc[gi][t][nt][e] = W(0);
    const int ntasks = v.ntasks;
    int64_t sn = h;  // this warp's stage number: k * H + h
    for (int ci = C0; ci < C1; ++ci, sn += H) {
        const int slot = (int)(sn % ns);
        if (!(dbg & 32)) tma::mbar_wait(&full[slot], (unsigned)((sn / ns) & 1));
        const uint8_t* base = ring + (size_t)slot * stage_bytes;
        // raw operands of both k-blocks -> registers, then the stage goes back to the producer
        W bv[kA3Kpw][NCT][4];
        constexpr bool PF = kA3Prefetch && AFMT >= 0;
        A3Raw<AFMT < 0 ? HODLR_FMT_FP32 : AFMT, NA> raw[PF ? kA3Kpw : 1][PF ? MAXT : 1];
#pragma unroll
        for (int q = 0; q < kA3Kpw; ++q) {
            const W* xs = reinterpret_cast<const W*>(base + a_bytes) + 16 * (wl + q) * ncol + g;
#pragma unroll
            for (int nt = 0; nt < NCT; ++nt)
#pragma unroll
                for (int j = 0; j < 4; ++j) bv[q][nt][j] = xs[kperm_row(tig, j) * ncol + 8 * nt];
            if constexpr (PF) {
                const uint8_t* ab = base + (size_t)(wl + q) * v.arow;
#pragma unroll
                for (int t = 0; t < MAXT; ++t)
                    if (t < ntasks) a3_load_raw<AFMT, NA>(ab + v.task_off[t], lane, raw[q][t]);
            }
        }
        if constexpr (PF) {
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&empty[slot]);
        }
#pragma unroll
        for (int q = 0; q < kA3Kpw; ++q) {
            typename Pol::BF bf[NCT];
#pragma unroll
            for (int nt = 0; nt < NCT; ++nt) Pol::prep_b(bf[nt], bv[q][nt]);
            const uint8_t* ab = base + (size_t)(wl + q) * v.arow;
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {
                const int nt_g = ntasks - gi * GT;  // tiles of this group in use (uniform)
                if (nt_g <= 0) continue;
                typename Pol::AF af[GT];
#pragma unroll
                for (int i = 0; i < GT; ++i) {
                    const int t = gi * GT + i;
                    W tmp[NA];
                    if (i < nt_g) {
                        if constexpr (PF) {
                            a3_decode<W, AFMT, NA, FW>(raw[q][t], tmp);
                        } else if constexpr (AFMT >= 0) {
                            A3Raw<AFMT, NA> r1;
                            a3_load_raw<AFMT, NA>(ab + v.task_off[t], lane, r1);
                            a3_decode<W, AFMT, NA, FW>(r1, tmp);
                        } else {
                            frag_load<W, NA, FW>(v.task_fmt[t], ab + v.task_off[t], lane, tmp);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < NA; ++j) tmp[j] = W(0);
                    }
                    W av[Pol::AR][4];
#pragma unroll
                    for (int a = 0; a < Pol::AR; ++a)
#pragma unroll
                        for (int j = 0; j < 4; ++j) av[a][j] = tmp[a * 4 + j];
                    Pol::prep_a(af[i], av);
                }
                if (dbg & 1) continue;
                if (nt_g >= GT)
                    Pol::template mma16_group<GT, NCT, GT>(acc[gi], af, bf);
                else if (nt_g == 3)
                    Pol::template mma16_group<(GT > 3 ? 3 : GT), NCT, GT>(acc[gi], af, bf);
                else if (nt_g == 2)
                    Pol::template mma16_group<(GT > 2 ? 2 : GT), NCT, GT>(acc[gi], af, bf);
                else
                    Pol::template mma16_group<1, NCT, GT>(acc[gi], af, bf);
            }
        }
        if constexpr (!PF) {
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&empty[slot]);
        }
        const unsigned mask = (dbg & 2) ? (ci + 1 == C1 ? s_mask[ci - C0] : 0u) : s_mask[ci - C0];
        if (!mask) continue;
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
            if (!(s_tmask[t] & mask)) continue;
            const unsigned it = fl++;
            const int buf = it % npark;
            if ((int)it >= npark) tma::mbar_wait(&rfree[buf], ((it / npark) - 1) & 1u);
            W* my = red + ((size_t)buf * kA3Warps + warp) * RE + lane * Pol::CR;
            if (!(dbg & 8))
#pragma unroll
            for (int nt = 0; nt < NCT; ++nt)
#pragma unroll
                for (int e = 0; e < Pol::CR; ++e) {
                    // only the rows whose node ends are parked (the reducers read no others)
                    const int lv = s_rowlv[t * Pol::MR + g + 8 * (e >> 1)];
                    if (lv >= 0 && ((mask >> lv) & 1u)) {
                        my[nt * 32 * Pol::CR + e] = acc[t / GT][t % GT][nt][e];
                        acc[t / GT][t % GT][nt][e] = W(0);
                    }
                }
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&rfull[buf]);
        }
    }
}

// ------------------------------------------------------------------ MA4
// The K-split phase A with a 4 x 4 warp arrangement: warp (tg, kg) owns the
// tile group tg (tiles 2 tg, 2 tg + 1 of the stacked rows) and the k-blocks
// 4 kg .. 4 kg + 3 of every chunk.  Against k_mr3_a (16 k-blocks x all tiles per
// warp): 4 accumulator tiles per warp instead of 14-16 (no register spills under
// the 96-register cap of a 19-warp CTA), and a tile's partial sums live in only 4
// warps, so a parked tile is 4 pieces, not 16 -- and the deep levels, whose nodes
// end every chunk or two, all sit in the last tile group: per chunk only its 4
// warps (which carry half the MMA work when the tile count is odd) park anything.
// Every tile group has its own parking channel (buffers, barriers, counters);
// reducer r serves the groups g = r (mod kA3Red).  Same stages, producer, flush
// table, slots and summation determinism (fixed pairwise tree) as k_mr3_a.
// X rows (128 B for 16 fp64 right-hand sides) all start at the same bank, so the
// B-fragment loads (lanes = 8 columns x 4 rows) were 4-way bank conflicted and,
// with four tile-group warps re-reading each k-block's X, took ~70% of the
// shared-memory pipe.  With `use_tmap` the X tile of a stage arrives by ONE
// tensor-map bulk copy (cp.async.bulk.tensor.2d) with the 128-byte swizzle: the
// 16-byte unit of row r, column pair c/2 lands at unit (c/2) ^ (r & 7), which
// spreads a lane group's rows over the banks: with the slab's k bijection
// (kperm_row: the four tig lanes on rows with distinct (row & 7) / 2) the loads
// are bank-conflict free.
constexpr int kA4TG = 2;                       // tiles per group
constexpr int kA4NG = 4;                       // tile groups (MAXT = 8)
constexpr int kA4KG = 4;                       // k-blocks per warp
constexpr int kA4Park = 3;                     // parking buffers per channel

template <class Pol, int NCT, int AFMT, bool FW>
__global__ void __launch_bounds__(kA3Threads, 1) k_mr4_a(PlanView p, const __grid_constant__ MrView m,
                                                        const __grid_constant__ Mr2View v,
                                                        const typename Pol::W* __restrict__ x, int64_t s, int spad,
                                                        int KH, int ns, int R, int nloc_max,
                                                        typename Pol::W* __restrict__ partial,
                                                        typename Pol::W* __restrict__ tbuf,
                                                        const __grid_constant__ CUtensorMap tmx, int use_tmap) {
    using W = typename Pol::W;
    constexpr int MAXT = kA4TG * kA4NG;
    constexpr int ncol = NCT * 8;
    constexpr int RE = ma3_red_elems<Pol, NCT>();
    constexpr int NA = Pol::AR * 4;
    constexpr int NCH = kA4NG * kA4Park;     // parking buffers in all
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [kRingMax]
    uint64_t* empty = full + kRingMax;                       // [kRingMax]
    uint64_t* rfull = empty + kRingMax;                      // [NCH]
    uint64_t* rfree = rfull + NCH;                           // [NCH]
    unsigned* s_tmask = reinterpret_cast<unsigned*>(rfree + NCH);          // [MAXT]
    int8_t* s_rowlv = reinterpret_cast<int8_t*>(s_tmask + MAXT);           // [MAXT * MR]
    const int a_bytes = KH * v.arow, x_bytes = KH * 16 * ncol * (int)sizeof(W);
    const int stage_bytes = a_bytes + x_bytes;
    // (barriers + tables: 128 + 192 + 32 + 128 bytes; stages 1024-byte aligned for the swizzled X tiles)
    const uint32_t base_u32 = tma::smem_u32(smem_raw);
    uint8_t* ring = smem_raw + (((base_u32 + 640u + 1023u) & ~1023u) - base_u32);
    W* red = reinterpret_cast<W*>(ring + (size_t)ns * stage_bytes);       // [NG][kA4Park][4 warps][RE]
    A3Dst* s_dst = reinterpret_cast<A3Dst*>(red + (size_t)NCH * 4 * RE);   // [nloc][nlev]
    unsigned* s_mask = reinterpret_cast<unsigned*>(s_dst + (size_t)nloc_max * p.nlev);  // [nloc]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = 16 / KH;
    const int nch = p.nchunks, nb = m.nb;
    const int vb0 = blockIdx.x * R, vb1 = min(vb0 + R, nb);
    if (vb0 >= nb) return;
    const int C0 = (int)((int64_t)vb0 * nch / nb), C1 = (int)((int64_t)vb1 * nch / nb);

    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) {
            tma::mbar_init(&full[i], 1);
            tma::mbar_init(&empty[i], KH);   // (KH / 4 k-groups) x 4 tile groups
        }
        for (int i = 0; i < NCH; ++i) {
            tma::mbar_init(&rfull[i], kA4KG);
            tma::mbar_init(&rfree[i], 1);
        }
        tma::fence_mbar_init();
    }
    if (threadIdx.x < MAXT * Pol::MR) {
        const int t = threadIdx.x / Pol::MR;
        s_rowlv[threadIdx.x] = (int8_t)(t < v.ntasks ? v.row_lv[threadIdx.x] : -1);
    }
    if (threadIdx.x < MAXT) {
        unsigned tm = 0;
        if ((int)threadIdx.x < v.ntasks)
            for (int r = 0; r < Pol::MR; ++r) {
                const int lv = v.row_lv[threadIdx.x * Pol::MR + r];
                if (lv >= 0) tm |= 1u << lv;
            }
        s_tmask[threadIdx.x] = tm;
    }
    __syncthreads();

    if (warp == kA3Warps) {
        // ---------------- producer (as k_mr3_a)
        if (lane == 0) {
            const uint64_t pol = tma::policy_evict_first();
            int slot = 0;
            unsigned ph = 0;
            int64_t n = 0;
            for (int ci = C0; ci < C1; ++ci) {
                const uint8_t* asrc = v.slab_a + (int64_t)ci * v.a_chunk_bytes;
                const W* xsrc = x + (int64_t)ci * kChunk * ncol;
                for (int h = 0; h < H; ++h, ++n) {
                    if (n >= ns) tma::mbar_wait(&empty[slot], ph ^ 1u);
                    uint8_t* dst = ring + (size_t)slot * stage_bytes;
                    tma::mbar_arrive_tx(&full[slot], (unsigned)stage_bytes);
                    tma::bulk_g2s(dst, asrc + (int64_t)h * a_bytes, (unsigned)a_bytes, &full[slot], pol);
                    if (use_tmap)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                                "r"(tma::smem_u32(dst + a_bytes)),
                            "l"(reinterpret_cast<uint64_t>(&tmx)), "r"(0), "r"(ci * kChunk + h * KH * 16), "r"(tma::smem_u32(&full[slot]))
                            : "memory");
                    else
                        tma::bulk_g2s_plain(dst + a_bytes, xsrc + (int64_t)h * KH * 16 * ncol, (unsigned)x_bytes, &full[slot]);
                    if (++slot == ns) {
                        slot = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ---------------- flush table of this CTA's chunks -> shared memory (all but the producer)
    {
        const int nthr = (kA3Warps + kA3Red) * 32;
        const int tid = warp > kA3Warps ? (int)threadIdx.x - 32 : (int)threadIdx.x;
        for (int i = tid; i < (C1 - C0) * p.nlev; i += nthr) {
            const MrFlush f = m.flush[(size_t)C0 * p.nlev + i];
            A3Dst d;
            d.base = f.row * (f.direct ? s : (int64_t)spad);
            d.clim = f.clim;
            d.direct = f.direct;
            s_dst[i] = d;
        }
        for (int k = tid; k < C1 - C0; k += nthr) s_mask[k] = m.flush_mask[C0 + k];
        asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    }

    if (warp > kA3Warps) {
        // ---------------- reducers: reducer ri serves the tile groups g = ri (mod kA3Red)
        const int ri = warp - (kA3Warps + 1);
        unsigned fl[kA4NG];
#pragma unroll
        for (int g_ = 0; g_ < kA4NG; ++g_) fl[g_] = 0;
        for (int ci = C0; ci < C1; ++ci) {
            const unsigned mask = s_mask[ci - C0];
            if (!mask) continue;
            const A3Dst* dk = s_dst + (size_t)(ci - C0) * p.nlev;
#pragma unroll
            for (int t = 0; t < MAXT; ++t) {
                const int grp = t / kA4TG;
                if (grp % kA3Red != ri) continue;
                if (!(s_tmask[t] & mask)) continue;
                unsigned rows = 0;
#pragma unroll
                for (int r = 0; r < Pol::MR; ++r) {
                    const int lv = s_rowlv[t * Pol::MR + r];
                    if (lv >= 0 && ((mask >> lv) & 1u)) rows |= 1u << r;
                }
                const unsigned it = fl[grp]++;
                const int buf = grp * kA4Park + (int)(it % kA4Park);
                tma::mbar_wait(&rfull[buf], (it / kA4Park) & 1u);
                const W* rb = red + (size_t)buf * kA4KG * RE;
                const int sub = lane / ncol, col = lane % ncol;
                while (rows) {
                    unsigned rr = rows;
                    for (int i = 0; i < sub && rr; ++i) rr &= rr - 1;
                    if (rr) {
                        const int row = __ffs(rr) - 1;
                        const int srow = t * Pol::MR + row;
                        const int lv = s_rowlv[srow], c = v.row_c[srow];
                        const A3Dst d = dk[lv];
                        const int e = ((row >> 3) << 1) | (col & 1);
                        const int e0 = (((col >> 3) * 32) + (row & 7) * 4 + ((col & 7) >> 1)) * Pol::CR + e;
                        // fixed order (deterministic): (kg0 + kg1) + (kg2 + kg3)
                        const W sum = (rb[e0] + rb[RE + e0]) + (rb[2 * RE + e0] + rb[3 * RE + e0]);
                        if (c < d.clim) {
                            if (d.direct) {
                                if (col < s) tbuf[d.base + (int64_t)c * s + col] = sum;
                            } else if (col < spad) {
                                partial[d.base + (int64_t)c * spad + col] = sum;
                            }
                        }
                    }
                    for (int i = 0; i < 32 / ncol && rows; ++i) rows &= rows - 1;
                }
                __syncwarp();
                if (lane == 0) tma::mbar_arrive(&rfree[buf]);
            }
        }
        return;
    }

    // ---------------- compute warps: warp = tg * 4 + kg (one warp of every tile group per sub-partition)
    const int g = lane >> 2, tig = lane & 3;
    const int tg = warp >> 2, kg = warp & 3;
    const int kb0 = kA4KG * kg;                 // first k-block of this warp
    const int wl = kb0 % KH, h = kb0 / KH;      // position inside its stage, stage of the chunk
    const int t0 = tg * kA4TG;                  // first tile of the group
    const int nt_g = min(kA4TG, v.ntasks - t0); // tiles of the group in use
    W acc[kA4TG][NCT][Pol::CR];
#pragma unroll
    for (int i = 0; i < kA4TG; ++i)
#pragma unroll
        for (int nt = 0; nt < NCT; ++nt)
#pragma unroll
            for (int e = 0; e < Pol::CR; ++e) acc[i][nt][e] = W(0);
    int toff[kA4TG], tfmt[kA4TG];
#pragma unroll
    for (int i = 0; i < kA4TG; ++i) {
        toff[i] = i < nt_g ? v.task_off[t0 + i] : 0;
        tfmt[i] = i < nt_g ? v.task_fmt[t0 + i] : HODLR_FMT_FP32;
    }
    unsigned fl = 0;  // parked tiles of this group so far
    int64_t sn = h;   // this warp's stage number: k * H + h
    for (int ci = C0; ci < C1; ++ci, sn += H) {
        const int slot = (int)(sn % ns);
        tma::mbar_wait(&full[slot], (unsigned)((sn / ns) & 1));
        const uint8_t* base = ring + (size_t)slot * stage_bytes;
        if (nt_g > 0) {
#pragma unroll
            for (int q = 0; q < kA4KG; ++q) {
                const uint8_t* xt = base + a_bytes;
                const int r0 = 16 * (wl + q);
                typename Pol::BF bf[NCT];
#pragma unroll
                for (int nt = 0; nt < NCT; ++nt) {
                    W bv[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int r = r0 + kperm_row(tig, j), c = 8 * nt + g;
                        // swizzled tile: 16-byte unit (c / 2) of row r sits at unit (c / 2) ^ (r & 7)
                        const int off = use_tmap ? r * 128 + ((((c >> 1) ^ (r & 7)) << 4) | ((c & 1) << 3))
                                                 : (r * ncol + c) * (int)sizeof(W);
                        bv[j] = *reinterpret_cast<const W*>(xt + off);
                    }
                    Pol::prep_b(bf[nt], bv);
                }
                const uint8_t* ab = base + (size_t)(wl + q) * v.arow;
                typename Pol::AF af[kA4TG];
#pragma unroll
                for (int i = 0; i < kA4TG; ++i) {
                    W tmp[NA];
                    if (i < nt_g) {
                        if constexpr (AFMT >= 0) {
                            A3Raw<AFMT, NA> r1;
                            a3_load_raw<AFMT, NA>(ab + toff[i], lane, r1);
                            a3_decode<W, AFMT, NA, FW>(r1, tmp);
                        } else {
                            frag_load<W, NA, FW>(tfmt[i], ab + toff[i], lane, tmp);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < NA; ++j) tmp[j] = W(0);
                    }
                    W av[Pol::AR][4];
#pragma unroll
                    for (int a = 0; a < Pol::AR; ++a)
#pragma unroll
                        for (int j = 0; j < 4; ++j) av[a][j] = tmp[a * 4 + j];
                    Pol::prep_a(af[i], av);
                }
                if (nt_g >= kA4TG)
                    Pol::template mma16_group<kA4TG, NCT, kA4TG>(acc, af, bf);
                else
                    Pol::template mma16_group<1, NCT, kA4TG>(acc, af, bf);
            }
        }
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&empty[slot]);
        const unsigned mask = s_mask[ci - C0];
        if (!mask) continue;
#pragma unroll
        for (int i = 0; i < kA4TG; ++i) {
            const int t = t0 + i;
            if (!(s_tmask[t] & mask)) continue;   // (s_tmask is 0 for unused tiles)
            const unsigned it = fl++;
            const int buf = tg * kA4Park + (int)(it % kA4Park);
            if (it >= (unsigned)kA4Park) tma::mbar_wait(&rfree[buf], ((it / kA4Park) - 1) & 1u);
            W* my = red + ((size_t)buf * kA4KG + kg) * RE + lane * Pol::CR;
#pragma unroll
            for (int nt = 0; nt < NCT; ++nt)
#pragma unroll
                for (int e = 0; e < Pol::CR; ++e) {
                    const int lv = s_rowlv[t * Pol::MR + g + 8 * (e >> 1)];
                    if (lv >= 0 && ((mask >> lv) & 1u)) {
                        my[nt * 32 * Pol::CR + e] = acc[i][nt][e];
                        acc[i][nt][e] = W(0);
                    }
                }
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&rfull[buf]);
        }
    }
}

// ------------------------------------------------------------------ MB2
// Persistent: CTA b takes works (chunk, column group) b, b + grid, ...
//   warps 0..15  compute: warp w owns chunk rows 16w..16w+15;
//   warp 16      producer: streams each work's B region through a CTA-wide
//                ring of ns stages (16 warps' D items of one k-step per stage,
//                then the U steps of every level), one cp.async.bulk per stage;
//   warp 17      stager: X and the coefficients of work k+1 into buffer
//                (k+1)&1 with cp.async while work k is computed.
// All hand-offs are mbarriers (full/empty per stage and per X buffer).
constexpr int kBStagers = 2;  // X / coefficient staging warps of the phase-B CTA
constexpr int kBThreads = (kBWarps + 1 + kBStagers) * 32;

template <class Pol, int NT, bool FW>
__global__ void __launch_bounds__(kBThreads) k_mr2_b(PlanView p, const __grid_constant__ MrView m,
                                                    const __grid_constant__ Mr2View v,
                                                    const typename Pol::W* __restrict__ x, int64_t ldx,
                                                    const typename Pol::W* __restrict__ tbuf,
                                                    typename Pol::W* __restrict__ b, int64_t ldb, int64_t s,
                                                    int ngrp, int ns, int trows, int nbuf, int chunk0, int chunk1) {
    using W = typename Pol::W;
    constexpr int MT = kBRows / Pol::MR;
    constexpr int ncol = NT * 8;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [kRingMax]
    uint64_t* empty = full + kRingMax;                       // [kRingMax]
    uint64_t* xfull = empty + kRingMax;                      // [2]
    uint64_t* xempty = xfull + 2;                            // [2]
    uint8_t* ring = smem_raw + (2 * kRingMax + 4) * 8 + 96;  // 128-aligned
    const int lslot = v.lslot, lstage = v.lslot + 4;         // stage = 16 D items
    const int stage_bytes = 1 << lstage;
    W* xsb = reinterpret_cast<W*>(ring + (size_t)ns * stage_bytes);  // [nbuf][256 x ncol]
    W* tsb = xsb + nbuf * kChunk * ncol;                            // [nbuf][trows x ncol]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int work0 = chunk0 * ngrp, nwork = chunk1 * ngrp;  // works [work0, nwork): chunks [chunk0, chunk1)
    const int64_t dbytes = 16LL << lstage;                           // D region of a chunk
    const int ustage = kBWarps * v.u_item;  // stacked U: one U k-block per stage
    const int nstage = v.ustack ? 16 + v.nku : 16 + (v.warp_bytes + stage_bytes - 1) / stage_bytes;

    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) {
            tma::mbar_init(&full[i], 1);
            tma::mbar_init(&empty[i], kBWarps);
        }
        for (int i = 0; i < 2; ++i) {
            tma::mbar_init(&xfull[i], 32 * kBStagers);
            tma::mbar_init(&xempty[i], kBWarps);
        }
        tma::fence_mbar_init();
    }
    __syncthreads();

    if (warp == kBWarps) {
        // ---------------- producer (one lane)
        if (lane == 0) {
            const uint64_t pol = tma::policy_evict_first();
            int slot = 0;
            unsigned ph = 0;
            int64_t n = 0;  // stages issued
            for (int work = work0 + blockIdx.x; work < nwork; work += gridDim.x) {
                const int chunk = ngrp == 1 ? work : work / ngrp;
                const uint8_t* src = v.slab_b + (int64_t)chunk * v.b_chunk_bytes;
                for (int st = 0; st < nstage; ++st, ++n) {
                    if (n >= ns) tma::mbar_wait(&empty[slot], ph ^ 1u);
                    int64_t off, bytes;
                    if (st < 16) {
                        off = (int64_t)st << lstage;
                        bytes = stage_bytes;
                    } else if (v.ustack) {
                        off = dbytes + (int64_t)(st - 16) * ustage;
                        bytes = ustage;
                    } else {
                        off = dbytes + ((int64_t)(st - 16) << lstage);
                        bytes = min((int64_t)stage_bytes, dbytes + v.warp_bytes - off);
                    }
                    tma::mbar_arrive_tx(&full[slot], (unsigned)bytes);
                    tma::bulk_g2s(ring + (size_t)slot * stage_bytes, src + off, (unsigned)bytes, &full[slot], pol);
                    if (++slot == ns) {
                        slot = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }
    if (warp > kBWarps) {
        // ---------------- stagers
        const int sl = threadIdx.x - (kBWarps + 1) * 32;
        int k = 0;
        for (int work = work0 + blockIdx.x; work < nwork; work += gridDim.x, ++k) {
            const int buf = nbuf == 2 ? (k & 1) : 0, use = nbuf == 2 ? (k >> 1) : k;
            if (use > 0) tma::mbar_wait(&xempty[buf], (unsigned)((use - 1) & 1));
            const int chunk = ngrp == 1 ? work : work / ngrp;
            const int64_t q0 = (int64_t)(work - chunk * ngrp) * ncol;
            const ChunkDesc ch = p.chunks[chunk];
            W* xs = xsb + buf * kChunk * ncol;
            for (int i = sl; i < kChunk * ncol; i += 32 * kBStagers) {
                const int r = i / ncol, q = i - r * ncol;
                W* dst = xs + xfrag<W>(r, q, NT);
                if (r < ch.nrows && q0 + q < s)
                    cp_async(dst, x + (ch.row0 + r) * ldx + q0 + q, (int)sizeof(W));
                else
                    *dst = W(0);
            }
            W* ts = tsb + buf * trows * ncol;
            if (v.ustack) {
                // coefficients of the stacked U columns, fragment order (like X)
                for (int i = sl; i < v.nku * 16 * ncol; i += 32 * kBStagers) {
                    const int r = i / ncol, q = i - r * ncol;
                    W* dst = ts + xfrag<W>(r, q, NT);
                    const int lv = v.urow_lv[r], c = v.urow_c[r];
                    bool put = false;
                    if (lv >= 0 && q0 + q < s) {
                        const NodeDesc* nd = &p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
                        if (c < nd->ru) {
                            cp_async(dst, tbuf + (nd->tsrc_off + c) * s + q0 + q, (int)sizeof(W));
                            put = true;
                        }
                    }
                    if (!put) *dst = W(0);
                }
            }
            int base = 0;
            for (int lv = v.ustack ? v.nlev : v.lev_lo; lv < v.nlev; ++lv) {
                const int steps = v.lev[lv].steps;
                if (steps == 0) continue;
                const NodeDesc nd = p.nodes[p.chunk_nodes[chunk * p.nlev + lv]];
                const W* t = tbuf + nd.tsrc_off * s;
                for (int i = sl; i < steps * Pol::KU * ncol; i += 32 * kBStagers) {
                    const int c = i / ncol, q = i - c * ncol;
                    const int step = c / Pol::KU, w = c - step * Pol::KU;
                    const int tg = w / Pol::UV, u = w - tg * Pol::UV;
                    W* dst = ts + base + ((step * NT + (q >> 3)) * 32 + (q & 7) * 4 + tg) * Pol::UV + u;
                    if (c < nd.ru && q0 + q < s)
                        cp_async(dst, t + (int64_t)c * s + q0 + q, (int)sizeof(W));
                    else
                        *dst = W(0);
                }
                base += steps * NT * 32 * Pol::UV;
            }
            cp_async_wait_all();
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tma::smem_u32(&xfull[buf]))
                         : "memory");
        }
        return;
    }

    // ---------------- compute warps
    const int g = lane >> 2, tig = lane & 3;
    int slot = 0;
    unsigned ph = 0;
    auto next_stage = [&]() -> const uint8_t* {
        tma::mbar_wait(&full[slot], ph);
        return ring + (size_t)slot * stage_bytes;
    };
    auto release_stage = [&]() {
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&empty[slot]);
        if (++slot == ns) {
            slot = 0;
            ph ^= 1u;
        }
    };
    const int lfmt = v.leaf_fmt;
    const int lfb = fmt_bytes(lfmt);
    int k = 0;
    for (int work = work0 + blockIdx.x; work < nwork; work += gridDim.x, ++k) {
        const int buf = nbuf == 2 ? (k & 1) : 0, use = nbuf == 2 ? (k >> 1) : k;
        const int chunk = ngrp == 1 ? work : work / ngrp;
        const int64_t q0 = (int64_t)(work - chunk * ngrp) * ncol;
        tma::mbar_wait(&xfull[buf], (unsigned)(use & 1));
        const W* xs = xsb + buf * kChunk * ncol;
        const W* ts = tsb + buf * trows * ncol;

        W acc[MT][NT][Pol::CR];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < Pol::CR; ++i) acc[mt][nt][i] = W(0);

        // D: stage kb holds every warp's item of k-step kb
        for (int kb = 0; kb < 16; ++kb) {
            const uint8_t* base = next_stage() + (warp << lslot);
            W tmp[MT][Pol::AR * 4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
                frag_load<W, Pol::AR * 4, FW>(lfmt, base + mt * 32 * Pol::AR * 4 * lfb, lane, tmp[mt]);
            release_stage();
            typename Pol::AF af[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                W av[Pol::AR][4];
#pragma unroll
                for (int a = 0; a < Pol::AR; ++a)
#pragma unroll
                    for (int j = 0; j < 4; ++j) av[a][j] = tmp[mt][a * 4 + j];
                Pol::prep_a(af[mt], av);
            }
            typename Pol::BF bf[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                W bv[4];
                load_bfrag<W>(xs + (kb * NT + nt) * 128, lane, bv);
                Pol::prep_b(bf[nt], bv);
            }
            Pol::template mma16_tile<MT, NT>(acc, af, bf);
        }
        // stacked U: nku more k-blocks, same shape as the D items
        if (v.ustack) {
            const int ufmt = v.ufmt_all;
            const int ufb = fmt_bytes(ufmt);
            for (int kb = 0; kb < v.nku; ++kb) {
                const uint8_t* base = next_stage() + warp * v.u_item;
                W tmp[MT][Pol::AR * 4];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
                    frag_load<W, Pol::AR * 4, FW>(ufmt, base + mt * 32 * Pol::AR * 4 * ufb, lane, tmp[mt]);
                release_stage();
                typename Pol::AF af[MT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    W av[Pol::AR][4];
#pragma unroll
                    for (int a = 0; a < Pol::AR; ++a)
#pragma unroll
                        for (int j = 0; j < 4; ++j) av[a][j] = tmp[mt][a * 4 + j];
                    Pol::prep_a(af[mt], av);
                }
                typename Pol::BF bf[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    W bv[4];
                    load_bfrag<W>(ts + (kb * NT + nt) * 128, lane, bv);
                    Pol::prep_b(bf[nt], bv);
                }
                Pol::template mma16_tile<MT, NT>(acc, af, bf);
            }
        }
        // U: per step, the 16 warps' blocks are adjacent; several steps per stage
        int tbase = 0;
        const uint8_t* sbase = nullptr;
        for (int lv = v.ustack ? v.nlev : v.lev_lo; lv < v.nlev; ++lv) {
            const Mr2Level& L = v.lev[lv];
            const int steps = L.steps;
            if (steps == 0) continue;
            const int ufmt = L.ufmt, usz = L.usz;
            const int ufb = fmt_bytes(ufmt);
            const int sstep = usz * kBWarps;
            int lo = L.ulo;
            for (int step = 0; step < steps; ++step, lo += sstep) {
                if (sbase == nullptr) sbase = next_stage();
                const uint8_t* base = sbase + (lo & (stage_bytes - 1)) + warp * usz;
                W tmp[MT][Pol::AR * Pol::UV];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
                    frag_load<W, Pol::AR * Pol::UV, FW>(ufmt, base + mt * 32 * Pol::AR * Pol::UV * ufb, lane, tmp[mt]);
                const int nlo = step + 1 < steps ? lo + sstep : L.unext;
                if (nlo < 0 || (nlo >> lstage) != (lo >> lstage)) {  // stage fully read
                    release_stage();
                    sbase = nullptr;
                }
                typename Pol::AUF af[MT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    W av[Pol::AR][Pol::UV];
#pragma unroll
                    for (int a = 0; a < Pol::AR; ++a)
#pragma unroll
                        for (int u = 0; u < Pol::UV; ++u) av[a][u] = tmp[mt][a * Pol::UV + u];
                    Pol::prep_au(af[mt], av);
                }
                typename Pol::BUF bf[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    W bv[Pol::UV];
#pragma unroll
                    for (int u = 0; u < Pol::UV; ++u) bv[u] = ts[tbase + ((step * NT + nt) * 32 + lane) * Pol::UV + u];
                    Pol::prep_bu(bf[nt], bv);
                }
                Pol::template mmau_tile<MT, NT>(acc, af, bf);
            }
            tbase += steps * NT * 32 * Pol::UV;
        }
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&xempty[buf]);
        const int row0 = p.chunks[chunk].row0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < Pol::CR; i += 2) {
                    const int row = warp * kBRows + mt * Pol::MR + g + 8 * (i >> 1);
                    const int64_t q = q0 + nt * 8 + 2 * tig;
                    W* dst = b + (int64_t)(row0 + row) * ldb + q;
                    if (q + 1 < s) {
                        dst[0] = acc[mt][nt][i];
                        dst[1] = acc[mt][nt][i + 1];
                    } else if (q < s) {
                        dst[0] = acc[mt][nt][i];
                    }
                }
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


// ---- slab path launchers
inline int pick_nt(int spad) { return spad >= 32 ? 4 : spad >= 16 ? 2 : 1; }

template <class Pol>
size_t ma2_smem(const Mr2View& v, int nct, int slot_bytes, int ns) {
    using W = typename Pol::W;
    return 256 + (size_t)3 * kChunk * nct * 8 * sizeof(W) + (size_t)v.ntasks * ma2_ks(v.ntasks) * nct * 32 * Pol::CR * sizeof(W) +
           (size_t)ns * slot_bytes;
}
template <class Pol>
int mb2_trows(const Mr2View& v) {
    if (v.ustack) return v.nku * 16;
    int trows = 0;
    for (int lv = v.lev_lo; lv < v.nlev; ++lv) trows += v.lev[lv].steps * Pol::KU;
    return trows;
}
template <class Pol>
size_t mb2_smem(const Mr2View& v, int nt, int ns, int nbuf = 2) {
    using W = typename Pol::W;
    return (2 * kRingMax + 4) * 8 + 96 + (size_t)ns * kBWarps * v.d_item +
           nbuf * ((size_t)kChunk + mb2_trows<Pol>(v)) * nt * 8 * sizeof(W);
}

template <class Pol, int NCT, int MAXTW>
cudaError_t launch_ma2_t(const PlanView& p, const MrView& m, const Mr2View& v, const typename Pol::W* x,
                         int64_t ldx, int64_t s, int spad, typename Pol::W* partial, typename Pol::W* tbuf,
                         cudaStream_t st) {
    // stage = G k-steps of every task, G * MAXTW * AR * 4 <= 16 values per lane
    int G = 16 / (MAXTW * Pol::AR);
    if (G < 1) G = 1;
    while (G > 1 && (size_t)G * v.arow > 32 * 1024) G /= 2;
    int ns = kRingMax;
    while (ns > 2 && ma2_smem<Pol>(v, NCT, G * v.arow, ns) > 225 * 1024) --ns;
    const size_t sm = ma2_smem<Pol>(v, NCT, G * v.arow, ns);
    if (sm > 227 * 1024) return cudaErrorInvalidConfiguration;
    auto k = k_mr2_a<Pol, NCT, MAXTW>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid(m.nb, (spad + NCT * 8 - 1) / (NCT * 8));
    k<<<grid, kAThreads, sm, st>>>(p, m, v, x, ldx, s, spad, G, ns, partial, tbuf);
    return cudaGetLastError();
}
template <class Pol, int NCT>
cudaError_t launch_ma2_n(const PlanView& p, const MrView& m, const Mr2View& v, const typename Pol::W* x,
                         int64_t ldx, int64_t s, int spad, typename Pol::W* partial, typename Pol::W* tbuf,
                         cudaStream_t st) {
    const int maxtw = (v.ntasks + kAWarps - 1) / kAWarps;
    if (maxtw <= 1) return launch_ma2_t<Pol, NCT, 1>(p, m, v, x, ldx, s, spad, partial, tbuf, st);
    if (maxtw <= 2) return launch_ma2_t<Pol, NCT, 2>(p, m, v, x, ldx, s, spad, partial, tbuf, st);
    return launch_ma2_t<Pol, NCT, 4>(p, m, v, x, ldx, s, spad, partial, tbuf, st);
}
// cuTensorMapEncodeTiled through the runtime (no libcuda link): a 2-D fp64 tensor
// [nrows][16] (128-byte rows), boxes of box_rows rows, 128-byte swizzle.
inline bool encode_x_tmap(CUtensorMap* tm, const void* x, uint64_t nrows, uint32_t box_rows) {
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            f = nullptr;
        }
        return (EncodeFn)f;
    }();
    if (!fn || box_rows > 256 || (((uintptr_t)x) & 15)) return false;
    const cuuint64_t dims[2] = {16, nrows};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {16, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(x), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K-split phase A (k_mr3_a): X contiguous (s = ldx = 8 or 16 columns), <= 8 tasks.
constexpr int kA3MaxT = 8;
template <class Pol, int NCT>
size_t ma3_smem(const Mr2View& v, int KH, int ns, int npark) {
    using W = typename Pol::W;
    return 640 + (size_t)ns * (KH * v.arow + KH * 16 * NCT * 8 * sizeof(W)) +
           (size_t)npark * kA3Warps * ma3_red_elems<Pol, NCT>() * sizeof(W);
}
inline size_t ma3_table_bytes(int nloc, int nlev) { return (size_t)nloc * nlev * sizeof(A3Dst) + (size_t)nloc * 4 + 16; }
template <class Pol, int NCT>
bool launch_ma3(const PlanView& p, const MrView& m, const Mr2View& v, const typename Pol::W* x, int64_t ldx,
                int64_t s, int spad, typename Pol::W* partial, typename Pol::W* tbuf, cudaStream_t st,
                cudaError_t* err) {
    if (s != NCT * 8 || ldx != s || spad != s || v.ntasks > kA3MaxT || v.ntasks < 1 || (((uintptr_t)x) & 15)) return false;
    if (const char* e = getenv("HODLR_B200_MA3"))
        if (e[0] == '0') return false;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int R = (m.nb + sms - 1) / sms;           // runs per CTA: one CTA per SM
    const int grid = (m.nb + R - 1) / R;
    const int nloc = (int)(((int64_t)p.nchunks * R + m.nb - 1) / m.nb) + 1;  // chunks per CTA, upper bound
    const size_t tab = ma3_table_bytes(nloc, p.nlev);
    if (tab > 32 * 1024) return false;
    const size_t budget = 225 * 1024 - tab;
    int KH = 8;
    if (const char* e = getenv("HODLR_B200_MA3_KH")) KH = atoi(e);
    if (KH != 4 && KH != 8 && KH != 16) KH = 8;  // (a multiple of kA3Kpw)
    int npark = 4;
    if (const char* e = getenv("HODLR_B200_MA3_PARK")) npark = std::max(kA3Red, std::min(kA3ParkMax, atoi(e)));  // >= kA3Red: a reducer is never two phases behind a buffer
    while (KH > 4 && ma3_smem<Pol, NCT>(v, KH, 3, npark) > budget) KH /= 2;
    int ns = kRingMax;
    while (ns > 2 && ma3_smem<Pol, NCT>(v, KH, ns, npark) > budget) --ns;
    if (const char* e = getenv("HODLR_B200_MA3_NS")) ns = std::max(2, std::min(ns, atoi(e)));
    const size_t sm = ma3_smem<Pol, NCT>(v, KH, ns, npark) + tab;
    if (sm > 227 * 1024 || ns < 16 / KH) return false;
    using W = typename Pol::W;
    // every task in one storage format (the usual case): the specialised instance
    int afmt = v.task_fmt[0];
    for (int t = 1; t < v.ntasks; ++t)
        if (v.task_fmt[t] != afmt) afmt = -1;
    if (sizeof(W) == 4 && afmt == HODLR_FMT_FP64) afmt = -1;
    if (const char* e = getenv("HODLR_B200_MA3_GENERIC"))
        if (e[0] == '1') afmt = -1;
    const bool fw = sizeof(W) == 8 && v.widen_fast && getenv("HODLR_B200_FASTWIDEN");  // measured slower than F2F (cfg4: 124 vs 120 us): off
    auto pick = [&](auto fwc) {
        constexpr bool F = decltype(fwc)::value;
        auto kk = k_mr3_a<Pol, NCT, kA3MaxT, -1, F>;
        switch (afmt) {
            case HODLR_FMT_Q52: kk = k_mr3_a<Pol, NCT, kA3MaxT, HODLR_FMT_Q52, F>; break;
            case HODLR_FMT_BF16: kk = k_mr3_a<Pol, NCT, kA3MaxT, HODLR_FMT_BF16, F>; break;
            case HODLR_FMT_FP16: kk = k_mr3_a<Pol, NCT, kA3MaxT, HODLR_FMT_FP16, F>; break;
            case HODLR_FMT_FP32: kk = k_mr3_a<Pol, NCT, kA3MaxT, HODLR_FMT_FP32, F>; break;
            case HODLR_FMT_FP64: kk = k_mr3_a<Pol, NCT, kA3MaxT, HODLR_FMT_FP64, F>; break;
            default: break;
        }
        return kk;
    };
    auto k = fw ? pick(std::true_type{}) : pick(std::false_type{});
    *err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (*err != cudaSuccess) return true;
    int dbg = 0;  // timing experiments only (results are wrong when set)
    if (const char* e = getenv("HODLR_B200_MA3_DBG")) dbg = atoi(e);
    bool use4 = true;
    if (const char* e = getenv("HODLR_B200_MA4")) use4 = e[0] != '0';
    if (use4) {
        // the 4 x 4 arrangement: its own parking geometry (4 channels x kA4Park buffers of 4 pieces)
        const size_t red4 = (size_t)kA4NG * kA4Park * kA4KG * ma3_red_elems<Pol, NCT>() * sizeof(W);
        const size_t stage = (size_t)KH * v.arow + (size_t)KH * 16 * NCT * 8 * sizeof(W);
        int ns4 = kRingMax;
        while (ns4 > 2 && 640 + 1024 + ns4 * stage + red4 > budget) --ns4;
        if (const char* e = getenv("HODLR_B200_MA3_NS")) ns4 = std::max(2, std::min(ns4, atoi(e)));
        const size_t sm4 = 640 + 1024 + ns4 * stage + red4 + tab;  // (+ slack: stages are 1024-byte aligned)
        if (sm4 <= 227 * 1024 && ns4 >= 16 / KH && KH >= kA4KG) {
            auto pick4 = [&](auto fwc) {
                constexpr bool F = decltype(fwc)::value;
                auto kk = k_mr4_a<Pol, NCT, -1, F>;
                switch (afmt) {
                    case HODLR_FMT_Q52: kk = k_mr4_a<Pol, NCT, HODLR_FMT_Q52, F>; break;
                    case HODLR_FMT_BF16: kk = k_mr4_a<Pol, NCT, HODLR_FMT_BF16, F>; break;
                    case HODLR_FMT_FP16: kk = k_mr4_a<Pol, NCT, HODLR_FMT_FP16, F>; break;
                    case HODLR_FMT_FP32: kk = k_mr4_a<Pol, NCT, HODLR_FMT_FP32, F>; break;
                    case HODLR_FMT_FP64: kk = k_mr4_a<Pol, NCT, HODLR_FMT_FP64, F>; break;
                    default: break;
                }
                return kk;
            };
            auto k4 = fw ? pick4(std::true_type{}) : pick4(std::false_type{});
            *err = cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
            if (*err != cudaSuccess) return true;
            // X tiles by tensor-map bulk copies with the 128-byte swizzle (fp64, 16 rhs: 128-byte rows)
            alignas(64) CUtensorMap tmx;
            memset(&tmx, 0, sizeof(tmx));
            int use_tmap = 0;
            if (sizeof(W) == 8 && NCT == 2 && ((size_t)KH * v.arow) % 1024 == 0 && !getenv("HODLR_B200_MA4_NO_TMAP"))
                use_tmap = encode_x_tmap(&tmx, x, (uint64_t)p.nchunks * kChunk, KH * 16) ? 1 : 0;
            k4<<<grid, kA3Threads, sm4, st>>>(p, m, v, x, s, spad, KH, ns4, R, nloc, partial, tbuf, tmx, use_tmap);
            *err = cudaGetLastError();
            return true;
        }
    }
    k<<<grid, kA3Threads, sm, st>>>(p, m, v, x, s, spad, KH, ns, R, nloc, npark, dbg, partial, tbuf);
    *err = cudaGetLastError();
    return true;
}

template <class Pol>
cudaError_t launch_ma2(const PlanView& p, const MrView& m, const Mr2View& v, const typename Pol::W* x,
                       int64_t ldx, int64_t s, int spad, typename Pol::W* partial, typename Pol::W* tbuf,
                       cudaStream_t st) {
    {
        cudaError_t e3 = cudaSuccess;
        if (spad == 16 && launch_ma3<Pol, 2>(p, m, v, x, ldx, s, spad, partial, tbuf, st, &e3)) return e3;
        if (spad == 8 && launch_ma3<Pol, 1>(p, m, v, x, ldx, s, spad, partial, tbuf, st, &e3)) return e3;
    }
    int nct = pick_nt(spad);
    while (nct > 1 && ma2_smem<Pol>(v, nct, 16 * 1024, 2) > 225 * 1024) nct /= 2;
    if (nct == 4) return launch_ma2_n<Pol, 4>(p, m, v, x, ldx, s, spad, partial, tbuf, st);
    if (nct == 2) return launch_ma2_n<Pol, 2>(p, m, v, x, ldx, s, spad, partial, tbuf, st);
    return launch_ma2_n<Pol, 1>(p, m, v, x, ldx, s, spad, partial, tbuf, st);
}

template <class Pol, int NT>
cudaError_t launch_mb2_t(const PlanView& p, const MrView& m, const Mr2View& v, const typename Pol::W* x,
                         int64_t ldx, const typename Pol::W* tbuf, typename Pol::W* b, int64_t ldb, int64_t s,
                         int spad, cudaStream_t st, int chunk0, int chunk1) {
    // one CTA per SM; X / coefficients double-buffered when it leaves >= 3 ring
    // stages, else single-buffered; the ring takes the rest of shared memory
    int nbuf = 2;
    if (mb2_smem<Pol>(v, NT, 3, 2) > 225 * 1024) nbuf = 1;
    if (const char* e = getenv("HODLR_B200_MB_NBUF")) nbuf = atoi(e) == 1 ? 1 : 2;
    int ns = kRingMax;
    while (ns > 2 && mb2_smem<Pol>(v, NT, ns, nbuf) > 225 * 1024) --ns;
    if (const char* e = getenv("HODLR_B200_MB_NS")) ns = std::max(2, std::min(ns, atoi(e)));
    const size_t sm = mb2_smem<Pol>(v, NT, ns, nbuf);
    if (sm > 227 * 1024) return cudaErrorInvalidConfiguration;
    const bool fw = sizeof(typename Pol::W) == 8 && v.widen_fast && getenv("HODLR_B200_FASTWIDEN");  // off by default (measured: no gain)
    auto k = fw ? k_mr2_b<Pol, NT, true> : k_mr2_b<Pol, NT, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int ngrp = (spad + NT * 8 - 1) / (NT * 8);
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kBThreads, sm);
    if (chunk1 <= chunk0) return cudaSuccess;
    const int nwork = (chunk1 - chunk0) * ngrp;
    const int grid = std::max(1, std::min(nwork, sms * std::max(occ, 1)));
    k<<<grid, kBThreads, sm, st>>>(p, m, v, x, ldx, tbuf, b, ldb, s, ngrp, ns, mb2_trows<Pol>(v), nbuf, chunk0, chunk1);
    return cudaGetLastError();
}
template <class Pol>
cudaError_t launch_mb2(const PlanView& p, const MrView& m, const Mr2View& v, const typename Pol::W* x,
                       int64_t ldx, const typename Pol::W* tbuf, typename Pol::W* b, int64_t ldb, int64_t s,
                       int spad, cudaStream_t st, int chunk0 = 0, int chunk1 = -1) {
    if (chunk1 < 0) chunk1 = p.nchunks;
    int nt = pick_nt(spad);
    while (nt > 1 && mb2_smem<Pol>(v, nt, 2, 1) > 225 * 1024) nt /= 2;
    if (nt == 4) return launch_mb2_t<Pol, 4>(p, m, v, x, ldx, tbuf, b, ldb, s, spad, st, chunk0, chunk1);
    if (nt == 2) return launch_mb2_t<Pol, 2>(p, m, v, x, ldx, tbuf, b, ldb, s, spad, st, chunk0, chunk1);
    return launch_mb2_t<Pol, 1>(p, m, v, x, ldx, tbuf, b, ldb, s, spad, st, chunk0, chunk1);
}

// Fixed-order reduction of the listed multi-slot nodes (mr.multi: nbig
// many-slot nodes, then the rest), one launch per class so no CTA is idle.
template <typename W>
cudaError_t launch_reduce(const PlanView& p, const MrPlan& mr, int64_t s, int spad, const W* partial, W* tbuf,
                          W* send, cudaStream_t st) {
    const int nsmall = mr.nmulti - mr.nbig;
    const int64_t tb = ((int64_t)mr.rmax_big * s + 31) / 32, ts = ((int64_t)mr.rmax_small * s + 255) / 256;
    const int ty_big = (int)std::max<int64_t>(1, std::min<int64_t>(tb, 1024));
    const int ty_small = (int)std::max<int64_t>(1, std::min<int64_t>(ts, 1024));
    const int64_t blocks = (int64_t)mr.nbig * ty_big + (int64_t)nsmall * ty_small;
    if (blocks <= 0) return cudaSuccess;
    k_mr_reduce<W><<<(unsigned)blocks, 256, 0, st>>>(p, mr.view, 0, s, spad, partial, tbuf, send, mr.multi, mr.nbig,
                                                      ty_big, ty_small);
    return cudaGetLastError();
}

template <class Pol>
cudaError_t mr_run(const PlanView& p, const MrPlan& mr, int lev_lo, const typename Pol::W* x, int64_t ldx,
                   typename Pol::W* b, int64_t ldb, int64_t s, typename Pol::W* partial,
                   typename Pol::W* tbuf, cudaStream_t st, int phases = 3, int chunk0 = 0, int chunk1 = -1) {
    using W = typename Pol::W;
    const MrView& m = mr.view;
    const int spad = (int)mr_spad(s);
    if (p.nchunks == 0) return cudaSuccess;
    const bool any_level = lev_lo < m.nlev;
    const int wfmt = sizeof(W) == 8 ? HODLR_FMT_FP64 : HODLR_FMT_FP32;
    if (mr_slab_used(mr, wfmt, lev_lo)) {
        cudaError_t e = cudaSuccess;
        if (any_level && (phases & 1)) {
            bool done = false;
            if constexpr (sizeof(W) == 4) {
                if (tca_usable(mr, s)) {
                    e = tc_phase_a(p, mr, x, ldx, s, partial, tbuf, st);
                    done = true;
                }
            }
            if (!done) e = launch_ma2<Pol>(p, m, mr.v2, x, ldx, s, spad, partial, tbuf, st);
            const int node_lo = m.lev[lev_lo].node0;
            const int nred = p.nnodes - node_lo;
            if (e == cudaSuccess && nred > 0 && mr.nmulti > 0)  // single-slot nodes were written by phase A
                e = launch_reduce<W>(p, mr, s, spad, partial, tbuf, nullptr, st);
        }
        if (e == cudaSuccess && (phases & 2)) {
            if constexpr (sizeof(W) == 4) {
                if (tc_usable(mr, s)) return tc_phase_b(p, mr, x, ldx, b, ldb, s, tbuf, st);
            }
            e = launch_mb2<Pol>(p, m, mr.v2, x, ldx, tbuf, b, ldb, s, spad, st, chunk0, chunk1);
        }
        return e;
    }
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
            k_mr_reduce<W><<<reduce_grid(m, node_lo, p.nnodes, s), 256, 0, st>>>(p, m, node_lo, s, spad, partial, tbuf, nullptr, nullptr);
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

// Fragment slabs for the policy of the handle's leaf (= working) format.
template <class Pol>
hodlr_status build_slab(const MrInput& in, MrPlan& mr) {
    constexpr int MT = kBRows / Pol::MR;
    const auto& nodes = *in.nodes;
    const auto& chunks = *in.chunks;
    const auto& leaves = *in.leaves;
    const int nlev = in.nlev, lev_lo = in.lev_lo;
    for (const ChunkDesc& c : chunks) {
        const LeafDesc& l = leaves[c.leaf];
        if (c.nrows != kChunk || l.m != kChunk || l.row0 != c.row0 || l.fmt != in.leaf_fmt) return HODLR_OK;
    }
    Mr2View& v = mr.v2;
    v = Mr2View{};
    v.nlev = nlev;
    // sharded handles: both regions cover every level, external ones included --
    // phase A sends their partials, phase B (after the exchange) applies their U
    v.lev_lo = 0;
    v.alev_lo = 0;
    (void)lev_lo;
    v.leaf_fmt = in.leaf_fmt;
    const int lfb = fmt_bytes(in.leaf_fmt);
    v.d_item = MT * 32 * Pol::AR * 4 * lfb;
    int64_t aoff = 0, uoff = 0;  // uoff: offset inside the chunk's U area
    int srows = 0, sfmt = -1;    // stacked phase-A rows so far, format of the open m-tile
    for (int i = 0; i < kMr2MaxRows; ++i) {
        v.row_lv[i] = -1;
        v.row_c[i] = 0;
    }
    for (int i = 0; i < kMr2MaxTasks; ++i) v.task_fmt[i] = HODLR_FMT_FP32;
    for (int lv = 0; lv < nlev; ++lv) {
        const MrLevel& L = mr.view.lev[lv];
        Mr2Level& M = v.lev[lv];
        const bool bpart = true;
        M.vfmt = M.ufmt = -1;
        for (int id = L.node0; id < L.node0 + L.nnodes; ++id) {
            const NodeDesc& nd = nodes[id];
            if (nd.rv > 0) {
                if (M.vfmt >= 0 && M.vfmt != nd.v_fmt) return HODLR_OK;  // one format per level
                M.vfmt = nd.v_fmt;
            }
            if (nd.ru > 0 && bpart) {
                if (M.ufmt >= 0 && M.ufmt != nd.u_fmt) return HODLR_OK;
                M.ufmt = nd.u_fmt;
            }
        }
        if (M.vfmt < 0) M.vfmt = HODLR_FMT_FP32;
        if (M.ufmt < 0) M.ufmt = HODLR_FMT_FP32;
        if (sizeof(typename Pol::W) == 4 && (M.vfmt == HODLR_FMT_FP64 || M.ufmt == HODLR_FMT_FP64)) return HODLR_OK;
        // stack this level's V' columns after the previous level's when the format
        // matches (shared m-tiles), else start a new m-tile
        if (L.rv_max > 0) {
            if (srows % Pol::MR != 0 && sfmt != M.vfmt) srows = (srows + Pol::MR - 1) / Pol::MR * Pol::MR;
            if (srows + L.rv_max > kMr2MaxRows) return HODLR_OK;
            for (int c = 0; c < L.rv_max; ++c) {
                v.row_lv[srows + c] = (int16_t)lv;
                v.row_c[srows + c] = (int16_t)c;
            }
            for (int tt = srows / Pol::MR; tt <= (srows + L.rv_max - 1) / Pol::MR; ++tt) v.task_fmt[tt] = M.vfmt;
            srows += L.rv_max;
            sfmt = M.vfmt;
        }
        if (!bpart) continue;
        M.steps = (L.ru_max + Pol::KU - 1) / Pol::KU;
        M.usz = MT * 32 * Pol::AR * Pol::UV * fmt_bytes(M.ufmt);
        // all 16 warps' blocks of one step are adjacent; a level starts at a
        // multiple of its step size so a step never straddles a ring stage
        const int64_t sstep = (int64_t)kBWarps * M.usz;
        uoff = (uoff + sstep - 1) / sstep * sstep;
        M.uoff = uoff;
        uoff += (int64_t)M.steps * sstep;
        v.nu_items += M.steps;
    }
    v.ntasks = (srows + Pol::MR - 1) / Pol::MR;
    if (v.ntasks > kMr2MaxTasks) return HODLR_OK;
    // stacked U layout when every level with U columns stores them in one format
    {
        int ufmt = -1, ucols = 0;
        bool same = true;
        for (int lv = 0; lv < nlev; ++lv) {
            const MrLevel& L = mr.view.lev[lv];
            if (L.ru_max <= 0) continue;
            if (ufmt >= 0 && v.lev[lv].ufmt != ufmt) same = false;
            ufmt = v.lev[lv].ufmt;
            ucols += L.ru_max;
        }
        for (int i = 0; i < kMr2MaxRows; ++i) {
            v.urow_lv[i] = -1;
            v.urow_c[i] = 0;
        }
        if (same && ufmt >= 0 && ucols <= kMr2MaxRows && !getenv("HODLR_B200_NO_USTACK")) {
            int r = 0;
            for (int lv = 0; lv < nlev; ++lv)
                for (int c = 0; c < mr.view.lev[lv].ru_max; ++c, ++r) {
                    v.urow_lv[r] = (int16_t)lv;
                    v.urow_c[r] = (int16_t)c;
                }
            v.ustack = 1;
            v.nku = (ucols + 15) / 16;
            v.ufmt_all = ufmt;
            v.u_item = MT * 32 * Pol::AR * 4 * fmt_bytes(ufmt);
            uoff = (int64_t)v.nku * kBWarps * v.u_item;  // U area bytes per chunk
        }
    }
    for (int t = 0; t < v.ntasks; ++t) {
        const int blk = 32 * Pol::AR * 4 * fmt_bytes(v.task_fmt[t]);
        v.task_off[t] = (int32_t)aoff;
        aoff += blk;
        v.max_ablk = std::max(v.max_ablk, blk);
    }
    if (v.max_ablk == 0) v.max_ablk = 128;
    if (v.d_item & (v.d_item - 1)) return HODLR_OK;
    while ((1 << v.lslot) < v.d_item) ++v.lslot;
    {
        int next = -1;
        for (int lv = nlev - 1; lv >= 0; --lv) {
            Mr2Level& M = v.lev[lv];
            M.ulo = (int32_t)M.uoff;
            M.unext = next;
            if (M.steps > 0) next = M.ulo;
        }
    }
    if (v.ntasks > 4 * kAWarps) return HODLR_OK;  // phase-A tasks per warp are register-resident (<= 4)
    v.arow = (int32_t)aoff;
    v.a_chunk_bytes = 16 * aoff;  // ablk is a multiple of 128
    v.warp_bytes = (int32_t)((uoff + 127) / 128 * 128);  // U area bytes per chunk (all warps)
    v.b_chunk_bytes = 16LL * kBWarps * v.d_item + v.warp_bytes;
    const size_t a_bytes = (size_t)v.a_chunk_bytes * chunks.size();
    const size_t b_bytes = (size_t)v.b_chunk_bytes * chunks.size();
    void* d = nullptr;
    if (cudaMalloc(&d, a_bytes + b_bytes + 512) != cudaSuccess) {
        cudaGetLastError();
        return HODLR_OK;  // no room for a second copy: the arena kernels serve
    }
    v.slab_a = (const uint8_t*)d;
    v.slab_b = (const uint8_t*)d + (a_bytes + 255) / 256 * 256;
    // (in the allocation's 512-byte tail, past both slabs: "a stored value is an
    // fp32 subnormal / inf / nan", which rules out the integer widening)
    int* special = (int*)((uint8_t*)d + ((a_bytes + b_bytes + 508) & ~(size_t)3));
    cudaError_t e = cudaMemset(special, 0, 4);
    if (e == cudaSuccess && a_bytes) {
        k_slab_a<Pol><<<148 * 8, 256>>>(*in.view, v, (uint8_t*)v.slab_a, special);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        k_slab_b<Pol><<<148 * 8, 256>>>(*in.view, v, (uint8_t*)v.slab_b, special);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    int sp = 1;
    if (e == cudaSuccess) e = cudaMemcpy(&sp, special, 4, cudaMemcpyDeviceToHost);
    v.widen_fast = sp == 0;
    if (e != cudaSuccess) {
        cudaFree(d);
        return HODLR_ERR_CUDA;
    }
    mr.slab_dev = d;
    mr.slab_ok = true;
    mr.slab_fmt = sizeof(typename Pol::W) == 8 ? HODLR_FMT_FP64 : HODLR_FMT_FP32;
    return HODLR_OK;
}

hodlr_status mr_prepare(const MrInput& in, MrPlan& mr) {
    mr = MrPlan{};
    mr.sharded = in.lev_lo > 0;
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
    // tcgen05 phase A runs one CTA per SM (512 TMEM columns): slots per SM
    mr.tca_cand = !mr.has_fp64_operand && in.view && in.d_arena && !getenv("HODLR_B200_NO_SLAB") &&
                  tc_a_candidate(in, v);
    if (mr.tca_cand) v.nb = std::max(1, std::min(nch, sms));
    // fragment-slab handles (uniform 256-row leaves): the slab phase-A kernels run
    // one CTA per SM, so one run per SM (fewer run-end flushes and partial slots)
    {
        bool uniform = in.view && in.d_arena && !getenv("HODLR_B200_NO_SLAB");
        for (const ChunkDesc& c : chunks) {
            const LeafDesc& l = (*in.leaves)[c.leaf];
            if (c.nrows != kChunk || l.m != kChunk || l.row0 != c.row0 || l.fmt != in.leaf_fmt) uniform = false;
        }
        if (uniform && (in.leaf_fmt == HODLR_FMT_FP64 || in.leaf_fmt == HODLR_FMT_FP32) && !getenv("HODLR_B200_NB2"))
            v.nb = std::max(1, std::min(nch, sms));
    }
    int64_t rows = 0;
    for (int lv = 0; lv < nlev; ++lv) {
        MrLevel& L = v.lev[lv];
        if (L.node0 < 0) return HODLR_OK;
        L.rv_pad = (L.rv_max + 7) / 8 * 8;
        L.part_rows = rows;
        rows += (int64_t)(v.nb + L.nnodes) * L.rv_pad;
    }
    v.part_rows = rows;
    // send-slot width of each external level (sharded handles; node ids 0..L-1)
    for (size_t id = 0; id < nodes.size(); ++id) {
        const NodeDesc& nd = nodes[id];
        if (nd.ext_slot < 0) continue;
        int64_t next = in.ext_count;
        for (size_t j = 0; j < nodes.size(); ++j)
            if (nodes[j].ext_slot > nd.ext_slot && nodes[j].ext_slot < next) next = nodes[j].ext_slot;
        v.lev[nd.level - 1].ext_w = (int32_t)(next - nd.ext_slot);
    }
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
    // nodes whose sum spans several phase-A CTAs (or goes to the send buffer)
    // listed many-slot nodes first (one warp per coefficient), then the others
    // (one thread per coefficient): two reduce launches sized for each class
    std::vector<int32_t> multi, small;
    for (size_t id = 0; id < nodes.size(); ++id)
        if (slots[id].b1 > slots[id].b0 || nodes[id].ext_slot >= 0) {
            const bool big = slots[id].b1 - slots[id].b0 + 1 > kMrBigSlots;
            const int w = std::max(nodes[id].rv, nodes[id].ext_slot >= 0 ? v.lev[nodes[id].level - 1].ext_w : 0);
            (big ? multi : small).push_back((int32_t)id);
            int& r = big ? mr.rmax_big : mr.rmax_small;
            r = std::max(r, w);
        }
    mr.nbig = (int)multi.size();
    multi.insert(multi.end(), small.begin(), small.end());
    mr.nmulti = (int)multi.size();
    const size_t sbytes = (slots.size() * sizeof(MrSlot) + 255) / 256 * 256;
    cudaError_t e = cudaMalloc(&mr.dev, sbytes + multi.size() * sizeof(int32_t) + 4);
    if (e == cudaSuccess)
        e = cudaMemcpy(mr.dev, slots.data(), slots.size() * sizeof(MrSlot), cudaMemcpyHostToDevice);
    mr.multi = (int32_t*)((uint8_t*)mr.dev + sbytes);
    if (e == cudaSuccess && !multi.empty())
        e = cudaMemcpy(mr.multi, multi.data(), multi.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        mr_release(mr);
        return HODLR_ERR_CUDA;
    }
    v.slots = (const MrSlot*)mr.dev;
    {
        // flush table of the K-split phase A: per chunk, the levels whose node ends
        // there (inside the chunk's run) and the destination of their rows
        std::vector<MrFlush> fl((size_t)nch * nlev, MrFlush{0, 0, 0});
        std::vector<uint32_t> fm((size_t)nch, 0u);
        for (int b = 0; b < v.nb; ++b) {
            const int c0 = (int)((int64_t)b * nch / v.nb), c1 = (int)((int64_t)(b + 1) * nch / v.nb);
            for (int ci = c0; ci < c1; ++ci)
                for (int lv = 0; lv < nlev; ++lv) {
                    const int n0 = cn[(size_t)ci * nlev + lv];
                    if (ci + 1 < c1 && cn[(size_t)(ci + 1) * nlev + lv] == n0) continue;
                    const MrSlot& sl = slots[n0];
                    const NodeDesc& nd = nodes[n0];
                    const MrLevel& L = v.lev[lv];
                    MrFlush& f = fl[(size_t)ci * nlev + lv];
                    if (sl.b0 == sl.b1 && nd.ext_slot < 0) {
                        f.direct = 1;
                        f.row = nd.t_off;
                        f.clim = nd.rv;
                    } else {
                        f.direct = 0;
                        f.row = L.part_rows + ((int64_t)b + sl.jrel) * L.rv_pad;
                        f.clim = L.rv_max;
                    }
                    fm[ci] |= 1u << lv;
                }
        }
        const size_t fbytes = fl.size() * sizeof(MrFlush);
        e = cudaMalloc(&mr.flush_dev, fbytes + fm.size() * 4 + 16);
        if (e == cudaSuccess) e = cudaMemcpy(mr.flush_dev, fl.data(), fbytes, cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy((uint8_t*)mr.flush_dev + fbytes, fm.data(), fm.size() * 4, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            mr_release(mr);
            return HODLR_ERR_CUDA;
        }
        v.flush = (const MrFlush*)mr.flush_dev;
        v.flush_mask = (const uint32_t*)((uint8_t*)mr.flush_dev + fbytes);
    }
    mr.ok = true;
    if (in.view && in.d_arena && !getenv("HODLR_B200_NO_SLAB")) {
        hodlr_status st = HODLR_OK;
        if (in.leaf_fmt == HODLR_FMT_FP64)
            st = build_slab<PolF64>(in, mr);
        else if (in.leaf_fmt == HODLR_FMT_FP32)
            st = build_slab<PolTF32>(in, mr);
        if (st == HODLR_OK && mr.slab_ok) st = tc_prepare(in, mr);
        if (st != HODLR_OK) {
            mr_release(mr);
            return st;
        }
    }
    return HODLR_OK;
}

void mr_release(MrPlan& mr) {
    if (mr.dev) cudaFree(mr.dev);
    if (mr.flush_dev) cudaFree(mr.flush_dev);
    mr.flush_dev = nullptr;
    if (mr.slab_dev) cudaFree(mr.slab_dev);
    if (mr.tc_dev) cudaFree(mr.tc_dev);
    if (mr.tca_dev) cudaFree(mr.tca_dev);
    mr.tca_dev = nullptr;
    mr.tca_ok = false;
    mr.dev = nullptr;
    mr.slab_dev = nullptr;
    mr.tc_dev = nullptr;
    mr.tc_ok = false;
    mr.ok = false;
    mr.slab_ok = false;
}

bool mr_usable(const MrPlan& mr, int working_fmt) {
    if (!mr.ok) return false;
    if (working_fmt == HODLR_FMT_FP64) return true;
    // TF32 kind: every operand must be exact in fp32 (fp64-stored factors under
    // fp32 working are multiplied in binary64 by the generic kernels)
    return working_fmt == HODLR_FMT_FP32 && !mr.has_fp64_operand;
}

int mr_launches() { return 3; }

bool mr_slab_begin_usable(const MrPlan& mr, int working_fmt) {
    return mr.slab_ok && mr.slab_fmt == working_fmt && mr.sharded && !getenv("HODLR_B200_NO_SLAB");
}

template <class Pol>
static cudaError_t shard_begin_t(const PlanView& p, const MrPlan& mr, const typename Pol::W* x, int64_t ldx,
                                 int64_t s, typename Pol::W* partial, typename Pol::W* tbuf,
                                 typename Pol::W* send, cudaStream_t st) {
    using W = typename Pol::W;
    const int spad = (int)mr_spad(s);
    cudaError_t e;
    if constexpr (sizeof(W) == 4) {
        e = tca_usable(mr, s) ? tc_phase_a(p, mr, x, ldx, s, partial, tbuf, st)
                              : launch_ma2<Pol>(p, mr.view, mr.v2, x, ldx, s, spad, partial, tbuf, st);
    } else {
        e = launch_ma2<Pol>(p, mr.view, mr.v2, x, ldx, s, spad, partial, tbuf, st);
    }
    if (e != cudaSuccess) return e;
    if (mr.nmulti == 0) return cudaSuccess;
    return launch_reduce<W>(p, mr, s, spad, partial, tbuf, send, st);
}
template <>
cudaError_t mr_shard_begin<double>(const PlanView& p, const MrPlan& mr, const double* x, int64_t ldx, int64_t s,
                                   double* partial, double* tbuf, double* send, cudaStream_t st) {
    return shard_begin_t<PolF64>(p, mr, x, ldx, s, partial, tbuf, send, st);
}
template <>
cudaError_t mr_shard_begin<float>(const PlanView& p, const MrPlan& mr, const float* x, int64_t ldx, int64_t s,
                                  float* partial, float* tbuf, float* send, cudaStream_t st) {
    return shard_begin_t<PolTF32>(p, mr, x, ldx, s, partial, tbuf, send, st);
}
template <>
cudaError_t mr_slab_phase_b<double>(const PlanView& p, const MrPlan& mr, const double* x, int64_t ldx, double* b,
                                    int64_t ldb, int64_t s, const double* tbuf, cudaStream_t st) {
    return launch_mb2<PolF64>(p, mr.view, mr.v2, x, ldx, tbuf, b, ldb, s, (int)mr_spad(s), st);
}
template <>
cudaError_t mr_slab_phase_b<float>(const PlanView& p, const MrPlan& mr, const float* x, int64_t ldx, float* b,
                                   int64_t ldb, int64_t s, const float* tbuf, cudaStream_t st) {
    if (tc_usable(mr, s)) return tc_phase_b(p, mr, x, ldx, b, ldb, s, tbuf, st);
    return launch_mb2<PolTF32>(p, mr.view, mr.v2, x, ldx, tbuf, b, ldb, s, (int)mr_spad(s), st);
}

// Host-buffer pipeline (capi.cu hodlr_matvec_host): phase A + reduce once, then
// phase B over chunk ranges, so each range's device-to-host copy overlaps the
// next ranges' kernels.  Fragment-slab DMMA path only (fp64 working).
bool mr_sliceable(const MrPlan& mr, int working_fmt, int64_t s) {
    return working_fmt == HODLR_FMT_FP64 && s > 1 && mr_slab_used(mr, working_fmt, 0);
}
cudaError_t mr_phase_a(const PlanView& p, const MrPlan& mr, const double* x, int64_t ldx, int64_t s, double* partial,
                       double* tbuf, cudaStream_t st) {
    return mr_run<PolF64>(p, mr, 0, x, ldx, nullptr, 0, s, partial, tbuf, st, 1);
}
cudaError_t mr_phase_b_range(const PlanView& p, const MrPlan& mr, const double* x, int64_t ldx, double* b, int64_t ldb,
                             int64_t s, double* tbuf, int chunk0, int chunk1, cudaStream_t st) {
    return mr_run<PolF64>(p, mr, 0, x, ldx, b, ldb, s, nullptr, tbuf, st, 2, chunk0, chunk1);
}

bool mr_slab_used(const MrPlan& mr, int working_fmt, int lev_lo) {
    return mr.slab_ok && mr.slab_fmt == working_fmt && !mr.sharded && lev_lo == 0 && !getenv("HODLR_B200_NO_SLAB");
}

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
