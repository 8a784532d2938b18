// Single-vector (s = 1) streaming fast path: ONE persistent kernel per matvec.
//
// Layout ("leaf slab", built at create time from the quantised level-batched
// arena): leaf L (M = 256 rows) owns one contiguous region
//     VS  V' of every level restricted to the leaf's rows, one row-major
//         M x vpad_g sub-slab per storage format g (q52, bf16, fp16, fp32,
//         fp64; columns level-major, padded with zeros to a multiple of 4)
//     DS  the dense leaf, 4 blocks of 64 rows, each stored column-major
//         (256 columns x 64 contiguous rows), working format
//     US  U of every level, 4 blocks of 64 rows, each with one column-major
//         ncols_g x 64 sub-block per format
// Every piece of work is then 1-6 contiguous byte ranges, and the arithmetic
// is reduction-free: for D and U a lane owns two output rows and walks the
// columns (x / coefficients broadcast from shared memory); for V' a lane owns
// four output columns and walks the rows.  Partial sums stay in registers for
// all pieces of a work item; warps combine once per item through shared memory.
//
// Schedule (one CTA per pipeline, kCtasPerSm per SM; no co-residency needed):
//   producer warp  pulls work from ONE atomic queue (fetched two ahead) and
//                  streams it with cp.async.bulk (1-D TMA, complete_tx on the
//                  stage's "full" mbarrier) into a ring of kNS stages;
//   consumer warps compute from shared memory and release stages ("empty").
// Queue = [A items][BC items, with the R pieces inserted at position pos_r]:
//   A  (leaf, row pair) -> partial V'^T x per column of every level, stored to
//      the partial buffer; each CTA publishes its A completions once
//      (fence + counter) after its last A item;
//   R  (level, node range) -> fixed-order sum of the nodes' partials (leaf
//      order: deterministic) into the coefficients t, published per piece;
//   BC (leaf, 64-row block) -> y = D x kept in a CTA-local slot; its U piece
//      (b = U t + y over every level, t bulk-copied next to U) is deferred in a
//      kFifo-deep FIFO until every R piece is published, then b is written
//      once (disjoint rows, no atomics).
// Every cross-CTA wait targets work EARLIER in the queue (R waits on all A
// items, U waits on all R pieces), so progress never assumes co-residency;
// pos_r is bounded by grid * (kFifo - 2) so the R pieces are always taken
// before running CTAs could fill their FIFOs (sv_prepare / sv_set_grid).
// Per-call state (queue, counters, epoch) lives in the zero-initialised
// workspace; the last CTA resets it and bumps the epoch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "sv.h"

// This file is compiled twice (Makefile): HODLR_SV_GEO = 0 with the default geometry and
// HODLR_SV_GEO = 1 with HODLR_CTAS / HODLR_CONSUMERS / HODLR_KNS / HODLR_KSTAGE of the
// binary32-working geometry (SvInput::geo).  The geometry-specific entry points carry a
// _g0 / _g1 suffix; the geometry-0 object also holds the dispatchers declared in sv.h.
#ifndef HODLR_SV_GEO
#define HODLR_SV_GEO 0
#endif
#define SVG_CAT(a, b) a##b
#define SVG_X(n, g) SVG_CAT(n, g)
#define SVG(n) SVG_X(n##_g, HODLR_SV_GEO)

namespace hodlr {

namespace {

constexpr int kM = 256;                 // leaf rows
constexpr int kRB = 64;                 // rows of a BC item (one leaf row block)
constexpr int kRPL = kRB / 32;          // rows per lane in B / C pieces
// (HODLR_KNS / HODLR_KSTAGE override the ring geometry for tools/build_variants.sh sweeps)
#ifndef HODLR_KNS
#define HODLR_KNS 3
#endif
#ifndef HODLR_KSTAGE
#define HODLR_KSTAGE 33280
#endif
constexpr int kNS = HODLR_KNS;          // ring stages per CTA
#ifndef HODLR_CTAS
#define HODLR_CTAS 2
#endif
constexpr int kCtasPerSm = HODLR_CTAS;  // independent pipelines per SM
constexpr int kStage = HODLR_KSTAGE;    // bytes per stage (= 512 B of x + a 64 x 64 fp64 D block; 2 x 48.75 KB measured
                                        // level on cfg2, 7-9% slower on cfg5 fp32 working)
#ifndef HODLR_CONSUMERS
#define HODLR_CONSUMERS 8
#endif
constexpr int kConsumers = HODLR_CONSUMERS;  // consumer warps (= column subsets of B/C pieces)
constexpr int kThreads = 32 * (kConsumers + 1);  // + producer warp
constexpr int kFifo = 8;                // BC items whose U piece waits for the coefficients
#ifndef HODLR_MAX_R
#define HODLR_MAX_R 256
#endif
constexpr int kMaxRPieces = HODLR_MAX_R;  // node-reduction pieces
constexpr int kMaxUPieces = 16;         // U chunks per BC item
constexpr int kMaxLev = 24;
constexpr int kMaxPieces = 32;          // phase-A pieces per leaf
#ifndef HODLR_MAX_COLS
#define HODLR_MAX_COLS 512
#endif
constexpr int kMaxCols = HODLR_MAX_COLS;  // columns (sum of ranks) per leaf
constexpr int kXB = 2048;               // x segment of an A piece (<= 256 rows)
constexpr int kMaxAG = 12;              // phase-A column groups

enum { PT_A = 1, PT_D = 2, PT_U = 3, PT_R = 5, PT_END = 4 };

#ifdef HODLR_PROFILE
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(i, dt) if (lane == 0) atomicAdd((unsigned long long*)&prof[i], (unsigned long long)(dt))
#else
#define PROF_T(v)
#define PROF_ADD(i, dt)
#endif

// HODLR_TRACE builds: per-CTA %globaltimer stamps into a.trace[cta * 16 + i]
// (tools/trace_run.py reads them back and prints the phase timeline).
#ifdef HODLR_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TR(i) do { if (a.trace) a.trace[blockIdx.x * 48 + (i)] = gtimer(); } while (0)
#define TRV(i, v) do { if (a.trace) a.trace[blockIdx.x * 48 + (i)] = (unsigned long long)(v); } while (0)
#else
#define TR(i) do { } while (0)
#define TRV(i, v) do { } while (0)
#endif

struct Level {
    int32_t r, fmt;
    int32_t slot;       // coefficient slot (elements) inside a U piece
    int32_t tstride;    // padded coefficients per node (multiple of 4)
    int32_t npc;        // A pieces (row chunks) per leaf of this level's format group
    int32_t cst;        // partials per (node, column): stride (multiple of 4) >= leaves_of_node * npc
    int64_t pbase;      // partial buffer base of the level's nodes
    int64_t tbase;      // coefficient buffer base
};

// A piece: rows [r0, r0 + nrows) of format group g's V' sub-slab.  A queue
// item is one piece (few leaves per CTA: the A phase spreads over every CTA)
// or a whole leaf (many leaves: 1/npc the partials).  Partials of a group are
// written at its item's last piece of that group (last_of_group), into slot
// chunk of npc slots per leaf.
struct APiece {
    int32_t g, r0, nrows, chunk, npc, last_of_group;  // g: A group (index into SvParams::ag)
};

// Phase-A column group: whole levels of one storage format, <= 256 columns
// (lanes own <= 2 column quads), stored as a row-major M x vpad V' sub-slab.
struct AGroup {
    int32_t fmt, c0, ncols, vpad;  // c0: first column inside the format's flat list
    int64_t voff;                  // sub-slab offset inside a leaf's V' region
};

// U chunk of a BC item: columns [c0, c0 + ncols) of format group g.
struct UPiece {
    int32_t g, c0, ncols, pad;
};

// Node reduction: level lv, nodes [j0, j1), rank columns [c0, c1) (whole nodes,
// or one node split by columns); its partials are contiguous.
struct RPiece {
    int16_t lv, pad;
    int32_t j0, j1, c0, c1;
};

struct SvParams {
    int32_t depth, nleaves, nnodes;
    int32_t leaf_fmt;
    int32_t num_a, num_d, num_r, pos_r;   // queue: BC items with the R pieces at pos_r
    int32_t napieces;
    int32_t a_group;                      // pieces per A queue item: 1 or napieces (whole leaf)
    int32_t dpieces_w[2], dcols_w[2];      // phase-B pieces per item / columns per piece, [fp32, fp64 working]
    // three regions, leaf-major inside each: [V' of every leaf][D blocks][U blocks]
    int64_t vs_bytes, ds_bytes, us_bytes;  // per leaf
    int64_t d_region, u_region;            // region offsets (the V' region starts at 0)
    int64_t dblock_bytes, ublock_bytes;
    int32_t gcols[5];                     // columns per storage format (U block, flat index)
    int64_t ugoff[5];                     // U sub-block offsets in a block
    AGroup ag[kMaxAG];                    // V' sub-slabs (phase A column groups)
    int32_t nag;
    int32_t coef_elems;
    int32_t u_data_off[2];                // U piece: coefficients, then the U chunk
    int32_t nupieces;                     // U pieces per BC item (column chunks of the U block)
    Level lev[kMaxLev];
    APiece ap[kMaxPieces];
    RPiece rp[kMaxRPieces];
    UPiece up[kMaxUPieces];
    int8_t col_level[kMaxCols];           // flattened (group, column) -> level (0-based)
    int16_t col_c[kMaxCols];              //                            -> rank column
    int16_t gstart[6];
    int32_t static_first;                 // 1: CTA b starts with queue entry b
    int32_t rdefer;                       // 1: park R pieces until the A partials exist
    int32_t mode;                         // 0: whole matvec; 1: A items only (split launch 1);
                                          // 2: R + BC items after launch 1 (PDL dependent)
};

struct SvSync {
    unsigned epoch, queue, done;
    unsigned a_done;     // phase-A leaves whose partials are written (this call)
    unsigned r_done;     // node-reduction pieces whose coefficients are written
    unsigned pad[3];
};

struct PieceHdr {
    int32_t type, leaf, a, b;   // A: a = piece index; B: a = row block, b = first column; C: a = row block
    int32_t last, pad0, pad1, pad2;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
#ifdef HODLR_EXP_NOLOAD
    (void)bytes;  // timing experiment: no matrix bytes move (results are garbage)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
#else
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
#endif
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
#ifdef HODLR_EXP_NOLOAD
    return;
#endif
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Streaming (read-once) matrix bytes: L2 evict-first, so they do not push the
// small, re-read state (x, partials, coefficients) out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                                uint64_t pol) {
#if defined(HODLR_NO_L2_HINT) || defined(HODLR_EXP_NOLOAD)
    (void)pol;
    bulk_g2s(dst, src, bytes, bar);
#else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
#endif
}
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
}
__host__ __device__ __forceinline__ int64_t round_up16_d(int64_t v) { return (v + 15) / 16 * 16; }
__host__ __device__ __forceinline__ int fmt_sz(int f) {
    return f == HODLR_FMT_Q52 ? 1 : f == HODLR_FMT_FP32 ? 4 : f == HODLR_FMT_FP64 ? 8 : 2;
}

// ------------------------------------------------------------ scalar math
// acc += v * x in the working type W; a binary64-stored operand under fp32
// working is multiplied in binary64 and the product rounded once (operands
// "enter as-is, only results are rounded", arithmetic.py:14-21).
template <typename W>
__device__ __forceinline__ W madd(float v, W x, W acc) { return fma((W)v, x, acc); }
template <typename W>
__device__ __forceinline__ W madd_d(double v, W x, W acc) {
    if constexpr (sizeof(W) == 8) return fma(v, x, acc);
    else return acc + __double2float_rn(v * (double)x);
}

// Two consecutive elements (rows r, r+1 of a column) of format FMT at p.
template <int FMT>
__device__ __forceinline__ void load2(const uint8_t* p, float& a, float& b) {
    if constexpr (FMT == HODLR_FMT_FP32) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        a = v.x; b = v.y;
    } else if constexpr (FMT == HODLR_FMT_BF16) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
        a = __uint_as_float(w << 16); b = __uint_as_float(w & 0xffff0000u);
    } else if constexpr (FMT == HODLR_FMT_FP16) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
        __half2_raw r; r.x = (unsigned short)(w & 0xffff); r.y = (unsigned short)(w >> 16);
        const float2 f = __half22float2(__half2(r));
        a = f.x; b = f.y;
    } else {  // q52: byte -> binary16 with bits << 8
        const uint32_t w = *reinterpret_cast<const uint16_t*>(p);
        __half2_raw r; r.x = (unsigned short)((w << 8) & 0xff00); r.y = (unsigned short)(w & 0xff00);
        const float2 f = __half22float2(__half2(r));
        a = f.x; b = f.y;
    }
}

// Four consecutive elements (one row, columns 4q..4q+3) of format FMT at p.
template <int FMT>
__device__ __forceinline__ void load4(const uint8_t* p, float v[4]) {
    if constexpr (FMT == HODLR_FMT_FP32) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else if constexpr (FMT == HODLR_FMT_BF16) {
        const uint2 t = *reinterpret_cast<const uint2*>(p);
        v[0] = __uint_as_float(t.x << 16); v[1] = __uint_as_float(t.x & 0xffff0000u);
        v[2] = __uint_as_float(t.y << 16); v[3] = __uint_as_float(t.y & 0xffff0000u);
    } else if constexpr (FMT == HODLR_FMT_FP16) {
        const uint2 t = *reinterpret_cast<const uint2*>(p);
        __half2_raw r0, r1;
        r0.x = (unsigned short)(t.x & 0xffff); r0.y = (unsigned short)(t.x >> 16);
        r1.x = (unsigned short)(t.y & 0xffff); r1.y = (unsigned short)(t.y >> 16);
        const float2 f0 = __half22float2(__half2(r0)), f1 = __half22float2(__half2(r1));
        v[0] = f0.x; v[1] = f0.y; v[2] = f1.x; v[3] = f1.y;
    } else {  // q52
        const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
        __half2_raw r0, r1;
        r0.x = (unsigned short)((w << 8) & 0xff00); r0.y = (unsigned short)(w & 0xff00);
        r1.x = (unsigned short)((w >> 8) & 0xff00); r1.y = (unsigned short)((w >> 16) & 0xff00);
        const float2 f0 = __half22float2(__half2(r0)), f1 = __half22float2(__half2(r1));
        v[0] = f0.x; v[1] = f0.y; v[2] = f1.x; v[3] = f1.y;
    }
}

// ------------------------------------------------------------ phase A
// Rows of the V' sub-slab of format FMT: lane owns column quad q = lane (and
// lane + 32 when vpad > 128), warp w owns rows w, w + 8, ...; sums stay in acc
// across pieces.  Lanes past the last quad read quad 0 (a valid address, the
// sums are never written), so the row loop has no divergent branches and the
// loads of four rows are in flight together.
template <int FMT, typename W>
__device__ __forceinline__ void a_quad(const uint8_t* p, W x, W acc[4]) {
    if constexpr (FMT == HODLR_FMT_FP64) {
        const double2 t0 = *reinterpret_cast<const double2*>(p);
        const double2 t1 = *reinterpret_cast<const double2*>(p + 16);
        acc[0] = madd_d<W>(t0.x, x, acc[0]);
        acc[1] = madd_d<W>(t0.y, x, acc[1]);
        acc[2] = madd_d<W>(t1.x, x, acc[2]);
        acc[3] = madd_d<W>(t1.y, x, acc[3]);
    } else {
        float v[4];
        load4<FMT>(p, v);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = madd<W>(v[e], x, acc[e]);
    }
}

template <int FMT, typename W, int NSET>
__device__ __forceinline__ void a_rows_n(const uint8_t* rows, int nrows, int nq, int row_bytes, const W* xs, int warp,
                                         int lane, W acc[2][4]) {
    constexpr int qb = 4 * (FMT == HODLR_FMT_Q52 ? 1 : FMT == HODLR_FMT_FP32 ? 4 : FMT == HODLR_FMT_FP64 ? 8 : 2);
    const uint8_t* b0 = rows + (lane < nq ? lane : 0) * qb;
    const uint8_t* b1 = rows + (lane + 32 < nq ? lane + 32 : 0) * qb;
    int j = warp;
    for (; j + 3 * kConsumers < nrows; j += 4 * kConsumers) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int jj = j + u * kConsumers;
            const W x = xs[jj];
            a_quad<FMT, W>(b0 + (size_t)jj * row_bytes, x, acc[0]);
            if constexpr (NSET == 2) a_quad<FMT, W>(b1 + (size_t)jj * row_bytes, x, acc[1]);
        }
    }
    for (; j < nrows; j += kConsumers) {
        const W x = xs[j];
        a_quad<FMT, W>(b0 + (size_t)j * row_bytes, x, acc[0]);
        if constexpr (NSET == 2) a_quad<FMT, W>(b1 + (size_t)j * row_bytes, x, acc[1]);
    }
}

template <int FMT, typename W>
__device__ __forceinline__ void a_rows(const uint8_t* rows, int nrows, int vpad, const W* xs, int warp, int lane,
                                       W acc[2][4]) {
    const int nq = vpad >> 2;
    const int row_bytes = vpad * fmt_sz(FMT);
    if (nq <= 32) a_rows_n<FMT, W, 1>(rows, nrows, nq, row_bytes, xs, warp, lane, acc);
    else a_rows_n<FMT, W, 2>(rows, nrows, nq, row_bytes, xs, warp, lane, acc);
}

template <typename W>
__device__ __forceinline__ void a_piece(int g, const uint8_t* rows, int nrows, int vpad, const W* xs, int warp,
                                        int lane, W acc[2][4]) {
    switch (g) {
        case HODLR_FMT_FP64: a_rows<HODLR_FMT_FP64, W>(rows, nrows, vpad, xs, warp, lane, acc); break;
        case HODLR_FMT_FP32: a_rows<HODLR_FMT_FP32, W>(rows, nrows, vpad, xs, warp, lane, acc); break;
        case HODLR_FMT_FP16: a_rows<HODLR_FMT_FP16, W>(rows, nrows, vpad, xs, warp, lane, acc); break;
        case HODLR_FMT_BF16: a_rows<HODLR_FMT_BF16, W>(rows, nrows, vpad, xs, warp, lane, acc); break;
        default: a_rows<HODLR_FMT_Q52, W>(rows, nrows, vpad, xs, warp, lane, acc); break;
    }
}

// ------------------------------------------------------------ phases B / C
// Column-major block (ncols x 64 rows) of format FMT: lane owns rows 2l, 2l+1,
// warp w takes columns w, w + 8, ...; the multiplier of column c is mul(c)
// (x or a coefficient).  4 independent accumulator pairs break the FMA chains.
template <int FMT, typename W>
__device__ __forceinline__ void col_elem(const uint8_t* p, W m, W acc[kRPL]) {
    if constexpr (FMT == HODLR_FMT_FP64) {
        if constexpr (kRPL == 2) {
            const double2 t = *reinterpret_cast<const double2*>(p);
            acc[0] = madd_d<W>(t.x, m, acc[0]);
            acc[1] = madd_d<W>(t.y, m, acc[1]);
        } else {
            acc[0] = madd_d<W>(*reinterpret_cast<const double*>(p), m, acc[0]);
        }
    } else if constexpr (kRPL == 2) {
        float a, b;
        load2<FMT>(p, a, b);
        acc[0] = madd<W>(a, m, acc[0]);
        acc[1] = madd<W>(b, m, acc[1]);
    } else {
        float a;
        if constexpr (FMT == HODLR_FMT_FP32) a = *reinterpret_cast<const float*>(p);
        else if constexpr (FMT == HODLR_FMT_BF16) a = __uint_as_float((uint32_t)(*reinterpret_cast<const uint16_t*>(p)) << 16);
        else if constexpr (FMT == HODLR_FMT_FP16) a = dec_fp16(*reinterpret_cast<const uint16_t*>(p));
        else a = dec_q52(*p);
        acc[0] = madd<W>(a, m, acc[0]);
    }
}

// Column-major block (ncols x kRB rows) of format FMT: lane owns rows
// kRPL*l .. kRPL*l + kRPL-1, warp w takes columns w, w + 8, ...; the multiplier
// of column c is mul(c) (x or a coefficient).  4 accumulator sets break the
// FMA chains.
template <int FMT, typename W, typename MulF>
__device__ __forceinline__ void col_block(const uint8_t* blk, int ncols, int warp, int lane, MulF mul,
                                          W acc[4][kRPL]) {
    constexpr int sz = FMT == HODLR_FMT_Q52 ? 1 : FMT == HODLR_FMT_FP32 ? 4 : FMT == HODLR_FMT_FP64 ? 8 : 2;
    int c = warp;
    for (; c + 3 * kConsumers < ncols; c += 4 * kConsumers) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int cc = c + k * kConsumers;
            col_elem<FMT, W>(blk + ((size_t)cc * kRB + kRPL * lane) * sz, mul(cc), acc[k]);
        }
    }
    // tail (< 4 columns, warp-uniform conditions): separate accumulator sets
    if (c < ncols) col_elem<FMT, W>(blk + ((size_t)c * kRB + kRPL * lane) * sz, mul(c), acc[0]);
    if (c + kConsumers < ncols)
        col_elem<FMT, W>(blk + ((size_t)(c + kConsumers) * kRB + kRPL * lane) * sz, mul(c + kConsumers), acc[1]);
    if (c + 2 * kConsumers < ncols)
        col_elem<FMT, W>(blk + ((size_t)(c + 2 * kConsumers) * kRB + kRPL * lane) * sz, mul(c + 2 * kConsumers),
                         acc[2]);
}

template <typename W, typename MulF>
__device__ __forceinline__ void col_block_any(int fmt, const uint8_t* blk, int ncols, int warp, int lane, MulF mul,
                                              W acc[4][kRPL]) {
    switch (fmt) {
        case HODLR_FMT_FP64: col_block<HODLR_FMT_FP64, W>(blk, ncols, warp, lane, mul, acc); break;
        case HODLR_FMT_FP32: col_block<HODLR_FMT_FP32, W>(blk, ncols, warp, lane, mul, acc); break;
        case HODLR_FMT_FP16: col_block<HODLR_FMT_FP16, W>(blk, ncols, warp, lane, mul, acc); break;
        case HODLR_FMT_BF16: col_block<HODLR_FMT_BF16, W>(blk, ncols, warp, lane, mul, acc); break;
        default: col_block<HODLR_FMT_Q52, W>(blk, ncols, warp, lane, mul, acc); break;
    }
}

template <typename W>
struct SvKernelArgs {
    const uint8_t* slab;
    const W* x;
    W* b;
    W* partial;            // fast-path layout: level bases P.lev[].pbase
    W* tbuf;
    SvSync* sync;
    unsigned long long* trace;  // HODLR_TRACE builds only (else unused)
};

struct SmemCtl {
    uint64_t full[kNS], empty[kNS];
    PieceHdr hdr[kNS];
    int fifo[kFifo];               // deferred U pieces: (leaf << 8) | row block
    alignas(16) double ybuf[kFifo][kRB];  // y = D x of those items (working type)
    alignas(16) int16_t cidx[kMaxCols];  // flattened U column -> coefficient slot
    int32_t pbase_c[kMaxCols];     // flattened V' column -> partial buffer base (level pbase + c*nch)
    int32_t pstride_c[kMaxCols];   //                     -> r * nch (stride between nodes)
    int8_t psh_c[kMaxCols];        //                     -> log2(nch)
};

template <typename W>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) k_stream(const __grid_constant__ SvParams P, SvKernelArgs<W> a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;
#ifdef HODLR_PROFILE
    __shared__ long long prof[8];
    if (threadIdx.x < 8) prof[threadIdx.x] = 0;
    const long long t_kernel = clock64();
#endif
    SmemCtl& C = *reinterpret_cast<SmemCtl*>(smem + kNS * kStage);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nlev = P.depth;
    const int nq = P.num_a + P.num_d + P.num_r;  // queue: A leaves, then BC items with R pieces at pos_r
    constexpr int kBlocks = kM / kRB;            // row blocks per leaf

    if (P.mode == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        TR(0);
        for (int s = 0; s < kNS; ++s) {
            mbar_init(&C.full[s], 1);
            mbar_init(&C.empty[s], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp != 0) {
        // consumers build the column tables while the producer starts streaming
        for (int i = threadIdx.x - 32; i < P.gstart[5]; i += kConsumers * 32) {
            const Level& L = P.lev[P.col_level[i]];
            const int sh = nlev - (P.col_level[i] + 1);
            C.cidx[i] = (int16_t)(L.slot + P.col_c[i]);
            C.pbase_c[i] = (int32_t)(L.pbase + (int64_t)P.col_c[i] * L.cst);
            C.pstride_c[i] = L.r * L.cst;
            C.psh_c[i] = (int8_t)sh;
        }
        consumer_sync();
        if (threadIdx.x == 32) TR(22);
    }

    if (warp == 0) {
        // =========================================================== producer
        int stage = 0;
        unsigned phase = 0;
        const uint64_t pol = policy_evict_first();
        unsigned a_items = 0, r_items = 0;
        int fh = 0, ft = 0;             // deferred-U FIFO (warp-uniform); slot = index % kFifo
        bool first_claim = true;
        auto claim = [&]() -> uint8_t* {
            // try_wait parks the warp in hardware until the stage is released: a
            // test_wait spin here steals shared-memory pipe slots from the consumers
            mbar_wait(&C.empty[stage], phase ^ 1u);
            if (first_claim) {
                first_claim = false;
                if (lane == 0) TR(1);
            }
            return stages + (size_t)stage * kStage;
        };
        auto next_stage = [&]() {
            if (++stage == kNS) {
                stage = 0;
                phase ^= 1u;
            }
        };
        // coefficients of every node exist?  (checked without blocking until the
        // deferred-U FIFO is full; the result is cached)
        bool r_ready = false;
        auto check_r = [&](bool block) {
            if (r_ready) return;
            unsigned v = 0;
            if (lane == 0) {
                v = ld_acquire(&a.sync->r_done);
                while (block && v != (unsigned)P.num_r) {
                    __nanosleep(128);
                    v = ld_acquire(&a.sync->r_done);
                }
            }
            r_ready = __shfl_sync(0xffffffffu, v, 0) == (unsigned)P.num_r;
            if (r_ready) asm volatile("fence.proxy.async.global;" ::: "memory");  // t read by TMA below
            if (r_ready && lane == 0) TR(6);
        };
        auto emit_u = [&](int leaf, int rb, int slot) {
            const int wi = sizeof(W) == 8 ? 1 : 0;
            const int wbytes = (int)sizeof(W);
            const uint8_t* ublk = a.slab + P.u_region + (int64_t)leaf * P.us_bytes + (int64_t)rb * P.ublock_bytes;
            for (int p = 0; p < P.nupieces; ++p) {
                const UPiece up = P.up[p];
                const unsigned cb = (unsigned)(up.ncols * kRB * fmt_sz(up.g));
                uint8_t* st = claim();
                if (lane == 0) {
                    if (fh == 0 && p == 0) TR(14);
                    PieceHdr& h = C.hdr[stage];
                    h.type = PT_U;
                    h.leaf = leaf;
                    h.a = rb;
                    h.b = slot;
                    h.last = p;
                    mbar_arrive_tx(&C.full[stage], (unsigned)P.u_data_off[wi] + cb);
                }
                __syncwarp();
                if (lane < nlev) {
                    const Level& L = P.lev[lane];
                    if (L.r > 0) {
                        const int k = lane + 1;
                        const int jsib = (leaf >> (nlev - k)) ^ 1;
                        const W* src = a.tbuf + L.tbase + (int64_t)jsib * L.tstride;
                        bulk_g2s(st + (size_t)L.slot * wbytes, src, (unsigned)(L.tstride * wbytes), &C.full[stage]);
                    }
                } else if (lane == 31) {
                    bulk_g2s_stream(st + P.u_data_off[wi], ublk + P.ugoff[up.g] + (int64_t)up.c0 * kRB * fmt_sz(up.g),
                                    cb, &C.full[stage], pol);
                }
                __syncwarp();
                next_stage();
            }
        };
        // R pieces wait for every A leaf's partials.  A producer that takes one
        // before that keeps streaming BC items and parks the piece (<= kRPend),
        // emitting it at the first item boundary that sees a_done complete.
        bool a_ready = false;
        auto check_a = [&](bool block) {
            if (a_ready) return;
            unsigned v = 0;
            if (lane == 0) {
                v = ld_acquire(&a.sync->a_done);
                while (block && v != (unsigned)P.num_a) {
                    __nanosleep(128);
                    v = ld_acquire(&a.sync->a_done);
                }
            }
            a_ready = __shfl_sync(0xffffffffu, v, 0) == (unsigned)P.num_a;
            if (a_ready) {
                asm volatile("fence.proxy.async.global;" ::: "memory");  // partials read by TMA below
                if (lane == 0) TR(5);
            }
        };
        // An R piece's descriptor and source are resolved when the piece is taken,
        // before the wait for the A partials: the parameter-table reads (cold in
        // the constant cache, ~us under full HBM load) stay off the critical path,
        // and the consumer gets the piece from the stage header.
        struct RJob {
            const W* src;
            unsigned bytes;
            int lv, j0, j1, c01;
        };
        auto make_r = [&](int ri) {
            const RPiece rp = P.rp[ri];
            const Level& L = P.lev[rp.lv];
            const int64_t cnt = (int64_t)(rp.j1 - rp.j0) * (rp.c1 - rp.c0) * L.cst;
            RJob j;
            j.src = a.partial + L.pbase + ((int64_t)rp.j0 * L.r + rp.c0) * L.cst;
            j.bytes = (unsigned)round_up16_d(cnt * (int64_t)sizeof(W));
            j.lv = rp.lv;
            j.j0 = rp.j0;
            j.j1 = rp.j1;
            j.c01 = rp.c0 | (rp.c1 << 16);
            asm volatile("" ::"l"(j.src), "r"(j.bytes), "r"(j.lv), "r"(j.j0), "r"(j.j1), "r"(j.c01));
            return j;
        };
        auto emit_r = [&](const RJob& j) {
            ++r_items;
            if (lane == 0) TRV(13, r_items);
            uint8_t* st = claim();
            if (lane == 0) {
                PieceHdr& h = C.hdr[stage];
                h.type = PT_R;
                h.a = j.lv;
                h.leaf = j.j0;
                h.b = j.j1;
                h.last = j.c01;
                mbar_arrive_tx(&C.full[stage], j.bytes);
                bulk_g2s(st, j.src, j.bytes, &C.full[stage]);
                TR(20);
            }
            __syncwarp();
            next_stage();
        };
        constexpr int kRPend = 4;
        RJob rpend[kRPend];
        int nrp = 0;
        auto flush_r = [&](bool block) {
            if (nrp == 0) return;
            check_a(block);
            if (!a_ready) return;
            for (int i = 0; i < nrp; ++i) emit_r(rpend[i]);
            nrp = 0;
        };
        auto flush_u = [&](bool block) {
            if (block) flush_r(true);  // never wait for the coefficients while holding an R piece
            if (fh == ft) return;
            check_r(block);
            if (!r_ready) return;
            while (fh != ft) {
                const int e = C.fifo[fh % kFifo];
                emit_u(e >> 8, e & 0xff, fh % kFifo);
                ++fh;
            }
        };

        // ---- one atomic queue, fetched two ahead:  [A leaves][BC items, R pieces at pos_r]
        // Every cross-CTA wait (R on all A leaves, U on all R pieces) targets work
        // that sits EARLIER in the queue, i.e. was already taken by a running CTA,
        // so progress never depends on CTAs being co-resident.
        // static_first: CTA b's first entry is b (no contended atomic before the
        // first load; the counter then hands out entries from gridDim.x on).
        // Progress still only needs every CTA of the grid to start eventually.
        const int qoff = P.static_first ? (int)gridDim.x : 0;
        int n1 = 0, n2 = 0;
        if (lane == 0) {
            if (P.static_first) {
                n1 = (int)blockIdx.x;
                n2 = (int)atomicAdd(&a.sync->queue, 1u) + qoff;
            } else {
                n1 = (int)atomicAdd(&a.sync->queue, 2u);
                n2 = n1 + 1;
            }
            TR(23);
        }
        const int dsz = fmt_sz(P.leaf_fmt);
        bool first_q = true;
        for (;;) {
            const int q = __shfl_sync(0xffffffffu, n1, 0);
            if (first_q) {
                first_q = false;
                if (lane == 0) TR(30);
            }
            if (q >= nq) break;
            n1 = n2;
            if (lane == 0) n2 = (int)atomicAdd(&a.sync->queue, 1u) + qoff;
            if (q < P.num_a) {
                // ---- A: partial V'^T x of one (leaf, piece) or one whole leaf
                const int per_leaf = P.napieces / P.a_group;
                const int leaf = q / per_leaf, p0 = (q - leaf * per_leaf) * P.a_group;
                const uint8_t* base = a.slab + (int64_t)leaf * P.vs_bytes;
                ++a_items;
                for (int p = p0; p < p0 + P.a_group; ++p) {
                    const APiece ap = P.ap[p];
                    uint8_t* st = claim();
                    const AGroup& G = P.ag[ap.g];
                    const unsigned cb = (unsigned)(ap.nrows * G.vpad * fmt_sz(G.fmt));
                    const unsigned xb = (unsigned)(ap.nrows * sizeof(W));
                    if (lane == 0) {
                        PieceHdr& h = C.hdr[stage];
                        h.type = PT_A;
                        h.leaf = leaf;
                        h.a = p;
                        // item end: 1; 2 = also this CTA's last A item (the next queue
                        // entry is not A): its consumers then publish the CTA's A items
                        h.last = p + 1 < p0 + P.a_group ? 0 : n1 >= P.num_a ? 2 : 1;
                        mbar_arrive_tx(&C.full[stage], xb + cb);
                        bulk_g2s(st, a.x + (int64_t)leaf * kM + ap.r0, xb, &C.full[stage]);
                        bulk_g2s_stream(st + kXB, base + G.voff + (int64_t)ap.r0 * G.vpad * fmt_sz(G.fmt),
                                        cb, &C.full[stage], pol);
                        TR(2);
                        TRV(11, a_items);
                    }
                    __syncwarp();
                    next_stage();
                }
                continue;
            }
            const int qq = q - P.num_a;
            if (qq >= P.pos_r && qq < P.pos_r + P.num_r) {
                // ---- R: reduce node partials (needs every leaf's partials)
                if (P.mode == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
                if (lane == 0 && r_items + nrp == 0) TR(4);
                if (nrp == kRPend) flush_r(true);
                rpend[nrp++] = make_r(qq - P.pos_r);
                flush_r(P.mode == 2 || P.rdefer == 0);
                continue;
            }
            // ---- BC: y = D x now (kept in this CTA's y slot), b = U t + y once t exists
            const int qb = qq < P.pos_r ? qq : qq - P.num_r;
            const int leaf = qb / kBlocks, rb = qb % kBlocks;
            if (lane == 0) {
                if (ft == 0) TR(3);
                TRV(12, ft + 1);
            }
            if (ft - fh == kFifo) flush_u(true);  // frees the y slot this item will use
            const int slot = ft % kFifo;
            const uint8_t* blk = a.slab + P.d_region + (int64_t)leaf * P.ds_bytes + (int64_t)rb * P.dblock_bytes;
            const int dcols = P.dcols_w[sizeof(W) == 8], dpieces = P.dpieces_w[sizeof(W) == 8];
            const int xoff = dcols * (int)sizeof(W);  // x segment, then the D columns (16-B aligned)
            for (int p = 0; p < dpieces; ++p) {
                uint8_t* st = claim();
                const int c0 = p * dcols;
                const int nc = min(dcols, kM - c0);
                const unsigned cb = (unsigned)(nc * kRB * dsz);
                const unsigned xb = (unsigned)(nc * sizeof(W));
                if (lane == 0) {
                    PieceHdr& h = C.hdr[stage];
                    h.type = PT_D;
                    h.leaf = leaf;
                    h.a = rb;
                    h.b = c0;
                    h.last = (p == dpieces - 1) ? 1 + slot : 0;
                    mbar_arrive_tx(&C.full[stage], xb + cb);
                    bulk_g2s(st, a.x + (int64_t)leaf * kM + c0, xb, &C.full[stage]);
                    bulk_g2s_stream(st + xoff, blk + (int64_t)c0 * kRB * dsz, cb, &C.full[stage], pol);
                }
                __syncwarp();
                next_stage();
            }
            if (lane == 0) C.fifo[ft % kFifo] = (leaf << 8) | rb;
            __syncwarp();
            ++ft;
            flush_r(false);
            flush_u(false);
        }
        if (lane == 0) TR(7);
        flush_u(true);
        if (lane == 0) TR(8);
        claim();
        if (lane == 0) {
            C.hdr[stage].type = PT_END;
            mbar_arrive(&C.full[stage]);
        }
        __syncwarp();
    } else {
        // =========================================================== consumers
        const int cw = warp - 1;
        const int ctid = threadIdx.x - 32;
        int stage = 0;
        unsigned phase = 0;
        unsigned my_a = 0;  // A pieces this CTA's consumers finished
        bool first_u_seen = false;
        W aacc[2][4];   // phase A: column sums of the current format group
        W bacc[4][kRPL];  // BC items: row sums (kRPL rows per lane, 4 chains)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) aacc[i][e] = W(0);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int r = 0; r < kRPL; ++r) bacc[k][r] = W(0);
#ifdef HODLR_TRACE
        long long wait_cyc = 0, t_loop = clock64();
        long long busy[6] = {0, 0, 0, 0, 0, 0}, nb[6] = {0, 0, 0, 0, 0, 0}, t_busy = 0;
        long long split[4] = {0, 0, 0, 0}, ts0 = 0;
        int busy_type = 0;
#endif
        for (;;) {
            PROF_T(tw);
#ifdef HODLR_TRACE
            const long long tw0 = clock64();
#endif
            mbar_wait(&C.full[stage], phase);
#ifdef HODLR_TRACE
            wait_cyc += clock64() - tw0;
            t_busy = clock64();
            busy_type = C.hdr[stage].type;
#endif
            const PieceHdr h = C.hdr[stage];
            uint8_t* st = stages + (size_t)stage * kStage;
            if (h.type == PT_END) {
                if (ctid == 0) {
                    TR(9);
#ifdef HODLR_TRACE
                    TRV(28, wait_cyc);
                    TRV(29, clock64() - t_loop);
                    for (int i = 0; i < 6; ++i) {
                        TRV(32 + i, busy[i]);
                        TRV(38 + i, nb[i]);
                    }
                    for (int i = 0; i < 4; ++i) TRV(44 + i, split[i]);
#endif
                }
                break;
            }
            PROF_ADD(h.type == PT_R ? 0 : h.type, clock64() - tw);  // [1] A [2] D [3] U [0] R
            bool scratch = false;  // the stage was reused as reduction scratch
            if (h.type == PT_A) {
                if (ctid == 0 && my_a < 4) TR(24 + my_a);  // arrival of this CTA's A pieces 1..4
                const APiece ap = P.ap[h.a];
#ifdef HODLR_TRACE
                ts0 = clock64();
#endif
                const AGroup& G = P.ag[ap.g];
                a_piece<W>(G.fmt, st + kXB, ap.nrows, G.vpad, reinterpret_cast<const W*>(st), cw, lane, aacc);
#ifdef HODLR_TRACE
                split[0] += clock64() - ts0;
                ts0 = clock64();
#endif
                if (ap.last_of_group) {
                    // combine the warps' column sums in warp order, write the partials
                    W* red = reinterpret_cast<W*>(st);
                    const int vp = G.vpad;
                    consumer_sync();
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int qq = lane + 32 * i;
                        if (4 * qq < vp)
#pragma unroll
                            for (int e = 0; e < 4; ++e) red[cw * vp + 4 * qq + e] = aacc[i][e];
                    }
                    consumer_sync();
                    for (int c = ctid; c < G.ncols; c += kConsumers * 32) {
                        W s = red[c];
#pragma unroll
                        for (int w = 1; w < kConsumers; ++w) s += red[w * vp + c];
                        const int flat = P.gstart[G.fmt] + G.c0 + c;
                        const int sh = C.psh_c[flat];
                        const int jn = h.leaf >> sh;
                        a.partial[(int64_t)C.pbase_c[flat] + (int64_t)jn * C.pstride_c[flat] +
                                  (int64_t)(h.leaf - (jn << sh)) * ap.npc + ap.chunk] = s;
                    }
#pragma unroll
                    for (int i = 0; i < 2; ++i)
#pragma unroll
                        for (int e = 0; e < 4; ++e) aacc[i][e] = W(0);
                    scratch = true;
                }
#ifdef HODLR_TRACE
                split[1] += clock64() - ts0;
#endif
            } else if (h.type == PT_D) {
                const W* xs = reinterpret_cast<const W*>(st);
                const int dcols = P.dcols_w[sizeof(W) == 8];
                const int nc = min(dcols, kM - h.b);
                auto mul = [&](int c) { return xs[c]; };
#ifdef HODLR_TRACE
                ts0 = clock64();
#endif
                col_block_any<W>(P.leaf_fmt, st + dcols * (int)sizeof(W), nc, cw, lane, mul, bacc);
#ifdef HODLR_TRACE
                split[2] += clock64() - ts0;
                ts0 = clock64();
#endif
                if (h.last) {
                    W* red = reinterpret_cast<W*>(st);
                    consumer_sync();
#pragma unroll
                    for (int r = 0; r < kRPL; ++r)
                        red[cw * kRB + kRPL * lane + r] = (bacc[0][r] + bacc[1][r]) + (bacc[2][r] + bacc[3][r]);
                    consumer_sync();
                    if (ctid < kRB) {
                        W s = red[ctid];
#pragma unroll
                        for (int w = 1; w < kConsumers; ++w) s += red[w * kRB + ctid];
                        reinterpret_cast<W*>(C.ybuf[h.last - 1])[ctid] = s;  // y = D x, kept for the U piece
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int r = 0; r < kRPL; ++r) bacc[k][r] = W(0);
                    scratch = true;
#ifdef HODLR_TRACE
                    split[3] += clock64() - ts0;
#endif
                }
            } else if (h.type == PT_R) {
                // t for (node, column) pairs: fixed-order sums over the node's leaves
                RPiece rp;
                rp.lv = (int16_t)h.a;
                rp.j0 = h.leaf;
                rp.j1 = h.b;
                rp.c0 = h.last & 0xffff;
                rp.c1 = h.last >> 16;
                const Level& L = P.lev[rp.lv];
                const int nch = (1 << (nlev - 1 - rp.lv)) * L.npc;  // partials per (node, column)
                const int ncol = rp.c1 - rp.c0;
                const int npairs = (rp.j1 - rp.j0) * ncol;
                const W* v = reinterpret_cast<const W*>(st);
                if (nch >= 32) {
                    for (int p = cw; p < npairs; p += kConsumers) {
                        W s = W(0);
                        for (int i = lane; i < nch; i += 32) s += v[(int64_t)p * L.cst + i];
                        s = warp_sum(s);
                        if (lane == 0) {
                            const int j = rp.j0 + p / ncol, c = rp.c0 + p % ncol;
                            a.tbuf[L.tbase + (int64_t)j * L.tstride + c] = s;
                        }
                    }
                } else {
                    for (int p = ctid; p < npairs; p += kConsumers * 32) {
                        W s = v[(int64_t)p * L.cst];
                        for (int i = 1; i < nch; ++i) s += v[(int64_t)p * L.cst + i];
                        const int j = rp.j0 + p / ncol, c = rp.c0 + p % ncol;
                        a.tbuf[L.tbase + (int64_t)j * L.tstride + c] = s;
                    }
                }
                scratch = true;
            } else {  // PT_U: b = U t + y, one column chunk of U per piece
                if (ctid == 0 && !first_u_seen) {
                    first_u_seen = true;
                    TR(15);
                }
                const int wi = sizeof(W) == 8 ? 1 : 0;
                const UPiece up = P.up[h.last];
                const W* coef = reinterpret_cast<const W*>(st);
                const W* ys = reinterpret_cast<const W*>(C.ybuf[h.b]);
                {
                    const int16_t* ci = C.cidx + P.gstart[up.g] + up.c0;
                    auto mul = [&](int c) { return coef[ci[c]]; };
                    col_block_any<W>(up.g, st + P.u_data_off[wi], up.ncols, cw, lane, mul, bacc);
                }
                if (h.last == P.nupieces - 1) {
                    W* red = reinterpret_cast<W*>(st);  // the stage is scratch once every warp is done with it
                    consumer_sync();
#pragma unroll
                    for (int r = 0; r < kRPL; ++r)
                        red[cw * kRB + kRPL * lane + r] = (bacc[0][r] + bacc[1][r]) + (bacc[2][r] + bacc[3][r]);
                    consumer_sync();
                    if (ctid < kRB) {
                        W s = red[ctid];
#pragma unroll
                        for (int w = 1; w < kConsumers; ++w) s += red[w * kRB + ctid];
                        a.b[(int64_t)h.leaf * kM + h.a * kRB + ctid] = s + ys[ctid];  // levels, then the leaf
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int r = 0; r < kRPL; ++r) bacc[k][r] = W(0);
                    scratch = true;
                }
            }
            if (scratch && ((h.type == PT_A && h.last) || h.type == PT_R)) {
                consumer_sync();  // scratch reads and the item's global stores are done
                // Publish GPU-wide from a consumer thread (it has no bulk copies
                // in flight, so its fence does not wait for the ring's loads):
                // all of this CTA's A pieces at once after its last one, every
                // R piece.  Release pattern: CTA barrier, fence.acq_rel.gpu,
                // relaxed reduction; readers ld.acquire the counter.
                if (h.type == PT_A && h.last) ++my_a;
                if (ctid == 0 && ((h.type == PT_A && h.last == 2 && P.mode == 0) || h.type == PT_R)) {
                    if (h.type == PT_A) TR(16); else TR(18);
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    if (h.type == PT_A) TR(17); else TR(19);
                    if (h.type == PT_A)
                        asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(&a.sync->a_done), "r"(my_a) : "memory");
                    else
                        asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(&a.sync->r_done), "r"(1u) : "memory");
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&C.empty[stage]);
#ifdef HODLR_TRACE
            busy[busy_type] += clock64() - t_busy;
            nb[busy_type] += 1;
#endif
            if (++stage == kNS) {
                stage = 0;
                phase ^= 1u;
            }
        }
    }
    // ---- teardown: the last CTA resets the per-call state and bumps the epoch
    __syncthreads();
#ifdef HODLR_PROFILE
    if (threadIdx.x == 0)
        printf("PROF cta %3d total %lld | A_emitted %lld firstC %lld firstC_ready %lld | cons_wait(sum 8 warps) A %lld D %lld U %lld R %lld\n",
               blockIdx.x, clock64() - t_kernel, prof[4], prof[5], prof[6], prof[1], prof[2], prof[3], prof[0]);
#endif
    __shared__ unsigned s_last;
    if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&a.sync->done) : "memory");
        s_last = old == gridDim.x - 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) TR(10);
    if (s_last) {
        if (threadIdx.x == 0) {
            a.sync->queue = 0u;
            a.sync->done = 0u;
            a.sync->a_done = 0u;
            a.sync->r_done = 0u;
            __threadfence();
            st_release(&a.sync->epoch, a.sync->epoch + 1u);  // calls completed (informational)
        }
    }
}

size_t smem_bytes() { return (size_t)kNS * kStage + sizeof(SmemCtl); }

// workspace: [SvSync | leaf B counters] (zeroed once, reset per call) [partials] [coefficients]
size_t sv_sync_bytes(int nleaves) {  // two SvSync (split launches), then the leaf counters
    return (2 * sizeof(SvSync) + (size_t)nleaves * sizeof(unsigned) + 255) / 256 * 256;
}

int64_t round_up16(int64_t v) { return (v + 15) / 16 * 16; }

}  // namespace

// ============================================================== host side
hodlr_status SVG(sv_prepare)(const SvInput& in, SvPlan& sv, bool* ok) {
    sv = SvPlan{};
    sv.geo = HODLR_SV_GEO;
    sv.ctas_per_sm = kCtasPerSm;
    *ok = false;
    const auto& nodes = *in.nodes;
    const auto& leaves = *in.leaves;
    const int depth = in.nlev;
    if (depth < 1 || depth > kMaxLev || leaves.empty()) return HODLR_OK;
    const int nleaves = (int)leaves.size();
    if (nleaves != (1 << depth) || (int)in.chunks->size() != nleaves) return HODLR_OK;
    const int lf = leaves[0].fmt;
    if (lf != HODLR_FMT_FP64 && lf != HODLR_FMT_FP32) return HODLR_OK;
    for (int i = 0; i < nleaves; ++i)
        if (leaves[i].m != kM || leaves[i].row0 != i * kM || leaves[i].fmt != lf || leaves[i].ld != kM)
            return HODLR_OK;
    if ((int)nodes.size() != (1 << (depth + 1)) - 2) return HODLR_OK;
    // uniform rank and format per level, node ids level-major
    SvParams P;
    memset(&P, 0, sizeof(P));
    P.depth = depth;
    P.nleaves = nleaves;
    P.nnodes = (int)nodes.size();
    P.leaf_fmt = lf;
    for (int k = 1; k <= depth; ++k) {
        const int base = (1 << k) - 2;
        const NodeDesc& n0 = nodes[base];
        int rmax = 0;
        for (int j = 0; j < (1 << k); ++j) {  // ranks may differ per block: padded to the level max
            const NodeDesc& nd = nodes[base + j];
            if (nd.level != k || nd.ext_slot >= 0 || nd.u_fmt != n0.u_fmt || nd.v_fmt != n0.u_fmt ||
                nd.nchunk != (1 << (depth - k)) || nd.row0 != j * (kM << (depth - k)))
                return HODLR_OK;
            rmax = std::max(rmax, std::max(nd.rv, nd.ru));
        }
        P.lev[k - 1].r = rmax;
        P.lev[k - 1].fmt = n0.u_fmt;
    }
    // column lists per format group (level-major inside a group)
    int flat = 0;
    for (int g = 0; g < 5; ++g) {
        P.gstart[g] = (int16_t)flat;
        int cnt = 0;
        for (int k = 0; k < depth; ++k) {
            if (P.lev[k].fmt != g) continue;
            for (int c = 0; c < P.lev[k].r; ++c) {
                if (flat >= kMaxCols) return HODLR_OK;
                P.col_level[flat] = (int8_t)k;
                P.col_c[flat] = (int16_t)c;
                ++flat;
                ++cnt;
            }
        }
        P.gcols[g] = cnt;
    }
    // phase-A column groups: whole levels of one format, <= 256 columns each
    P.nag = 0;
    int lev_ag[kMaxLev];
    for (int k = 0; k < depth; ++k) lev_ag[k] = -1;
    for (int g = 0; g < 5; ++g) {
        int c0 = 0, cur = -1;
        for (int k = 0; k < depth; ++k) {
            if (P.lev[k].fmt != g || P.lev[k].r == 0) continue;
            const int r = P.lev[k].r;
            if (r > 256) return HODLR_OK;
            if (cur < 0 || P.ag[cur].ncols + r > 256) {
                if (P.nag == kMaxAG) return HODLR_OK;
                cur = P.nag++;
                P.ag[cur] = AGroup{g, c0, 0, 0, 0};
            }
            P.ag[cur].ncols += r;
            lev_ag[k] = cur;
            c0 += r;
        }
    }
    for (int i = 0; i < P.nag; ++i) P.ag[i].vpad = (P.ag[i].ncols + 3) / 4 * 4;
    P.gstart[5] = (int16_t)flat;
    if (flat == 0) return HODLR_OK;  // all ranks zero: generic path
    // coefficient slots and partial / coefficient buffers
    int slot = 0;
    int64_t tb = 0, pb = 0;
    for (int k = 0; k < depth; ++k) {
        Level& L = P.lev[k];
        L.tstride = (L.r + 3) / 4 * 4;
        L.slot = slot;
        slot += L.tstride;
        L.tbase = tb;
        tb += (int64_t)L.tstride << (k + 1);
    }
    P.coef_elems = slot;
    // slab geometry
    const int dsz = fmt_bytes(lf);
    int64_t vs = 0;
    for (int i = 0; i < P.nag; ++i) {
        P.ag[i].voff = vs;
        vs += (int64_t)kM * P.ag[i].vpad * fmt_bytes(P.ag[i].fmt);
    }
    P.dblock_bytes = (int64_t)kM * kRB * dsz;
    int64_t ub = 0;
    for (int g = 0; g < 5; ++g) {
        P.ugoff[g] = ub;
        ub += round_up16((int64_t)P.gcols[g] * kRB * fmt_bytes(g));
    }
    P.ublock_bytes = ub;
    P.vs_bytes = vs;
    P.ds_bytes = (kM / kRB) * P.dblock_bytes;
    P.us_bytes = (kM / kRB) * P.ublock_bytes;
    P.d_region = round_up16((int64_t)nleaves * P.vs_bytes + 240);
    P.u_region = round_up16(P.d_region + (int64_t)nleaves * P.ds_bytes + 240);
    const int64_t slab_total = P.u_region + (int64_t)nleaves * P.us_bytes;
    // phase-A pieces: row blocks of each format's V' sub-slab (multiples of 8 rows)
    P.napieces = 0;
    for (int g = 0; g < P.nag; ++g) {
        int rows = (kStage - kXB) / (P.ag[g].vpad * fmt_bytes(P.ag[g].fmt));
        rows = std::min(kM, rows / 8 * 8);
        if (rows < 8) return HODLR_OK;
        for (int r0 = 0; r0 < kM; r0 += rows) {
            if (P.napieces == kMaxPieces) return HODLR_OK;
            const int nr = std::min(rows, kM - r0);
            P.ap[P.napieces++] = APiece{g, r0, nr, r0 / rows, (kM + rows - 1) / rows, r0 + nr == kM};
        }
    }
    // A items: single pieces while leaves are scarce (cfg2: 256 leaves for ~300
    // CTAs), whole leaves once every CTA gets a few (1/npc the partials)
    int sms_now = 148, dev_now = 0;
    cudaGetDevice(&dev_now);
    cudaDeviceGetAttribute(&sms_now, cudaDevAttrMultiProcessorCount, dev_now);
    // (pairs of pieces when leaves are scarce and one column group: half the
    // partials for the reduction; cfg2 42.5 -> 41.5 us, profiles/round1_sv_sweep_cfg2.txt)
    P.a_group = nleaves >= 2 * kCtasPerSm * sms_now ? P.napieces
                : (P.nag == 1 && P.napieces > 2 && P.napieces % 2 == 0) ? 2 : 1;
    // 4-CTA geometry (small stages, so more pieces per leaf): whole leaves already at one leaf
    // per CTA once a leaf has >= 4 pieces (cfg5 eps=1e-4: 74.6 -> 72.7 us; with 2 pieces per
    // leaf, eps=1e-2, single pieces stay 1% ahead)
    if (kCtasPerSm >= 4 && nleaves >= kCtasPerSm * sms_now && P.napieces >= 4) P.a_group = P.napieces;
    if (getenv("HODLR_B200_A_GROUP")) {
        // 1: single pieces; k (one format group, k | napieces): k consecutive row
        // pieces per item, npc = napieces / k partials per leaf; else whole leaves
        const int k = atoi(getenv("HODLR_B200_A_GROUP"));
        P.a_group = k <= 1 ? 1 : (P.nag == 1 && k < P.napieces && P.napieces % k == 0) ? k : P.napieces;
    }
    if (P.a_group > 1 && P.a_group < P.napieces) {
        for (int i = 0; i < P.napieces; ++i) {
            P.ap[i].chunk = i / P.a_group;
            P.ap[i].npc = P.napieces / P.a_group;
            P.ap[i].last_of_group = i % P.a_group == P.a_group - 1;
        }
    } else for (int i = 0; i < P.napieces; ++i) {
        if (P.a_group > 1) {
            P.ap[i].chunk = 0;
            P.ap[i].npc = 1;
        } else {
            P.ap[i].last_of_group = 1;
        }
    }
    // partials: per level [node][column][cst], entries (leaf of node, chunk) in
    // leaf-major order, each (node, column) run 32-byte aligned
    for (int k = 0; k < depth; ++k) {
        Level& L = P.lev[k];
        L.npc = 0;
        for (int i = 0; i < P.napieces; ++i)
            if (P.ap[i].g == lev_ag[k]) L.npc = P.ap[i].npc;
        if (L.r > 0 && L.npc == 0) return HODLR_OK;
        L.cst = (int)(((int64_t)(nleaves >> (k + 1)) * std::max(L.npc, 1) + 3) / 4 * 4);
        L.pbase = pb;
        pb += (int64_t)L.r * L.cst << (k + 1);
    }
    if (pb >= (int64_t(1) << 31)) return HODLR_OK;  // int32 partial indices in shared tables
    // reduction scratch in an A piece's stage: kConsumers x vpad values
    for (int g = 0; g < P.nag; ++g)
        if ((size_t)kConsumers * P.ag[g].vpad * 8 > (size_t)kStage) return HODLR_OK;
    // phase-B pieces: column blocks of a 64-row block
    // [x segment: dcols working values][dcols D columns]; balanced pieces
    for (int wi = 0; wi < 2; ++wi) {
        const int wsz = wi ? 8 : 4;
        int dc = std::min(kM, (int)(kStage / (kRB * dsz + wsz)) / 8 * 8);
        const int np = (kM + dc - 1) / dc;
        dc = ((kM + np - 1) / np + 7) / 8 * 8;
        P.dcols_w[wi] = dc;
        P.dpieces_w[wi] = (kM + dc - 1) / dc;
    }
    // U pieces: coefficients | column chunk of the U block | reduction scratch
    for (int wi = 0; wi < 2; ++wi) P.u_data_off[wi] = (int)round_up16((int64_t)P.coef_elems * (wi ? 8 : 4));
    {
        const int64_t room = kStage - P.u_data_off[1] - 16;
        if ((size_t)kConsumers * kRB * 8 > (size_t)kStage) return HODLR_OK;  // combine scratch
        P.nupieces = 0;
        for (int g = 0; g < 5; ++g) {
            if (P.gcols[g] == 0) continue;
            int per = (int)(room / ((int64_t)kRB * fmt_bytes(g)));
            per = per >= 8 ? per / 8 * 8 : per;  // keep chunk offsets 16-byte aligned
            if (per < 1 || (per < 8 && P.gcols[g] > per)) return HODLR_OK;
            if (per >= 8) {  // balance the chunks of this group
                const int np = (P.gcols[g] + per - 1) / per;
                per = std::min(per, ((P.gcols[g] + np - 1) / np + 7) / 8 * 8);
            }
            for (int c0 = 0; c0 < P.gcols[g]; c0 += per) {
                if (P.nupieces == kMaxUPieces) return HODLR_OK;
                P.up[P.nupieces++] = UPiece{g, c0, std::min(per, P.gcols[g] - c0), 0};
            }
        }
        if (P.nupieces == 0) return HODLR_OK;
    }
    P.num_a = nleaves * (P.napieces / P.a_group);
    P.num_d = nleaves * (kM / kRB);
    // node-reduction pieces (R items): a level's partials are [node][column][leaf]
    // R pieces of <= 8 KB spread the reduction over more CTAs (cfg2 41.6 -> 41.0 us
    // flushed, 39.0 -> 37.0 us hot; profiles/round1_sv_sweep_cfg2.txt); trees whose
    // pieces would not fit kMaxRPieces or whose (node, column) runs exceed 8 KB use
    // whole stages.  HODLR_R_BYTES overrides (sweeps).
    auto build_r = [&](int64_t rcap) -> bool {
        P.num_r = 0;
        for (int k = 0; k < depth; ++k) {
            const Level& L = P.lev[k];
            if (L.r == 0) continue;
            const int nodes_k = 1 << (k + 1);
            const int64_t nch = L.cst;
            const int64_t node_bytes = (int64_t)L.r * nch * 8;
            auto add = [&](int j0, int j1, int c0, int c1) {
                if (P.num_r == kMaxRPieces) return false;
                if ((L.pbase + ((int64_t)j0 * L.r + c0) * nch) % 4) return false;  // 16-B aligned source
                P.rp[P.num_r++] = RPiece{(int16_t)k, 0, j0, j1, c0, c1};
                return true;
            };
            if (node_bytes <= rcap) {
                int per = (int)std::min<int64_t>(nodes_k, rcap / node_bytes);
                if (per >= 4) per = per / 4 * 4;
                for (int j0 = 0; j0 < nodes_k; j0 += per)
                    if (!add(j0, std::min(nodes_k, j0 + per), 0, L.r)) return false;
            } else {
                const int cols = (int)(rcap / (nch * 8));
                if (cols < 1) return false;
                for (int j = 0; j < nodes_k; ++j)
                    for (int c0 = 0; c0 < L.r; c0 += cols)
                        if (!add(j, j + 1, c0, std::min(L.r, c0 + cols))) return false;
            }
        }
        return true;
    };
    int64_t rcap = 8192;
    if (const char* e = getenv("HODLR_R_BYTES")) rcap = std::max<int64_t>(1024, std::min<int64_t>(kStage, atoll(e)));
    if (!build_r(rcap) && !(rcap != kStage && build_r(kStage))) return HODLR_OK;
    // R pieces: late enough that the A leaves are (nearly) done, early enough that
    // they are taken before any running CTA could fill its deferred-U FIFO
    P.pos_r = std::min(P.num_d / 6, kFifo * 16);  // (assumes >= 16 CTAs can run at once)
    // parking R pieces (HODLR_R_DEFER=1) measured slower on cfg2 (42.5 -> 45.1 us):
    // a parked piece is only re-checked at BC item boundaries, so the partial
    // reduction starts ~6 us later than with the blocking wait
    P.rdefer = 0;
    P.static_first = 0;
    if (const char* e = getenv("HODLR_SV_STATIC")) P.static_first = atoi(e) != 0;
    if (const char* e = getenv("HODLR_R_DEFER")) P.rdefer = atoi(e) != 0;
    if (const char* e = getenv("HODLR_POS_R")) P.pos_r = std::max(0, std::min(P.num_d, atoi(e)));  // tuning sweeps

    // ---- relayout the quantised level-batched arena into leaf slabs (bytes)
    std::vector<uint8_t> arena(in.arena_bytes);
    if (cudaMemcpy(arena.data(), in.d_arena, in.arena_bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        return HODLR_OK;
    std::vector<uint8_t> slab((size_t)slab_total, 0);
    for (int leaf = 0; leaf < nleaves; ++leaf) {
        uint8_t* out_v = slab.data() + (size_t)leaf * P.vs_bytes;
        uint8_t* out_d = slab.data() + P.d_region + (size_t)leaf * P.ds_bytes;
        uint8_t* out_u = slab.data() + P.u_region + (size_t)leaf * P.us_bytes;
        for (int g = 0; g < 5; ++g) {
            const int w = fmt_bytes(g);
            int col = 0;  // flat column inside format g (levels padded to their max rank)
            for (int k = 0; k < depth; ++k) {
                if (P.lev[k].fmt != g || P.lev[k].r == 0) continue;
                const int lvl = k + 1;
                const NodeDesc& nd = nodes[(1 << lvl) - 2 + (leaf >> (depth - lvl))];
                const int64_t roff = (int64_t)leaf * kM - nd.row0;
                const AGroup& G = P.ag[lev_ag[k]];
                for (int c = 0; c < P.lev[k].r; ++c, ++col) {
                    if (c < nd.rv) {  // V' row-major inside the level's A group
                        const uint8_t* vsrc = arena.data() + nd.v_off + ((int64_t)c * nd.v_ld + roff) * w;
                        for (int r = 0; r < kM; ++r)
                            memcpy(out_v + G.voff + ((int64_t)r * G.vpad + (col - G.c0)) * w, vsrc + (int64_t)r * w,
                                   (size_t)w);
                    }
                    if (c < nd.ru) {  // U column-major per 64-row block
                        const uint8_t* usrc = arena.data() + nd.u_off + ((int64_t)c * nd.u_ld + roff) * w;
                        for (int rb = 0; rb < kM / kRB; ++rb)
                            memcpy(out_u + rb * P.ublock_bytes + P.ugoff[g] + (int64_t)col * kRB * w,
                                   usrc + (int64_t)rb * kRB * w, (size_t)kRB * w);
                    }
                }
            }
        }
        const uint8_t* dsrc = arena.data() + leaves[leaf].off;  // row-major m x ld
        for (int rb = 0; rb < kM / kRB; ++rb)
            for (int c = 0; c < kM; ++c)
                for (int r = 0; r < kRB; ++r)
                    memcpy(out_d + rb * P.dblock_bytes + ((int64_t)c * kRB + r) * dsz,
                           dsrc + ((int64_t)(rb * kRB + r) * kM + c) * dsz, (size_t)dsz);
    }
    int dev = 0, sms = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    const size_t smem = smem_bytes();
    (void)coop;
    if (sms <= 0 ||
        cudaFuncSetAttribute(k_stream<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(k_stream<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return HODLR_OK;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<double>, kThreads, smem);
    if (occ < 1) return HODLR_OK;
    void* d = nullptr;
    if (cudaMalloc(&d, slab.size()) != cudaSuccess) return HODLR_OK;
    if (cudaMemcpy(d, slab.data(), slab.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return HODLR_OK;
    }
    sv.dev = d;
    sv.dev_bytes = slab.size();
    sv.slab = (const uint8_t*)d;
    sv.nleaves = nleaves;
    sv.nnodes = P.nnodes;
    sv.depth = depth;
    sv.rb = kRB;
    sv.num_items_a = P.num_a;
    sv.num_items_b = P.num_d + P.num_r;
    sv.grid = std::min(sms * std::min(occ, kCtasPerSm), P.num_a + P.num_d + P.num_r);
    if (const char* g = getenv("HODLR_B200_GRID")) sv.grid = std::min(sv.grid, atoi(g));
    {
        const char* e = getenv("HODLR_SV_SPLIT");
        // opt-in: measured slower (cfg2 41.8 -> 49.0 us, cfg5 eps=1e-2 76.5 -> 84.2 us):
        // launch 2's CTAs cannot start before launch 1's leave the SMs, and the
        // grid-completion wait costs more than the in-kernel publication
        sv.split = e ? atoi(e) != 0 : 0;
        sv.launches = sv.split ? 2 : 1;
    }
    if (getenv("HODLR_B200_VERBOSE"))
        fprintf(stderr, "[hodlr_b200] fused path: grid %d (sms %d occ %d) smem %zu items A %d BC %d R %d U pieces %d\n",
                sv.grid, sms, occ, smem, P.num_a, P.num_d, P.num_r, P.nupieces);
    sv.tfast_count = tb;
    sv.extra_ws = sv_sync_bytes(P.nleaves) + (size_t)(pb + tb) * 8;  // (leaf counters unused now)
    sv.part_count = pb;
    sv.leaf_fmt = lf;
    // every CTA parks at most kFifo - 2 deferred U pieces before it must see
    // the R pieces: with fewer CTAs than pos_r / (kFifo - 2) the R pieces could
    // sit behind full FIFOs forever, so pos_r follows the final grid
    P.pos_r = std::min(P.pos_r, sv.grid * (kFifo - 2));
    sv.params = new SvParams(P);
    *ok = true;
    return HODLR_OK;
}

void SVG(sv_set_grid)(SvPlan& sv, int grid) {
    sv.grid = std::max(1, std::min(sv.grid, grid));
    SvParams& P = *reinterpret_cast<SvParams*>(sv.params);
    P.pos_r = std::min(P.pos_r, sv.grid * (kFifo - 2));
}

void SVG(sv_release)(SvPlan& sv) {
    if (sv.dev) cudaFree(sv.dev);
    delete reinterpret_cast<SvParams*>(sv.params);
    sv = SvPlan{};
}

template <typename W>
cudaError_t SVG(sv_matvec)(const PlanView& p, const SvPlan& sv, const W* x, W* b, W* partial, W* tbuf_unused,
                      void* extra, cudaStream_t st) {
    (void)p;
    (void)tbuf_unused;
    const SvParams& P = *reinterpret_cast<const SvParams*>(sv.params);
    if (((uintptr_t)x & 15) || ((uintptr_t)b & 15) || ((uintptr_t)partial & 15))
        return cudaErrorMisalignedAddress;
    SvKernelArgs<W> a;
    a.slab = sv.slab;
    a.x = x;
    a.b = b;
    (void)partial;
    uint8_t* e = (uint8_t*)extra;
    a.sync = (SvSync*)e;
    a.partial = (W*)(e + sv_sync_bytes(P.nleaves));
    a.tbuf = (W*)(e + sv_sync_bytes(P.nleaves) + sv.part_count * 8);
    a.trace = nullptr;
#ifdef HODLR_TRACE
    static unsigned long long* trace_buf = nullptr;
    static int trace_cap = 0;
    if (trace_cap < sv.grid) {
        if (trace_buf) cudaFree(trace_buf);
        cudaMalloc(&trace_buf, (size_t)sv.grid * 48 * 8);
        trace_cap = sv.grid;
    }
    cudaMemsetAsync(trace_buf, 0, (size_t)sv.grid * 48 * 8, st);
    a.trace = trace_buf;
#endif
    cudaError_t err;
    if (!sv.split) {
        void* args[] = {(void*)&P, &a};
        err = cudaLaunchKernel((const void*)k_stream<W>, dim3(sv.grid), dim3(kThreads), args, smem_bytes(), st);
    } else {
        // Split: launch 1 streams the phase-A items only (its completion publishes
        // the partials, no GPU-scope fences under load); launch 2 (programmatic
        // dependent launch: its CTAs start as launch 1's retire) streams D and U
        // and reduces the partials into coefficients after griddepcontrol.wait.
        static thread_local SvParams P1, P2;
        P1 = P;
        P1.num_d = P1.num_r = P1.pos_r = 0;
        P1.mode = 1;
        P2 = P;
        P2.num_a = 0;
        P2.mode = 2;
        SvKernelArgs<W> a2 = a;
        a2.sync = a.sync + 1;
        void* args1[] = {(void*)&P1, &a};
        err = cudaLaunchKernel((const void*)k_stream<W>, dim3(std::min(sv.grid, P.num_a)), dim3(kThreads), args1,
                               smem_bytes(), st);
        if (err == cudaSuccess) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(std::min(sv.grid, P.num_d + P.num_r));
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = smem_bytes();
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            void* args2[] = {(void*)&P2, &a2};
            err = cudaLaunchKernelExC(&cfg, (const void*)k_stream<W>, args2);
        }
    }
#ifdef HODLR_TRACE
    if (err == cudaSuccess) {
        std::vector<unsigned long long> h((size_t)sv.grid * 48);
        cudaStreamSynchronize(st);
        cudaMemcpy(h.data(), trace_buf, h.size() * 8, cudaMemcpyDeviceToHost);
        if (const char* f = getenv("HODLR_B200_TRACE_FILE")) {
            if (FILE* fp = fopen(f, "wb")) {
                int hdr[4] = {sv.grid, 48, P.num_a, P.num_r};
                fwrite(hdr, sizeof(hdr), 1, fp);
                fwrite(h.data(), 8, h.size(), fp);
                fclose(fp);
            }
        }
    }
#endif
    return err;
}

template cudaError_t SVG(sv_matvec)<double>(const PlanView&, const SvPlan&, const double*, double*, double*, double*,
                                       void*, cudaStream_t);
template cudaError_t SVG(sv_matvec)<float>(const PlanView&, const SvPlan&, const float*, float*, float*, float*, void*,
                                      cudaStream_t);

#if HODLR_SV_GEO == 0
// ------------------------------------------------------------ dispatch on SvPlan::geo
hodlr_status sv_prepare_g1(const SvInput& in, SvPlan& sv, bool* ok);
void sv_set_grid_g1(SvPlan& sv, int grid);
void sv_release_g1(SvPlan& sv);
template <typename W>
cudaError_t sv_matvec_g1(const PlanView& p, const SvPlan& sv, const W* x, W* b, W* partial, W* tbuf, void* extra,
                         cudaStream_t st);

hodlr_status sv_prepare(const SvInput& in, SvPlan& sv, bool* ok) {
    if (in.geo == 1) {
        hodlr_status st = sv_prepare_g1(in, sv, ok);
        if (st != HODLR_OK || *ok) return st;
        sv_release_g1(sv);  // the shape does not fit that geometry: the default one may
    }
    return sv_prepare_g0(in, sv, ok);
}
void sv_set_grid(SvPlan& sv, int grid) { sv.geo == 1 ? sv_set_grid_g1(sv, grid) : sv_set_grid_g0(sv, grid); }
void sv_release(SvPlan& sv) { sv.geo == 1 ? sv_release_g1(sv) : sv_release_g0(sv); }
size_t sv_extra_ws(const SvPlan& sv, int64_t) { return sv.extra_ws; }
int sv_launches(const SvPlan& sv) { return sv.launches; }
template <typename W>
cudaError_t sv_matvec(const PlanView& p, const SvPlan& sv, const W* x, W* b, W* partial, W* tbuf, void* extra,
                      cudaStream_t st) {
    return sv.geo == 1 ? sv_matvec_g1<W>(p, sv, x, b, partial, tbuf, extra, st)
                       : sv_matvec_g0<W>(p, sv, x, b, partial, tbuf, extra, st);
}
template cudaError_t sv_matvec<double>(const PlanView&, const SvPlan&, const double*, double*, double*, double*,
                                       void*, cudaStream_t);
template cudaError_t sv_matvec<float>(const PlanView&, const SvPlan&, const float*, float*, float*, float*, void*,
                                      cudaStream_t);
#endif

}  // namespace hodlr
