// Single-vector (s = 1) streaming fast path: ONE persistent kernel per matvec.
//
// Layout ("leaf slab", built from the quantised level-batched arena at create
// time): leaf L owns one contiguous region
//     [ V' columns of every level restricted to the leaf's M rows,
//       grouped by storage format (q52, bf16, fp16, fp32, fp64), column-major ]
//     [ U rows of every level, grouped by format, row-major (M x ncols_g) ]
//     [ dense leaf D, M x M row-major, working format ]
// so every unit of work is a handful of contiguous byte ranges.
//
// Kernel: 1 producer warp + 8 consumer warps per CTA, one CTA per SM
// (cooperative launch), a ring of kNS shared-memory stages guarded by
// mbarriers.  The producer pulls work items from one global atomic queue and
// streams them with cp.async.bulk (TMA bulk copies, complete_tx on the stage's
// "full" mbarrier); consumers compute from shared memory and release the stage.
//   item < A        phase A (leaf L): pieces of <= kStage bytes of V' columns
//                   (+ x_L): partial V'^T x per column -> partial buffer.  After
//                   the last piece the CTA bumps the counters of the leaf's l
//                   ancestor nodes; the last leaf of a node reduces the node's
//                   partials in leaf order (deterministic) into t and publishes
//                   the node flag (release).
//   item >= A       phase B (leaf L, RBI rows): D pieces first (y = D x, written
//                   to b), then a U piece once the t of every ancestor level is
//                   published: the producer bulk-copies the l coefficient
//                   vectors next to the U rows; consumers form
//                   b = U t + y  (rows disjoint -> no atomics on b).
// U pieces wait in a small producer-side FIFO while their flags are not yet
// set, so the level-1 grid-wide dependency of Alg. 3 never idles the memory
// pipe: D pieces of later items keep streaming.  All phase-A items precede all
// phase-B items in the queue and never wait, so progress is guaranteed with all
// CTAs co-resident.  Per-call state (queue, counters, flags, epoch) lives in
// the zero-initialised workspace; the last CTA resets it and bumps the epoch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "sv.h"

namespace hodlr {

namespace {

constexpr int kM = 256;                 // leaf rows
constexpr int kNS = 3;                  // ring stages per CTA
constexpr int kCtasPerSm = 2;           // independent pipelines per SM
constexpr int kStage = 34 * 1024;       // bytes per stage
constexpr int kConsumers = 8;           // consumer warps
constexpr int kReducers = 2;            // reducer warps (phase-A node reductions)
constexpr int kThreads = 32 * (kConsumers + 1 + kReducers);  // + producer + reducers
constexpr int kDList = 64;              // D items per CTA between completion publishes
constexpr int kEvQ = 16;                // pending phase-A completion events
constexpr int kZeroSlot = 4;            // zero coefficients for padded U columns
constexpr int kMaxLev = 24;
constexpr int kMaxPieces = 32;          // phase-A pieces per leaf
constexpr int kXB = kM * 8;             // bytes reserved for x_L in a stage

enum { PT_A = 1, PT_D = 2, PT_U = 3, PT_END = 4 };

#ifdef HODLR_PROFILE
// per-CTA cycle accounting (debug build only): [0] producer empty-wait, [1] producer
// fifo-block, [2] consumer full-wait, [3..5] consumer busy A/D/U, [6] kernel total
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(i, dt) if (lane == 0) atomicAdd((unsigned long long*)&prof[i], (unsigned long long)(dt))
#else
#define PROF_T(v)
#define PROF_ADD(i, dt)
#endif

struct Level {
    int32_t r, fmt;
    int32_t col;        // first column of this level inside its format group
    int32_t slot;       // coefficient slot (elements) inside a U piece
    int64_t pbase;      // partial buffer base of the level's nodes
    int64_t tbase;      // coefficient buffer base
    int32_t tstride;    // padded coefficients per node (multiple of 4)
    int32_t pad;
};

struct APiece {
    int32_t g, col, ncols, pad;
};

struct SvParams {
    int32_t depth, nleaves, nnodes;
    int32_t rbi, rbd, dpieces, napieces;
    int32_t num_a, num_d, num_u;
    int32_t leaf_fmt;
    int64_t slab_bytes, us_off, d_off;
    int32_t gcols[5];              // columns per format group (V' slab)
    int32_t gpad[5];               // U slab row length per group, padded to 4 columns
    int32_t gstart_pad[5];         // first padded U column of each group
    int32_t ucols_total;
    int32_t tpr_shift;             // log2(threads per U row)
    int32_t ubytes[2];             // U-piece transaction bytes for fp32 / fp64 working
    int32_t uy_off[2];             // offset of the staged y rows inside a U piece
    int64_t vgoff[5], ugoff[5];    // byte offsets of the groups inside the V' / U slabs
    int32_t coef_elems;            // padded coefficient elements per U piece
    Level lev[kMaxLev];
    APiece ap[kMaxPieces];
    int8_t col_level[512];         // flattened (group, column) -> level (0-based)
    int16_t col_c[512];            //                            -> rank column
    int16_t gstart[6];
    int16_t ucidx[512];            // padded U column -> coefficient slot (zero slot for padding)
};

struct SvSync {
    unsigned epoch, queue, done, published;  // published: nodes whose t exists (this call)
    unsigned leaves_done, pad[3];            // leaves whose D results are all in b
};

struct PieceHdr {
    int32_t type, leaf, r0, rows, slot, pad0, pad1, pad2;
    int32_t g, col, ncols, last;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
}
__device__ __forceinline__ void reducer_sync() {
    asm volatile("bar.sync 2, %0;" ::"n"(kReducers * 32) : "memory");
}

__host__ __device__ __forceinline__ int fmt_sz(int f) {
    return f == HODLR_FMT_Q52 ? 1 : f == HODLR_FMT_FP32 ? 4 : f == HODLR_FMT_FP64 ? 8 : 2;
}

// ---------------------------------------------------------------- decode + dot
template <int FMT, typename W>
__device__ __forceinline__ W dot_word(uint32_t w, const W* xs, W acc) {
    if constexpr (FMT == HODLR_FMT_FP32) {
        acc = fma((W)__uint_as_float(w), xs[0], acc);
    } else if constexpr (FMT == HODLR_FMT_BF16) {
        acc = fma((W)__uint_as_float(w << 16), xs[0], acc);
        acc = fma((W)__uint_as_float(w & 0xffff0000u), xs[1], acc);
    } else if constexpr (FMT == HODLR_FMT_FP16) {
        __half2_raw r;
        r.x = (unsigned short)(w & 0xffff);
        r.y = (unsigned short)(w >> 16);
        float2 f = __half22float2(__half2(r));
        acc = fma((W)f.x, xs[0], acc);
        acc = fma((W)f.y, xs[1], acc);
    } else {  // q52 = e5m2: byte b is the binary16 with bits b << 8
        __half2_raw lo, hi;
        lo.x = (unsigned short)((w << 8) & 0xff00);
        lo.y = (unsigned short)(w & 0xff00);
        hi.x = (unsigned short)((w >> 8) & 0xff00);
        hi.y = (unsigned short)((w >> 16) & 0xff00);
        float2 a = __half22float2(__half2(lo)), c = __half22float2(__half2(hi));
        acc = fma((W)a.x, xs[0], acc);
        acc = fma((W)a.y, xs[1], acc);
        acc = fma((W)c.x, xs[2], acc);
        acc = fma((W)c.y, xs[3], acc);
    }
    return acc;
}

template <typename W>
__device__ __forceinline__ W dot_f64(uint32_t lo, uint32_t hi, W xv, W acc) {
    const double d = __hiloint2double((int)hi, (int)lo);
    if constexpr (sizeof(W) == 8) return fma(d, xv, acc);
    else return acc + __double2float_rn(d * (double)xv);
}

// 16 bytes of format FMT (E = 16/size values) dotted with xs[0..E).
template <int FMT, typename W>
__device__ __forceinline__ W dot16(const uint4& v, const W* xs, W acc) {
    if constexpr (FMT == HODLR_FMT_FP64) {
        acc = dot_f64<W>(v.x, v.y, xs[0], acc);
        acc = dot_f64<W>(v.z, v.w, xs[1], acc);
    } else {
        constexpr int PW = FMT == HODLR_FMT_FP32 ? 1 : FMT == HODLR_FMT_Q52 ? 4 : 2;
        acc = dot_word<FMT, W>(v.x, xs + 0 * PW, acc);
        acc = dot_word<FMT, W>(v.y, xs + 1 * PW, acc);
        acc = dot_word<FMT, W>(v.z, xs + 2 * PW, acc);
        acc = dot_word<FMT, W>(v.w, xs + 3 * PW, acc);
    }
    return acc;
}

template <int FMT>
struct FmtInfo {
    static constexpr int bytes =
        FMT == HODLR_FMT_Q52 ? 1 : FMT == HODLR_FMT_FP32 ? 4 : FMT == HODLR_FMT_FP64 ? 8 : 2;
    static constexpr int E = 16 / bytes;  // values per 16-byte vector
    static constexpr int NV = kM / E;     // vectors per M-row column
    static constexpr int PER = NV >= 32 ? NV / 32 : 1;
};

// Phase A: warp-cooperative dot products of `ncols` M-row columns (shared
// memory) with the stage's x; lane owns the 16-byte vectors lane + 32 i.
template <int FMT, typename W>
__device__ __forceinline__ void a_piece_cols(const uint8_t* cols, int ncols, const W* xs, int warp, int lane,
                                             const SvParams& P, int leaf, int g, int col0, W* partial) {
    using F = FmtInfo<FMT>;
    const bool active = F::NV >= 32 || lane < F::NV;
    W xr[F::PER][F::E];
#pragma unroll
    for (int i = 0; i < F::PER; ++i)
#pragma unroll
        for (int e = 0; e < F::E; ++e) xr[i][e] = active ? xs[(lane + 32 * i) * F::E + e] : W(0);
    for (int j = warp; j < ncols; j += 2 * kConsumers) {
        const int j2 = j + kConsumers;
        const bool two = j2 < ncols;
        const uint8_t* col = cols + (size_t)j * kM * F::bytes;
        const uint8_t* col2 = cols + (size_t)(two ? j2 : j) * kM * F::bytes;
        W acc = W(0), acc2 = W(0);
        if (active) {
            uint4 v[F::PER], v2[F::PER];
#pragma unroll
            for (int i = 0; i < F::PER; ++i) {
                v[i] = *reinterpret_cast<const uint4*>(col + (lane + 32 * i) * 16);
                v2[i] = *reinterpret_cast<const uint4*>(col2 + (lane + 32 * i) * 16);
            }
#pragma unroll
            for (int i = 0; i < F::PER; ++i) {
                acc = dot16<FMT, W>(v[i], xr[i], acc);
                acc2 = dot16<FMT, W>(v2[i], xr[i], acc2);
            }
        }
        // transposed reduction: lanes 0-15 finish column j, lanes 16-31 column j2
        const bool hi = lane & 16;
        W v = hi ? acc2 : acc;
        v += __shfl_xor_sync(0xffffffffu, hi ? acc : acc2, 16);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((lane & 15) == 0 && (!hi || two)) {
            const int jj = hi ? j2 : j;
            const int flat = P.gstart[g] + col0 + jj;
            const int k = P.col_level[flat];
            const int c = P.col_c[flat];
            const Level& L = P.lev[k];
            const int sh = P.depth - (k + 1);
            const int jn = leaf >> sh;
            const int nch = 1 << sh;
            partial[L.pbase + ((int64_t)jn * L.r + c) * nch + (leaf - (jn << sh))] = v;
        }
    }
}

template <typename W>
__device__ __forceinline__ void a_piece(int fmt, const uint8_t* cols, int ncols, const W* xs, int warp, int lane,
                                        const SvParams& P, int leaf, int col0, W* partial) {
    switch (fmt) {
        case HODLR_FMT_FP64: a_piece_cols<HODLR_FMT_FP64, W>(cols, ncols, xs, warp, lane, P, leaf, fmt, col0, partial); break;
        case HODLR_FMT_FP32: a_piece_cols<HODLR_FMT_FP32, W>(cols, ncols, xs, warp, lane, P, leaf, fmt, col0, partial); break;
        case HODLR_FMT_FP16: a_piece_cols<HODLR_FMT_FP16, W>(cols, ncols, xs, warp, lane, P, leaf, fmt, col0, partial); break;
        case HODLR_FMT_BF16: a_piece_cols<HODLR_FMT_BF16, W>(cols, ncols, xs, warp, lane, P, leaf, fmt, col0, partial); break;
        default: a_piece_cols<HODLR_FMT_Q52, W>(cols, ncols, xs, warp, lane, P, leaf, fmt, col0, partial); break;
    }
}

// Phase B, leaf part: y = D[rows] x_L (rows of M values, format FMT) -> b.
template <int FMT, typename W>
__device__ __forceinline__ void d_piece(const uint8_t* drows, int rows, const W* xs, int warp, int lane, W* b) {
    using F = FmtInfo<FMT>;
    W xr[F::PER][F::E];
#pragma unroll
    for (int i = 0; i < F::PER; ++i)
#pragma unroll
        for (int e = 0; e < F::E; ++e) xr[i][e] = xs[(lane + 32 * i) * F::E + e];
    for (int r = warp; r < rows; r += 2 * kConsumers) {
        const int r2 = r + kConsumers;
        const bool two = r2 < rows;
        const uint8_t* row = drows + (size_t)r * kM * F::bytes;
        const uint8_t* row2 = drows + (size_t)(two ? r2 : r) * kM * F::bytes;
        uint4 v[F::PER], v2[F::PER];
#pragma unroll
        for (int i = 0; i < F::PER; ++i) {
            v[i] = *reinterpret_cast<const uint4*>(row + (lane + 32 * i) * 16);
            v2[i] = *reinterpret_cast<const uint4*>(row2 + (lane + 32 * i) * 16);
        }
        W acc = W(0), acc2 = W(0);
#pragma unroll
        for (int i = 0; i < F::PER; ++i) {
            acc = dot16<FMT, W>(v[i], xr[i], acc);
            acc2 = dot16<FMT, W>(v2[i], xr[i], acc2);
        }
        const bool hi = lane & 16;
        W s = hi ? acc2 : acc;
        s += __shfl_xor_sync(0xffffffffu, hi ? acc : acc2, 16);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) b[r] = s;
        if (lane == 16 && two) b[r2] = s;
    }
}

template <typename W>
__device__ __forceinline__ W u_elem(int fmt, const uint8_t* p, int idx) {
    switch (fmt) {
        case HODLR_FMT_FP64: return (W)reinterpret_cast<const double*>(p)[idx];
        case HODLR_FMT_FP32: return (W)reinterpret_cast<const float*>(p)[idx];
        case HODLR_FMT_FP16: return (W)dec_fp16(reinterpret_cast<const uint16_t*>(p)[idx]);
        case HODLR_FMT_BF16: return (W)dec_bf16(reinterpret_cast<const uint16_t*>(p)[idx]);
        default: return (W)dec_q52(p[idx]);
    }
}

// U piece: 4 consecutive columns j..j+3 of one row (format g, padded row) times
// their coefficients (slot indices packed 4 x int16 in one 8-byte word).
template <typename W>
__device__ __forceinline__ W u_dot4(int g, const uint8_t* ub, int j, const int16_t* ci, const W* coef, W acc) {
    const uint2 iw = *reinterpret_cast<const uint2*>(ci + j);
    const int i0 = (int)(int16_t)(iw.x & 0xffff), i1 = (int)(int16_t)(iw.x >> 16);
    const int i2 = (int)(int16_t)(iw.y & 0xffff), i3 = (int)(int16_t)(iw.y >> 16);
    W u0, u1, u2, u3;
    switch (g) {
        case HODLR_FMT_FP64: {
            const double4 v = *reinterpret_cast<const double4*>(ub + (size_t)j * 8);
            u0 = (W)v.x; u1 = (W)v.y; u2 = (W)v.z; u3 = (W)v.w;
            break;
        }
        case HODLR_FMT_FP32: {
            const float4 v = *reinterpret_cast<const float4*>(ub + (size_t)j * 4);
            u0 = (W)v.x; u1 = (W)v.y; u2 = (W)v.z; u3 = (W)v.w;
            break;
        }
        case HODLR_FMT_FP16: {
            const uint2 v = *reinterpret_cast<const uint2*>(ub + (size_t)j * 2);
            u0 = (W)dec_fp16(v.x & 0xffff); u1 = (W)dec_fp16(v.x >> 16);
            u2 = (W)dec_fp16(v.y & 0xffff); u3 = (W)dec_fp16(v.y >> 16);
            break;
        }
        case HODLR_FMT_BF16: {
            const uint2 v = *reinterpret_cast<const uint2*>(ub + (size_t)j * 2);
            u0 = (W)__uint_as_float(v.x << 16); u1 = (W)__uint_as_float(v.x & 0xffff0000u);
            u2 = (W)__uint_as_float(v.y << 16); u3 = (W)__uint_as_float(v.y & 0xffff0000u);
            break;
        }
        default: {
            const uint32_t v = *reinterpret_cast<const uint32_t*>(ub + j);
            u0 = (W)dec_q52(v & 0xff); u1 = (W)dec_q52((v >> 8) & 0xff);
            u2 = (W)dec_q52((v >> 16) & 0xff); u3 = (W)dec_q52(v >> 24);
            break;
        }
    }
    acc = fma(u0, coef[i0], acc);
    acc = fma(u1, coef[i1], acc);
    acc = fma(u2, coef[i2], acc);
    acc = fma(u3, coef[i3], acc);
    return acc;
}

template <typename W>
struct SvKernelArgs {
    const uint8_t* slab;
    const uint8_t* zeros;  // 32 zero bytes (coefficient of padded U columns)
    const W* x;
    W* b;
    W* partial;
    W* tbuf;
    SvSync* sync;
    unsigned* counters;    // [nnodes]: leaves counted into each node (last arriver reduces)
    unsigned* dcount;      // [nleaves]: consumer-warp arrivals of the leaf's D pieces
};

// shared-memory bookkeeping next to the stage ring
struct SmemCtl {
    uint64_t full[kNS], empty[kNS];
    PieceHdr hdr[kNS];
    unsigned epoch;
    volatile int ev_tail;          // phase-A completion events pushed by the producer
    volatile int ev_head;          // ... and retired by the reducer warps
    int ev_leaf[kEvQ];
    unsigned ev_done[kEvQ];        // consumer warps finished with the event's leaf
    int last_mask;
    unsigned d_done;               // consumer-warp completions of this CTA's D pieces
    int dlist[kDList];             // leaves of D items emitted but not yet published (FIFO)
    unsigned dend[kDList];         // ... and the cumulative D-piece count at their end
    alignas(16) int16_t cidx[512];  // U column (padded groups) -> coefficient slot
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
    const int nq = P.num_d + P.num_u;  // dynamic queue: D items, then U items
    const unsigned d_expect = (unsigned)(kM / P.rbi);  // D items per leaf

    if (threadIdx.x == 0) {
        C.epoch = ld_acquire(&a.sync->epoch);
        C.ev_tail = 0;
        C.ev_head = 0;
        C.d_done = 0u;
        for (int s = 0; s < kNS; ++s) {
            mbar_init(&C.full[s], 1);
            mbar_init(&C.empty[s], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < kEvQ; i += kThreads) C.ev_done[i] = 0u;
    for (int i = threadIdx.x; i < P.ucols_total; i += kThreads) C.cidx[i] = P.ucidx[i];
    __syncthreads();
    const unsigned target = C.epoch + 1u;

    if (warp == 0) {
        // =========================================================== producer
        int stage = 0;
        unsigned phase = 0;
        int ev = 0;  // phase-A events pushed
        auto next_stage = [&]() {
            if (++stage == kNS) {
                stage = 0;
                phase ^= 1u;
            }
        };
        auto push_event = [&](int leaf) {  // lane 0
            while (ev - C.ev_head >= kEvQ) __nanosleep(64);
            C.ev_leaf[ev % kEvQ] = leaf;
            __threadfence_block();
            C.ev_tail = ev + 1;
        };
        bool coef_ready = false;
        int dh = 0, dt = 0;        // D-item FIFO head / tail (warp-uniform)
        unsigned d_pieces = 0;     // D pieces emitted by this CTA
        // Publish, in order, every listed D item whose pieces this CTA's consumers
        // have finished (their b stores are ordered by the CTA-scope release on
        // C.d_done): one GPU-scope release per item.  block: wait for all.
        auto publish_d = [&](bool block) {
            while (dh != dt) {
                int n = 0;
                if (lane == 0) {
                    const unsigned done = *(volatile unsigned*)&C.d_done;
                    while (dh + n != dt && done >= C.dend[(dh + n) % kDList] * kConsumers) ++n;
                    if (n) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
                n = __shfl_sync(0xffffffffu, n, 0);
                for (int i = lane; i < n; i += 32)
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.dcount + C.dlist[(dh + i) % kDList])
                                 : "memory");
                dh += n;
                __syncwarp();
                if (!block || dh == dt) return;
                if (n == 0) __nanosleep(64);
            }
        };
        auto claim = [&]() -> uint8_t* {
            PROF_T(t0);
            while (!mbar_test(&C.empty[stage], phase ^ 1u)) publish_d(false);
            PROF_ADD(0, clock64() - t0);
            return stages + (size_t)stage * kStage;
        };

        // ---- phase A: leaves dealt round-robin, every CTA starts with its share
        for (int leaf = blockIdx.x; leaf < P.num_a; leaf += gridDim.x) {
            const uint8_t* base = a.slab + (int64_t)leaf * P.slab_bytes;
            if (lane == 0) push_event(leaf);
            ++ev;
            __syncwarp();
            for (int p = 0; p < P.napieces; ++p) {
                const APiece ap = P.ap[p];
                uint8_t* st = claim();
                const unsigned cb = (unsigned)(ap.ncols * kM * fmt_sz(ap.g));
                if (lane == 0) {
                    PieceHdr& h = C.hdr[stage];
                    h.type = PT_A;
                    h.leaf = leaf;
                    h.g = ap.g;
                    h.col = ap.col;
                    h.ncols = ap.ncols;
                    h.last = (p == P.napieces - 1);
                    mbar_arrive_tx(&C.full[stage], (unsigned)(kM * sizeof(W)) + cb);
                    bulk_g2s(st, a.x + (int64_t)leaf * kM, (unsigned)(kM * sizeof(W)), &C.full[stage]);
                    bulk_g2s(st + kXB, base + P.vgoff[ap.g] + (int64_t)ap.col * kM * fmt_sz(ap.g), cb, &C.full[stage]);
                }
                __syncwarp();
                next_stage();
            }
        }
        // ---- phases B (D items) and C (U items) from one atomic queue, two ahead
        int n1 = 0, n2 = 0;
        if (lane == 0) {
            n1 = (int)atomicAdd(&a.sync->queue, 1u);
            n2 = (int)atomicAdd(&a.sync->queue, 1u);
        }
        const int per_leaf = kM / P.rbi;
        for (;;) {
            const int q = __shfl_sync(0xffffffffu, n1, 0);
            if (q >= nq) break;
            n1 = n2;
            if (lane == 0) n2 = (int)atomicAdd(&a.sync->queue, 1u);
            if (q < P.num_d) {
                const int leaf = q / per_leaf;
                const int r0 = (q % per_leaf) * P.rbi;
                const uint8_t* dbase = a.slab + (int64_t)leaf * P.slab_bytes + P.d_off;
                const int dsz = fmt_sz(P.leaf_fmt);
                if (dt - dh == kDList) publish_d(true);
                d_pieces += (unsigned)P.dpieces;
                if (lane == 0) {
                    C.dlist[dt % kDList] = leaf;
                    C.dend[dt % kDList] = d_pieces;
                }
                __syncwarp();
                ++dt;
                for (int p = 0; p < P.dpieces; ++p) {
                    uint8_t* st = claim();
                    const int rr = r0 + p * P.rbd;
                    const unsigned cb = (unsigned)(P.rbd * kM * dsz);
                    if (lane == 0) {
                        PieceHdr& h = C.hdr[stage];
                        h.type = PT_D;
                        h.leaf = leaf;
                        h.r0 = rr;
                        h.rows = P.rbd;
                        mbar_arrive_tx(&C.full[stage], (unsigned)(kM * sizeof(W)) + cb);
                        bulk_g2s(st, a.x + (int64_t)leaf * kM, (unsigned)(kM * sizeof(W)), &C.full[stage]);
                        bulk_g2s(st + kXB, dbase + (int64_t)rr * kM * dsz, cb, &C.full[stage]);
                    }
                    __syncwarp();
                    next_stage();
                }
            } else {
                const int u = q - P.num_d;
                const int leaf = u / per_leaf;
                const int r0 = (u % per_leaf) * P.rbi;
                // the coefficients of every node, and this leaf's D results, must exist
                publish_d(true);  // own D items first (another CTA's U item may wait on them)
                PROF_T(tr0);
                if (!coef_ready) {
                    unsigned pub = 0;
                    if (lane == 0)
                        while ((pub = ld_acquire(&a.sync->published)) != (unsigned)P.nnodes) __nanosleep(128);
                    coef_ready = true;
                }
                if (lane == 0)
                    while (ld_acquire(&a.dcount[leaf]) != d_expect) __nanosleep(64);
                PROF_ADD(6, clock64() - tr0);
                __syncwarp();
                uint8_t* st = claim();
                const int wbytes = (int)sizeof(W);
                const int coef_bytes = P.coef_elems * wbytes;
                const int yoff = P.uy_off[sizeof(W) == 8 ? 1 : 0];
                if (lane == 0) {
                    PieceHdr& h = C.hdr[stage];
                    h.type = PT_U;
                    h.leaf = leaf;
                    h.r0 = r0;
                    h.rows = P.rbi;
                    mbar_arrive_tx(&C.full[stage], (unsigned)P.ubytes[sizeof(W) == 8 ? 1 : 0]);
                }
                __syncwarp();
                // coefficients and y were written by other SMs (generic proxy, made
                // visible by the acquires above); order them before the async-proxy reads
                asm volatile("fence.proxy.async.global;" ::: "memory");
                if (lane < nlev) {
                    const Level& L = P.lev[lane];
                    if (L.r > 0) {
                        const int k = lane + 1;
                        const int jsib = (leaf >> (nlev - k)) ^ 1;
                        const W* src = a.tbuf + L.tbase + (int64_t)jsib * L.tstride;
                        bulk_g2s(st + (size_t)L.slot * wbytes, src, (unsigned)(L.tstride * wbytes), &C.full[stage]);
                    }
                } else if (lane >= 24 && lane < 29) {
                    const int g = lane - 24;
                    if (P.gpad[g] > 0) {
                        const uint8_t* src = a.slab + (int64_t)leaf * P.slab_bytes + P.us_off + P.ugoff[g] +
                                             (int64_t)r0 * P.gpad[g] * fmt_sz(g);
                        int off = coef_bytes + kZeroSlot * wbytes;
                        for (int g2 = 0; g2 < g; ++g2) off += P.rbi * P.gpad[g2] * fmt_sz(g2);
                        bulk_g2s(st + off, src, (unsigned)(P.rbi * P.gpad[g] * fmt_sz(g)), &C.full[stage]);
                    }
                } else if (lane == 30) {
                    bulk_g2s(st + yoff, a.b + (int64_t)leaf * kM + r0, (unsigned)(P.rbi * wbytes), &C.full[stage]);
                } else if (lane == 31) {
                    bulk_g2s(st + coef_bytes, a.zeros, (unsigned)(kZeroSlot * wbytes), &C.full[stage]);
                }
                __syncwarp();
                next_stage();
            }
        }
        publish_d(true);
        claim();
#ifdef HODLR_PROFILE
        if (lane == 0) prof[1] = clock64() - t_kernel;
#endif
        if (lane == 0) {
            C.hdr[stage].type = PT_END;
            mbar_arrive(&C.full[stage]);
            while (ev - C.ev_head >= kEvQ) __nanosleep(64);
            C.ev_leaf[ev % kEvQ] = -1;  // reducers: done
            __threadfence_block();
            C.ev_tail = ev + 1;
        }
        __syncwarp();
    } else if (warp <= kReducers) {
        // =========================================================== reducers
        // Retire phase-A events in order: once all consumer warps finished the
        // leaf's partials, bump the counters of its l ancestor nodes; for every
        // node whose last leaf this was, reduce the node's partials in leaf order
        // (fixed thread mapping -> deterministic) into t and count it published.
        const int rt = threadIdx.x - 32;  // 0 .. 32*kReducers-1
        for (int ev = 0;; ++ev) {
            if (rt == 0)
                while (C.ev_tail <= ev) __nanosleep(256);
            reducer_sync();
            const int leaf = C.ev_leaf[ev % kEvQ];
            if (leaf < 0) break;
            if (rt == 0)
                while (*(volatile unsigned*)&C.ev_done[ev % kEvQ] < (unsigned)kConsumers) __nanosleep(64);
            if (warp == 1) {
                if (lane == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                __syncwarp();
                bool last = false;
                if (lane < nlev) {
                    const int k = lane + 1;
                    const int sh = nlev - k;
                    const int id = (1 << k) - 2 + (leaf >> sh);
                    unsigned old;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.counters + id) : "memory");
                    last = old == (1u << sh) - 1u;
                }
                const unsigned m = __ballot_sync(0xffffffffu, last);
                if (lane == 0) C.last_mask = (int)m;
            }
            reducer_sync();
            unsigned mask = (unsigned)C.last_mask;
            int published = 0;
            while (mask) {
                const int lv = __ffs(mask) - 1;
                mask &= mask - 1;
                const int k = lv + 1;
                const int sh = nlev - k;
                const int jn = leaf >> sh;
                const int nch = 1 << sh;
                const Level& L = P.lev[lv];
                if (L.r > 0) {
                    int tpc = 32;  // threads per column (power of two, divides 32)
                    while (tpc > 1 && tpc * L.r > 32 * kReducers) tpc >>= 1;
                    const int cpr = 32 * kReducers / tpc;  // columns per round
                    for (int c0 = 0; c0 < L.r; c0 += cpr) {
                        const int c = c0 + rt / tpc, sl = rt % tpc;
                        W acc = W(0);
                        if (c < L.r) {
                            const W* src = a.partial + L.pbase + ((int64_t)jn * L.r + c) * nch;
                            constexpr int B = 8;  // loads in flight per thread
                            for (int i0 = sl; i0 < nch; i0 += B * tpc) {
                                W v[B];
#pragma unroll
                                for (int u = 0; u < B; ++u) {
                                    const int i = i0 + u * tpc;
                                    v[u] = i < nch ? __ldcg(src + i) : W(0);
                                }
#pragma unroll
                                for (int u = 0; u < B; ++u) acc += v[u];
                            }
                        }
                        for (int o = tpc >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                        if (sl == 0 && c < L.r) a.tbuf[L.tbase + (int64_t)jn * L.tstride + c] = acc;
                    }
                }
                if (rt == 0) a.counters[(1 << k) - 2 + jn] = 0u;
                ++published;
            }
            reducer_sync();
            if (rt == 0) {
                if (published)
                    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&a.sync->published), "r"(published)
                                 : "memory");
                C.ev_done[ev % kEvQ] = 0u;
                __threadfence_block();
                C.ev_head = ev + 1;
            }
        }
    } else {
        // =========================================================== consumers
        const int cw = warp - 1 - kReducers;
        const int ctid = threadIdx.x - 32 * (1 + kReducers);
        int stage = 0;
        unsigned phase = 0;
        int ev = 0;
        for (;;) {
            PROF_T(tw);
            mbar_wait(&C.full[stage], phase);
            PROF_T(tb);
            PROF_ADD(2, tb - tw);
            const PieceHdr h = C.hdr[stage];
            const uint8_t* st = stages + (size_t)stage * kStage;
            if (h.type == PT_END) {
#ifdef HODLR_PROFILE
                if (ctid == 0) prof[7] = clock64() - t_kernel;
#endif
                break;
            }
            if (h.type == PT_A) {
                a_piece<W>(h.g, st + kXB, h.ncols, reinterpret_cast<const W*>(st), cw, lane, P, h.leaf, h.col,
                           a.partial);
            } else if (h.type == PT_D) {
                W* brow = a.b + (int64_t)h.leaf * kM + h.r0;
                const W* xs = reinterpret_cast<const W*>(st);
                if (P.leaf_fmt == HODLR_FMT_FP64) d_piece<HODLR_FMT_FP64, W>(st + kXB, h.rows, xs, cw, lane, brow);
                else d_piece<HODLR_FMT_FP32, W>(st + kXB, h.rows, xs, cw, lane, brow);
            } else {  // PT_U: b = U t + y (y = D x, staged from b)
                const int row = ctid >> P.tpr_shift, q = ctid & ((1 << P.tpr_shift) - 1);
                const W* coef = reinterpret_cast<const W*>(st);
                const W* ys = reinterpret_cast<const W*>(st + P.uy_off[sizeof(W) == 8 ? 1 : 0]);
                W acc = W(0);
                int off = (P.coef_elems + kZeroSlot) * (int)sizeof(W);
                for (int g = 0; g < 5; ++g) {
                    const int nc = P.gpad[g];
                    if (nc == 0) continue;
                    const uint8_t* ub = st + off + (size_t)row * nc * fmt_sz(g);
                    const int16_t* ci = C.cidx + P.gstart_pad[g];
                    for (int j = 4 * q; j < nc; j += 4 << P.tpr_shift) acc = u_dot4<W>(g, ub, j, ci, coef, acc);
                    off += h.rows * nc * fmt_sz(g);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
                    if (o < (1 << P.tpr_shift)) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (q == 0) a.b[(int64_t)h.leaf * kM + h.r0 + row] = acc + ys[row];  // levels, then leaf
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&C.empty[stage]);
            PROF_ADD(2 + h.type, clock64() - tb);
            if (h.type == PT_A && h.last) {
                // this warp's partials of the leaf are written: tell the reducers
                if (lane == 0) {
                    asm volatile("fence.acq_rel.cta;" ::: "memory");
                    atomicAdd(&C.ev_done[ev % kEvQ], 1u);
                }
                ++ev;
            } else if (h.type == PT_D && lane == 0) {
                // this warp's rows of y are in b (ordered by the __syncwarp above):
                // CTA-scope release; the producer publishes GPU-wide per D item
                asm volatile("fence.acq_rel.cta;" ::: "memory");
                atomicAdd(&C.d_done, 1u);
            }
            if (++stage == kNS) {
                stage = 0;
                phase ^= 1u;
            }
        }
    }
    // ---- teardown: the last CTA resets the per-call state and bumps the epoch
    __syncthreads();
#ifdef HODLR_PROFILE
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 101 || blockIdx.x == 250))
        printf("PROF cta %d: total %lld END_emitted %lld END_seen %lld prod_empty %lld wait_ready %lld | cons_wait %lld busyA %lld busyD %lld busyU %lld (consumer sums over %d warps)\n",
               blockIdx.x, clock64() - t_kernel, prof[1], prof[7], prof[0], prof[6], prof[2], prof[3], prof[4], prof[5], kConsumers);
#endif
    __shared__ unsigned s_last;
    if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&a.sync->done) : "memory");
        s_last = old == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        for (int i = threadIdx.x; i < P.nleaves; i += kThreads) a.dcount[i] = 0u;
        __syncthreads();
        if (threadIdx.x == 0) {
            a.sync->queue = 0u;
            a.sync->done = 0u;
            a.sync->published = 0u;
            a.sync->leaves_done = 0u;
            __threadfence();
            st_release(&a.sync->epoch, target);
        }
    }
}

size_t smem_bytes() { return (size_t)kNS * kStage + sizeof(SmemCtl); }

// workspace head: SvSync, node counters, leaf D counters (zeroed once, reset per call)
size_t sv_sync_bytes(int nnodes, int nleaves) {
    return (sizeof(SvSync) + ((size_t)nnodes + nleaves) * sizeof(unsigned) + 255) / 256 * 256;
}

}  // namespace

// ============================================================== host side
hodlr_status sv_prepare(const SvInput& in, SvPlan& sv, bool* ok) {
    sv = SvPlan{};
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
        for (int j = 0; j < (1 << k); ++j) {
            const NodeDesc& nd = nodes[base + j];
            if (nd.level != k || nd.ext_slot >= 0 || nd.rv != n0.rv || nd.ru != n0.rv || nd.u_fmt != n0.u_fmt ||
                nd.v_fmt != n0.u_fmt || nd.nchunk != (1 << (depth - k)) || nd.row0 != j * (kM << (depth - k)) ||
                nd.part_off != n0.part_off + (int64_t)j * n0.rv * n0.nchunk)
                return HODLR_OK;
        }
        P.lev[k - 1].r = n0.rv;
        P.lev[k - 1].fmt = n0.u_fmt;
    }
    // column lists per format group (level-major inside a group)
    int flat = 0;
    for (int g = 0; g < 5; ++g) {
        P.gstart[g] = (int16_t)flat;
        int cnt = 0;
        for (int k = 0; k < depth; ++k) {
            if (P.lev[k].fmt != g) continue;
            P.lev[k].col = cnt;
            for (int c = 0; c < P.lev[k].r; ++c) {
                if (flat >= 512) return HODLR_OK;
                P.col_level[flat] = (int8_t)k;
                P.col_c[flat] = (int16_t)c;
                ++flat;
                ++cnt;
            }
        }
        P.gcols[g] = cnt;
    }
    P.gstart[5] = (int16_t)flat;
    // coefficient slots and partial / coefficient buffers
    int slot = 0;
    int64_t tb = 0;
    for (int k = 0; k < depth; ++k) {
        Level& L = P.lev[k];
        L.tstride = (L.r + 3) / 4 * 4;
        L.slot = slot;
        slot += L.tstride;
        L.pbase = nodes[(1 << (k + 1)) - 2].part_off;
        L.tbase = tb;
        tb += (int64_t)L.tstride << (k + 1);
    }
    P.coef_elems = slot;
    // slab geometry (U rows padded to 4-column groups; padding -> zero coefficient)
    int64_t vs = 0, us = 0;
    int upad = 0;
    for (int g = 0; g < 5; ++g) {
        P.vgoff[g] = vs;
        vs += (int64_t)P.gcols[g] * kM * fmt_bytes(g);
        P.gpad[g] = (P.gcols[g] + 3) / 4 * 4;
        P.gstart_pad[g] = upad;
        for (int j = 0; j < P.gpad[g]; ++j) {
            if (upad + j >= 512) return HODLR_OK;
            if (j < P.gcols[g]) {
                const int f = P.gstart[g] + j;
                P.ucidx[upad + j] = (int16_t)(P.lev[P.col_level[f]].slot + P.col_c[f]);
            } else {
                P.ucidx[upad + j] = (int16_t)P.coef_elems;  // zero slot
            }
        }
        upad += P.gpad[g];
        P.ugoff[g] = us;
        us += (int64_t)P.gpad[g] * kM * fmt_bytes(g);
    }
    P.ucols_total = upad;
    const int dsz = fmt_bytes(lf);
    P.us_off = vs;
    P.d_off = vs + us;
    P.slab_bytes = vs + us + (int64_t)kM * kM * dsz;
    // phase-B geometry: D pieces of rbd rows, items / U pieces of rbi rows
    P.rbd = 1;
    while (P.rbd * 2 <= kM && kXB + P.rbd * 2 * kM * dsz <= kStage) P.rbd *= 2;
    int ubytes_row = 0;
    for (int g = 0; g < 5; ++g) ubytes_row += P.gpad[g] * fmt_bytes(g);
    const int cfix = (P.coef_elems + kZeroSlot) * 8;
    P.rbi = 32;
    const int min_rbi = kConsumers;  // U-piece reduction: <= 32 threads per row
    while (P.rbi > min_rbi && cfix + P.rbi * (ubytes_row + 8) > kStage) P.rbi /= 2;
    if (cfix + P.rbi * (ubytes_row + 8) > kStage) return HODLR_OK;
    P.tpr_shift = 0;
    while ((1 << P.tpr_shift) * P.rbi < kConsumers * 32) ++P.tpr_shift;
    if ((1 << P.tpr_shift) * P.rbi != kConsumers * 32 || P.tpr_shift > 5) return HODLR_OK;
    for (int wi = 0; wi < 2; ++wi) {
        const int wb = wi ? 8 : 4;
        P.uy_off[wi] = (P.coef_elems + kZeroSlot) * wb + P.rbi * ubytes_row;  // 16-B multiple
        P.ubytes[wi] = P.uy_off[wi] + P.rbi * wb;
    }
    if (P.rbd > P.rbi) P.rbd = P.rbi;
    if (P.rbi % P.rbd) return HODLR_OK;
    for (int g = 0; g < 5; ++g)  // bulk copies: 16-byte granules
        if ((P.rbi * P.gpad[g] * fmt_bytes(g)) % 16) return HODLR_OK;
    P.dpieces = P.rbi / P.rbd;
    // phase-A pieces
    P.napieces = 0;
    for (int g = 0; g < 5; ++g) {
        const int cpp = (kStage - kXB) / (kM * fmt_bytes(g));
        for (int c = 0; c < P.gcols[g]; c += cpp) {
            if (P.napieces == kMaxPieces) return HODLR_OK;
            P.ap[P.napieces++] = APiece{g, c, std::min(cpp, P.gcols[g] - c), 0};
        }
    }
    if (P.napieces == 0) return HODLR_OK;  // all ranks zero: generic path
    P.num_a = nleaves;
    P.num_d = nleaves * (kM / P.rbi);
    P.num_u = nleaves * (kM / P.rbi);

    // ---- relayout the quantised level-batched arena into leaf slabs (bytes)
    std::vector<uint8_t> arena(in.arena_bytes);
    if (cudaMemcpy(arena.data(), in.d_arena, in.arena_bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        return HODLR_OK;
    std::vector<uint8_t> slab((size_t)P.slab_bytes * nleaves);
    for (int leaf = 0; leaf < nleaves; ++leaf) {
        uint8_t* out = slab.data() + (size_t)leaf * P.slab_bytes;
        for (int g = 0; g < 5; ++g) {
            const int w = fmt_bytes(g);
            int col = 0;
            for (int k = 0; k < depth; ++k) {
                if (P.lev[k].fmt != g) continue;
                const int lvl = k + 1;
                const NodeDesc& nd = nodes[(1 << lvl) - 2 + (leaf >> (depth - lvl))];
                const int64_t roff = (int64_t)leaf * kM - nd.row0;
                for (int c = 0; c < nd.rv; ++c, ++col) {
                    memcpy(out + P.vgoff[g] + (int64_t)col * kM * w,
                           arena.data() + nd.v_off + ((int64_t)c * nd.v_ld + roff) * w, (size_t)kM * w);
                    const uint8_t* src = arena.data() + nd.u_off + ((int64_t)c * nd.u_ld + roff) * w;
                    uint8_t* dst = out + P.us_off + P.ugoff[g] + (int64_t)col * w;
                    for (int r = 0; r < kM; ++r)
                        memcpy(dst + (int64_t)r * P.gpad[g] * w, src + (int64_t)r * w, (size_t)w);
                }
            }
        }
        memcpy(out + P.d_off, arena.data() + leaves[leaf].off, (size_t)kM * kM * dsz);
    }
    int dev = 0, sms = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    const size_t smem = smem_bytes();
    if (!coop || sms <= 0 ||
        cudaFuncSetAttribute(k_stream<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(k_stream<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return HODLR_OK;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<double>, kThreads, smem);
    if (occ < 1) return HODLR_OK;
    void* d = nullptr;
    slab.resize(slab.size() + 256, 0);  // + zero coefficients for padded U columns
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
    sv.rb = P.rbi;
    sv.num_items_a = P.num_a;
    sv.num_items_b = P.num_d + P.num_u;
    sv.grid = std::min(sms * std::min(occ, kCtasPerSm), P.num_a + P.num_d + P.num_u);
    sv.launches = 1;
    sv.tfast_count = tb;
    sv.extra_ws = sv_sync_bytes(P.nnodes, P.nleaves) + (size_t)tb * 8;
    sv.leaf_fmt = lf;
    sv.params = new SvParams(P);
    *ok = true;
    return HODLR_OK;
}

void sv_release(SvPlan& sv) {
    if (sv.dev) cudaFree(sv.dev);
    delete reinterpret_cast<SvParams*>(sv.params);
    sv = SvPlan{};
}
size_t sv_extra_ws(const SvPlan& sv, int64_t) { return sv.extra_ws; }
int sv_launches(const SvPlan& sv) { return sv.launches; }

template <typename W>
cudaError_t sv_matvec(const PlanView& p, const SvPlan& sv, const W* x, W* b, W* partial, W* tbuf_unused,
                      void* extra, cudaStream_t st) {
    (void)p;
    (void)tbuf_unused;
    const SvParams& P = *reinterpret_cast<const SvParams*>(sv.params);
    if (((uintptr_t)x & 15) || ((uintptr_t)b & 15) || ((uintptr_t)partial & 15))
        return cudaErrorMisalignedAddress;
    SvKernelArgs<W> a;
    a.slab = sv.slab;
    a.zeros = sv.slab + sv.dev_bytes - 256;
    a.x = x;
    a.b = b;
    a.partial = partial;
    uint8_t* e = (uint8_t*)extra;
    a.sync = (SvSync*)e;
    a.counters = (unsigned*)(e + sizeof(SvSync));
    a.dcount = a.counters + P.nnodes;
    const size_t toff = sv_sync_bytes(P.nnodes, P.nleaves);
    a.tbuf = (W*)(e + toff);
    void* args[] = {(void*)&P, &a};
    return cudaLaunchCooperativeKernel((const void*)k_stream<W>, dim3(sv.grid), dim3(kThreads), args,
                                       smem_bytes(), st);
}

template cudaError_t sv_matvec<double>(const PlanView&, const SvPlan&, const double*, double*, double*, double*,
                                       void*, cudaStream_t);
template cudaError_t sv_matvec<float>(const PlanView&, const SvPlan&, const float*, float*, float*, float*, void*,
                                      cudaStream_t);

}  // namespace hodlr
