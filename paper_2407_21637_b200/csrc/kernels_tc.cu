// Multi-RHS phase B on the 5th-generation tensor cores (tcgen05, kind::tf32),
// fp32 working precision.  Layout and item order: tcb.h.
//
// Per leaf (256 rows) and pass of up to 64 right-hand sides:
//     b[rows, q0:q0+N] = sum over items of A_item (256 x c) * B_item (c x N)
// A_item = leaf columns (D) or one level's U columns, streamed once from HBM;
// B_item = the matching rows of X (D items) or of the coefficients T_k of the
// sibling node (U items), staged from global memory (L2).
//
// 3xTF32: every fp32 operand a = hi + lo (both tf32, tc::split_tf32), and
//     acc += A_hi B_hi + A_hi B_lo + A_lo B_hi
// which keeps fp32-level accuracy (the dropped A_lo B_lo and the tf32
// roundings are O(2^-22) relative).  Storage formats narrower than fp32 (fp16,
// bf16, q52) are exact tf32 values: A_lo = 0 and the third product is skipped.
// Accumulation is fp32 in tensor memory.
//
// Warp roles (one CTA per SM, persistent over (leaf, column block) work units):
//   warps 0-15  converters: warp w owns m-tile (w/4)%2 (leaf rows 128*m ..), TMEM lane
//               quarter w%4 and column half w/8 of the item; thread = one leaf row.
//               Per item: warp 0 polls the item's two mbarriers (raw bytes landed, A stage
//               free), the other 15 wait at a hardware barrier (no polling instructions);
//               then four 16-byte loads, split, two tcgen05.st.x16 (hi, lo) into the item's
//               TMEM A stage.  They also run the epilogue of the previous leaf (tcgen05.ld
//               of the accumulator, b written once: disjoint rows, no atomics), deferred by
//               one item so it overlaps the next leaf's first MMAs.
//   warp 16     producer: lane 0 moves the A item (one cp.async.bulk into a 4-slot ring) and
//               does every mbarrier wait of the warp; the B source rows (X or T, fp32) of
//               the item go as one bulk copy (contiguous rows) or one row per lane into a
//               second 4-slot ring.  A per-leaf table holds every item's source pointer.
//   warp 17     MMA issuer (whole warp in uniform control flow, the tcgen05.mma / commit
//               predicated on one elected lane: tc::mma_tf32_ts_u) and TMEM owner.
//   warps 18-25 B stagers: source rows (shared memory) -> tf32 hi/lo in the K-major
//               no-swizzle canonical layout (core matrix = 8 columns x 4 k), 3-slot ring;
//               warp 18 polls, the others wait at a hardware barrier.  Operands that are
//               not 16-byte aligned take the register-staged path (loads from global).
// TMEM columns: accumulator [2 m-tiles][64] at 0..127, A stages [3][2 m-tiles][hi 32 | lo 32]
// at 128..511.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

#include "async.cuh"
#include "formats.cuh"
#include "mrhs.h"
#include "tc.cuh"

namespace hodlr {
namespace {

// Build with -DHODLR_TC_TRACE for per-item clock traces of CTA 0 (printf at exit).
#ifdef HODLR_TC_TRACE
#define TC_TRACE_DECL long long tra[48] = {}, trb[48] = {}, trc[48] = {}, trw[48] = {};
#define TC_TR(arr, cond) if ((cond) && blockIdx.x == 0 && g < 48) arr[g] = clock64();
#define TC_TRACE_DUMP(role, lead) \
    if (blockIdx.x == 0 && (lead)) \
        for (int i_ = 0; i_ < 48; ++i_) \
            printf("TRACE role %d item %d a %lld b %lld c %lld w %lld\n", role, i_, tra[i_], trb[i_], trc[i_], trw[i_]);
#else
#define TC_TRACE_DECL
#define TC_TR(arr, cond)
#define TC_TRACE_DUMP(role, lead)
#endif

// Build with -DHODLR_TC_PROGRESS: lane 0 of every warp of CTA 0 of k_tc_a publishes (item << 8 | step)
// to host-mapped memory; a host thread prints the table 3 s after the launch (who is stuck where).
#ifdef HODLR_TC_PROGRESS
__device__ volatile int* g_progress = nullptr;
#define TC_PROG(step) if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && g_progress) g_progress[threadIdx.x >> 5] = (int)(pg << 8) | (step);
#else
#define TC_PROG(step)
#endif

constexpr int kTcConvWarps = 16;   // warp w: m-tile (w>>2)&1, lane quarter w&3, column half w>>3
constexpr int kTcProdWarp = 16;
constexpr int kTcMmaWarp = 17;
constexpr int kTcStageWarp0 = 18;
constexpr int kTcStageWarps = 8;   // thread t: right-hand side t % 64, column quads t / 64 and t / 64 + 4
constexpr int kTcThreads = (kTcStageWarp0 + kTcStageWarps) * 32;
constexpr int kTcRawStages = 4;
constexpr int kTcRawSlot = kTcRows * kTcItemCols * 4;  // 32 KB
constexpr int kTcAStages = 3;
constexpr int kTcBStages = 3;
constexpr int kTcBHalf = kTcItemCols * kTcN * 4;       // 8 KB: hi (or lo) of one item
constexpr int kTcBSlot = 2 * kTcBHalf;
constexpr uint32_t kTcAcc = 0, kTcAStage = 128;        // accumulator [2 m-tiles][64]; A stages [3][2][hi 32 | lo 32]
constexpr int kChunkRowsTa = 256;  // rows of a phase-A chunk (= leaf)
constexpr int kTcBRawSlots = 4;                   // B source rows (fp32) in flight, filled by the producer's bulk copies
constexpr int kTcBars = 2 * kTcRawStages + 2 * kTcAStages + 2 * kTcBStages + 2 + 2 * kTcBRawSlots;
constexpr int kTcBRawSlot = kTcItemCols * kTcN * 4;  // 8 KB: the fp32 source rows of one item
struct BSrc {  // source rows of one item's B operand (X or T), first right-hand side of the pass
    const float* p;
    int32_t ld, nvalid;
};
constexpr size_t kTcSmem = (size_t)kTcRawStages * kTcRawSlot + (size_t)kTcBStages * kTcBSlot +
                           (size_t)kTcBRawSlots * kTcBRawSlot + kTcBars * 8 + 2 * kTcMaxItems * sizeof(BSrc) +
                           2 * 2 * kMrMaxLevels * 8 + 16;

__device__ __forceinline__ float4 load_quad(int fmt, const uint8_t* p) {
    switch (fmt) {
        case HODLR_FMT_FP32:
            return *reinterpret_cast<const float4*>(p);
        case HODLR_FMT_FP16: {
            const uint2 u = *reinterpret_cast<const uint2*>(p);
            return make_float4(dec_fp16((uint16_t)(u.x & 0xFFFF)), dec_fp16((uint16_t)(u.x >> 16)),
                               dec_fp16((uint16_t)(u.y & 0xFFFF)), dec_fp16((uint16_t)(u.y >> 16)));
        }
        case HODLR_FMT_BF16: {
            const uint2 u = *reinterpret_cast<const uint2*>(p);
            return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                               __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
        }
        default: {  // q52
            const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
            return make_float4(dec_q52((uint8_t)(u & 0xFF)), dec_q52((uint8_t)((u >> 8) & 0xFF)),
                               dec_q52((uint8_t)((u >> 16) & 0xFF)), dec_q52((uint8_t)(u >> 24)));
        }
    }
}

__global__ void __launch_bounds__(kTcThreads, 1)
    k_tc_b(PlanView p, const __grid_constant__ TcView v, const float* __restrict__ x, int64_t ldx,
           const float* __restrict__ tbuf, float* __restrict__ b, int64_t ldb, int64_t s, int nblk, int dbg) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint8_t* ring = smem_raw;                                              // [4][32 KB]
    uint8_t* bring = ring + (size_t)kTcRawStages * kTcRawSlot;             // [3][hi 8 KB | lo 8 KB]
    float* rawb = reinterpret_cast<float*>(bring + (size_t)kTcBStages * kTcBSlot);  // [4][32 rows][64] fp32 source rows
    uint64_t* bars = reinterpret_cast<uint64_t*>(rawb + (size_t)kTcBRawSlots * (kTcBRawSlot / 4));
    uint64_t* raw_full = bars;
    uint64_t* raw_empty = raw_full + kTcRawStages;
    uint64_t* a_full = raw_empty + kTcRawStages;
    uint64_t* a_empty = a_full + kTcAStages;
    uint64_t* b_full = a_empty + kTcAStages;
    uint64_t* b_empty = b_full + kTcBStages;
    uint64_t* acc_full = b_empty + kTcBStages;
    uint64_t* acc_empty = acc_full + 1;
    uint64_t* braw_full = acc_empty + 1;
    uint64_t* braw_empty = braw_full + kTcBRawSlots;
    // per-leaf B source rows of every item (aligned path) / node table (register-staged path),
    // both double-buffered by leaf parity
    BSrc* btab = reinterpret_cast<BSrc*>(braw_empty + kTcBRawSlots);
    int64_t* ntab_off = reinterpret_cast<int64_t*>(btab + 2 * kTcMaxItems);
    int32_t* ntab_ru = reinterpret_cast<int32_t*>(ntab_off + 2 * kMrMaxLevels);
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(ntab_ru + 2 * kMrMaxLevels);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwork = p.nchunks * nblk;
    const int nitems = v.nitems;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kTcRawStages; ++i) {
            tma::mbar_init(&raw_full[i], 1);
            tma::mbar_init(&raw_empty[i], kTcConvWarps);
        }
        for (int i = 0; i < kTcAStages; ++i) {
            tma::mbar_init(&a_full[i], kTcConvWarps);
            tma::mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < kTcBStages; ++i) {
            tma::mbar_init(&b_full[i], kTcStageWarps);
            tma::mbar_init(&b_empty[i], 1);
        }
        tma::mbar_init(acc_full, 1);
        tma::mbar_init(acc_empty, kTcConvWarps);
        for (int i = 0; i < kTcBRawSlots; ++i) {
            tma::mbar_init(&braw_full[i], 1);
            tma::mbar_init(&braw_empty[i], kTcStageWarps);
        }
        tma::fence_mbar_init();
    }
    if (warp == kTcMmaWarp) tc::tmem_alloc<512>(tbase_s);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tbase_s;
    TC_TRACE_DECL
    // Aligned fp32 operands: the producer warp bulk-copies every item's B source rows (X or
    // T) into a 4-slot ring ahead of the stagers, so no L2 latency and no address work sits
    // on the stagers' per-item chain.  Otherwise the stagers load through registers.
    const bool bfast = ((ldx | s) & 3) == 0 && ldx <= 0x7fffffff && s <= 0x7fffffff &&
                       ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(tbuf)) & 15) == 0 && !(dbg & 16);

    if (warp < kTcConvWarps) {
        // ---------------------------------------------------------- converters + epilogue
        const int mt = (warp >> 2) & 1, qd = warp & 3, half = warp >> 3;
        const int row = mt * 128 + qd * 32 + lane;
        const uint32_t tl = tbase + ((uint32_t)(qd * 32) << 16);
        int64_t g = 0;
        int lc = 0;
        int pend_chunk = -1, pend_q0 = 0;
        // epilogue of the lc-th leaf: this warp's 32 accumulator columns -> b
        auto epilogue = [&](int chunk, int q0) {
            tma::mbar_wait_sleep(acc_full, (unsigned)(lc & 1));
            tc::fence_after();
            const int64_t r = p.chunks[chunk].row0 + row;
            float* brow = b + r * ldb + q0;
            const bool vec = ((ldb & 3) == 0) && ((reinterpret_cast<uintptr_t>(b) & 15) == 0);
#pragma unroll
            for (int c = half * 32; c < half * 32 + 32; c += 16) {
                if (q0 + c >= s) break;  // warp-uniform
                uint32_t a[16];
                tc::ld_x16(tl + kTcAcc + mt * 64 + c, a);
                tc::wait_ld();
                if (vec && q0 + c + 16 <= s) {
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<float4*>(brow + c + j) =
                            make_float4(__uint_as_float(a[j]), __uint_as_float(a[j + 1]),
                                        __uint_as_float(a[j + 2]), __uint_as_float(a[j + 3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (q0 + c + j < s) brow[c + j] = __uint_as_float(a[j]);
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(acc_empty);
            ++lc;
        };
        // Ring positions as counters (no 64-bit division per item).  Only converter warp 0
        // polls the item's two mbarriers; the other 15 warps wait at a hardware barrier, so
        // their waiting takes no issue slots from the warps that are working.
        int rs = 0, ts = 0;
        unsigned rpar = 0, apar = 0;
        bool a_first = true;
        const bool fin = v.finite != 0;
        const uint8_t* rrow = ring + (size_t)row * 16;
        for (int work = blockIdx.x; work < nwork; work += gridDim.x) {
            const int chunk = work / nblk;
            const int q0 = (work % nblk) * kTcN;
            for (int i = 0; i < nitems; ++i, ++g) {
                const TcItem it = v.item[i];
                if (warp == 0) {
                    tma::mbar_wait_sleep(&raw_full[rs], rpar);
                    TC_TR(tra, lane == 0)
                    if (!a_first) tma::mbar_wait_sleep(&a_empty[ts], apar);
                    TC_TR(trb, lane == 0)
                }
                asm volatile("bar.sync 2, %0;" ::"n"(32 * kTcConvWarps) : "memory");
                tc::fence_after();
                TC_TR(trc, warp == 0 && lane == 0)
                const uint32_t ah = tl + kTcAStage + ts * 128 + mt * 64;
                if (it.fmt == HODLR_FMT_FP32 && it.ncols == kTcItemCols && !(dbg & 4)) {
                    // full fp32 item: this thread's 16 columns = 4 column quads, one 16-byte load each
                    const uint8_t* rp = rrow + (size_t)rs * kTcRawSlot + (size_t)half * 4 * (kTcRows * 16);
                    float f[16];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float4 u = *reinterpret_cast<const float4*>(rp + (size_t)q * (kTcRows * 16));
                        f[4 * q] = u.x, f[4 * q + 1] = u.y, f[4 * q + 2] = u.z, f[4 * q + 3] = u.w;
                    }
                    uint32_t hi[16], lo[16];
                    if (fin) {
#pragma unroll
                        for (int e = 0; e < 16; ++e) tc::split_tf32_fast(f[e], hi[e], lo[e]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) tc::split_tf32(f[e], hi[e], lo[e]);
                    }
                    tc::st_x16(ah + half * 16, hi);
                    tc::st_x16(ah + 32 + half * 16, lo);
                } else {
                    const int w = fmt_bytes(it.fmt);
                    const uint8_t* rp = ring + (size_t)rs * kTcRawSlot + (size_t)row * 4 * w;
                    const bool full = it.fmt == HODLR_FMT_FP32;
                    const int j0 = half * 16, j1 = min((int)it.ncols, j0 + 16);
                    for (int j = j0; j < j1; j += 8) {
                        float4 f0 = make_float4(0.f, 0.f, 0.f, 0.f), f1 = f0;
                        if (!(dbg & 4)) {
                            f0 = load_quad(it.fmt, rp + (size_t)(j >> 2) * kTcRows * 4 * w);
                            f1 = load_quad(it.fmt, rp + (size_t)((j >> 2) + 1) * kTcRows * 4 * w);
                        }
                        const float f[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
                        uint32_t hi[8], lo[8];
                        if (full) {
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                if (fin)
                                    tc::split_tf32_fast(f[e], hi[e], lo[e]);
                                else
                                    tc::split_tf32(f[e], hi[e], lo[e]);
                            }
                            tc::st_x8(ah + j, hi);
                            tc::st_x8(ah + 32 + j, lo);
                        } else {
#pragma unroll
                            for (int e = 0; e < 8; ++e) hi[e] = __float_as_uint(f[e]);
                            tc::st_x8(ah + j, hi);
                        }
                    }
                }
                TC_TR(trw, warp == 0 && lane == 0)
                tc::wait_st();
                tc::fence_before();
                __syncwarp();
                if (lane == 0) {
                    tma::mbar_arrive(&raw_empty[rs]);
                    tma::mbar_arrive(&a_full[ts]);
                }
                if (++rs == kTcRawStages) rs = 0, rpar ^= 1u;
                if (++ts == kTcAStages) {
                    ts = 0;
                    if (a_first) a_first = false; else apar ^= 1u;
                }
                if (i == 0 && pend_chunk >= 0) {
                    epilogue(pend_chunk, pend_q0);
                    pend_chunk = -1;
                }
            }
            pend_chunk = chunk;
            pend_q0 = q0;
        }
        if (pend_chunk >= 0) epilogue(pend_chunk, pend_q0);
    } else if (warp == kTcProdWarp) {
        // ---------------------------------------------------------- producer
        // (whole warp: lane 0 moves the A item; the B source rows go row by row, one lane each,
        // or as one copy when the rows are contiguous)
        const uint64_t pol = tma::policy_evict_first();
        int rs = 0, bslot = 0, lc = 0;
        [[maybe_unused]] int64_t g = 0;
        unsigned rpar = 1, bpar = 1;  // parity of the *_empty waits from the second pass on
        bool r_first = true, b_first = true;
        for (int work = blockIdx.x; work < nwork; work += gridDim.x, ++lc) {
            const int chunk = work / nblk;
            const int q0 = (work % nblk) * kTcN;
            const uint8_t* src = v.slab + (int64_t)chunk * v.leaf_bytes;
            BSrc* tab = btab + (lc & 1) * kTcMaxItems;
            const unsigned rowbytes = (unsigned)min((int64_t)kTcN, s - q0) * 4u;
            if (bfast) {
                // per leaf: the source rows of every item (one dependent node lookup per item, once)
                const int64_t row0 = p.chunks[chunk].row0;
                for (int t = lane; t < nitems; t += 32) {
                    const TcItem it = v.item[t];
                    BSrc e;
                    if (it.lv < 0) {  // rows [col0, col0 + ncols) of X (leaf rows)
                        e.p = x + (row0 + it.col0) * ldx + q0;
                        e.ld = (int32_t)ldx;
                        e.nvalid = it.ncols;
                    } else {          // ... or of T of the sibling node
                        const NodeDesc& nd = p.nodes[p.chunk_nodes[(int64_t)chunk * p.nlev + it.lv]];
                        e.p = tbuf + (nd.tsrc_off + it.col0) * s + q0;
                        e.ld = (int32_t)s;
                        e.nvalid = max(0, min((int)it.ncols, nd.ru - it.col0));
                    }
                    tab[t] = e;
                }
                __syncwarp();
            }
            for (int i = 0; i < nitems; ++i, ++g) {
                if (lane == 0) {
                    if (!r_first) tma::mbar_wait_sleep(&raw_empty[rs], rpar ^ 1u);
                    TC_TR(trw, true)
                    const int bytes = v.item[i].bytes;
                    tma::mbar_arrive_tx(&raw_full[rs], (unsigned)bytes);
                    tma::bulk_g2s(ring + (size_t)rs * kTcRawSlot, src + v.item[i].off, (unsigned)bytes, &raw_full[rs],
                                  pol);
                }
                if (++rs == kTcRawStages) {
                    rs = 0;
                    if (r_first) r_first = false; else rpar ^= 1u;
                }
                if (bfast) {
                    // (lane 0 does every mbarrier wait of this warp: the other lanes block at the
                    // __syncwarp below instead of spinning on a divergent path next to lane 0's)
                    const BSrc e = tab[i];
                    const int nv = (dbg & 8) ? 0 : e.nvalid;
                    float* dst = rawb + (size_t)bslot * (kTcBRawSlot / 4);
                    const bool one = (unsigned)e.ld * 4u == rowbytes && rowbytes == kTcN * 4;
                    if (lane == 0) {
                        if (!b_first) tma::mbar_wait_sleep(&braw_empty[bslot], bpar ^ 1u);
                        tma::mbar_arrive_tx(&braw_full[bslot], (unsigned)nv * rowbytes);
                    }
                    __syncwarp();
                    if (one) {
                        if (lane == 0 && nv > 0)
                            tma::bulk_g2s_plain(dst, e.p, (unsigned)nv * rowbytes, &braw_full[bslot]);
                    } else if (lane < nv) {
                        tma::bulk_g2s_plain(dst + lane * kTcN, e.p + (int64_t)lane * e.ld, rowbytes, &braw_full[bslot]);
                    }
                    if (++bslot == kTcBRawSlots) {
                        bslot = 0;
                        if (b_first) b_first = false; else bpar ^= 1u;
                    }
                }
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ---------------------------------------------------------- MMA issuer
        // (whole warp, uniform control flow; the MMAs and commits are predicated on one elected lane)
        const uint32_t leader = tc::elect_one();
        {
            int64_t g = 0;
            int lc = 0;
            int ts = 0, bs = 0;
            unsigned a_par = 0, b_par = 0;
            for (int work = blockIdx.x; work < nwork; work += gridDim.x, ++lc) {
                const int q0 = (work % nblk) * kTcN;
                const int nn = (int)min((int64_t)kTcN, (s - q0 + 15) / 16 * 16);
                const uint32_t idesc = tc::idesc_tf32(128, nn);
                const uint32_t lbo = (uint32_t)(nn / 8) * 128;
                if (lc >= 1) tma::mbar_wait_sleep(acc_empty, (unsigned)((lc - 1) & 1));
                for (int i = 0; i < nitems; ++i, ++g) {
                    tma::mbar_wait_sleep(&a_full[ts], a_par);
                    TC_TR(tra, true)
                    tma::mbar_wait_sleep(&b_full[bs], b_par);
                    TC_TR(trb, true)
                    tc::fence_after();
                    const int ncols = v.item[i].ncols;
                    const bool full = v.item[i].fmt == HODLR_FMT_FP32 && !(dbg & 1);
                    const uint32_t bh = tc::smem_u32(bring) + (uint32_t)bs * kTcBSlot;
                    // descriptors of the item's first k-step; a k-step (two column quads) further = + 2 lbo bytes
                    uint64_t dh = tc::smem_desc(bh, lbo, 128), dl = tc::smem_desc(bh + kTcBHalf, lbo, 128);
                    const uint64_t dstep = (uint64_t)((2 * lbo) >> 4);
                    const uint32_t d0 = tbase + kTcAcc, d1 = d0 + 64;
                    uint32_t a0 = tbase + kTcAStage + ts * 128;
                    uint32_t acc = i != 0;
                    if (!(dbg & 2)) {
#pragma unroll 1
                        for (int j = 0; j < ncols; j += 8) {
                            // the two m-tiles alternate: consecutive MMAs never accumulate into the same tile
                            tc::mma_tf32_ts_u(d0, a0, dh, idesc, acc, leader);
                            tc::mma_tf32_ts_u(d1, a0 + 64, dh, idesc, acc, leader);
                            tc::mma_tf32_ts_u(d0, a0, dl, idesc, 1, leader);
                            tc::mma_tf32_ts_u(d1, a0 + 64, dl, idesc, 1, leader);
                            if (full) {
                                tc::mma_tf32_ts_u(d0, a0 + 32, dh, idesc, 1, leader);
                                tc::mma_tf32_ts_u(d1, a0 + 96, dh, idesc, 1, leader);
                            }
                            acc = 1;
                            a0 += 8;
                            dh += dstep;
                            dl += dstep;
                        }
                    }
                    tc::commit_u(&a_empty[ts], leader);
                    tc::commit_u(&b_empty[bs], leader);
                    TC_TR(trc, true)
                    if (++ts == kTcAStages) ts = 0, a_par ^= 1u;
                    if (++bs == kTcBStages) bs = 0, b_par ^= 1u;
                }
                tc::commit_u(acc_full, leader);
            }
        }
    } else {
        // ---------------------------------------------------------- B stagers
        const int t = threadIdx.x - kTcStageWarp0 * 32;
        // Aligned operands: the source rows (X or T, fp32) of item g + 3 are copied into a
        // 4-slot shared-memory ring with cp.async while item g is split and stored, so no
        // L2 latency sits on the per-item chain.  Otherwise: register-staged loads below.
        if (bfast) {
            // thread: right-hand side n = t % 64, column quads t / 64 and t / 64 + 4.  Stager warp 0
            // polls the two mbarriers of the item; the others wait at a hardware barrier.
            const int n = t & 63, kq = t >> 6;
            int64_t g = 0;
            int bs = 0, cslot = 0, lc = 0;
            unsigned bpar = 0, cpar = 0;
            bool first_pass = true;
            for (int work = blockIdx.x; work < nwork; work += gridDim.x, ++lc) {
                const int q0 = (work % nblk) * kTcN;
                const int nn = (int)min((int64_t)kTcN, (s - q0 + 15) / 16 * 16);
                const int lbo = (nn / 8) * 128;
                const bool colok = q0 + n < s;
                const BSrc* tab = btab + (lc & 1) * kTcMaxItems;
                for (int i = 0; i < nitems; ++i, ++g) {
                    const int nkc = v.item[i].ncols >> 2;
                    if (warp == kTcStageWarp0) {
                        tma::mbar_wait_sleep(&braw_full[cslot], cpar);
                        TC_TR(trw, t == 0)
                        if (!first_pass) tma::mbar_wait_sleep(&b_empty[bs], bpar);
                        TC_TR(tra, t == 0)
                    }
                    asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcStageWarps) : "memory");
                    const int nvalid = colok ? tab[i].nvalid : 0;
                    const float* rb = rawb + (size_t)cslot * (kTcBRawSlot / 4) + n;
                    float vals[2][4];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int kc = kq + 4 * e;
#pragma unroll
                        for (int k = 0; k < 4; ++k) vals[e][k] = kc * 4 + k < nvalid ? rb[(kc * 4 + k) * kTcN] : 0.0f;
                    }
                    TC_TR(trb, t == 0)
                    uint8_t* bh = bring + (size_t)bs * kTcBSlot;
                    uint8_t* bl = bh + kTcBHalf;
                    if (n < nn) {
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int kc = kq + 4 * e;
                            if (kc >= nkc) break;
                            uint4 h, l;
                            tc::split_tf32(vals[e][0], h.x, l.x);
                            tc::split_tf32(vals[e][1], h.y, l.y);
                            tc::split_tf32(vals[e][2], h.z, l.z);
                            tc::split_tf32(vals[e][3], h.w, l.w);
                            const int off = kc * lbo + (n >> 3) * 128 + (n & 7) * 16;
                            *reinterpret_cast<uint4*>(bh + off) = h;
                            *reinterpret_cast<uint4*>(bl + off) = l;
                        }
                    }
                    tma::fence_proxy_async_smem();
                    __syncwarp();
                    TC_TR(trc, t == 0)
                    if (lane == 0) {
                        tma::mbar_arrive(&b_full[bs]);
                        tma::mbar_arrive(&braw_empty[cslot]);
                    }
                    if (++cslot == kTcBRawSlots) cslot = 0, cpar ^= 1u;
                    if (++bs == kTcBStages) {
                        bs = 0;
                        if (first_pass) first_pass = false; else bpar ^= 1u;
                    }
                }
            }
        } else {
            int64_t g = 0;
            int lc = 0;
            for (int work = blockIdx.x; work < nwork; work += gridDim.x, ++lc) {
                const int chunk = work / nblk;
                const int q0 = (work % nblk) * kTcN;
                const int nn = (int)min((int64_t)kTcN, (s - q0 + 15) / 16 * 16);
                const int64_t row0 = p.chunks[chunk].row0;
                const int lbo = (nn / 8) * 128;
                // node table of this leaf (one dependent lookup per level, not per item)
                int64_t* toff = ntab_off + (lc & 1) * kMrMaxLevels;
                int32_t* tru = ntab_ru + (lc & 1) * kMrMaxLevels;
                if (t < v.nlev) {
                    const NodeDesc& nd = p.nodes[p.chunk_nodes[(int64_t)chunk * p.nlev + t]];
                    toff[t] = nd.tsrc_off;
                    tru[t] = nd.ru;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcStageWarps) : "memory");
                // thread t: column n = t % 64, column quads kc = t / 64 + 2e (no division).  The
                // loads of item i + 1 are issued before item i is split and stored (and before
                // the wait for its slot), so one L2 latency per item leaves the critical path.
                const int n = t & 63, kq = t >> 6;
                const bool colok = n < nn && q0 + n < s && !(dbg & 8);
                auto load_item = [&](int i, float (&vals)[2][4]) {
                    const TcItem it = v.item[i];
                    const float* src;
                    int64_t ld;
                    int nvalid;
                    if (it.lv < 0) {  // source rows [col0, col0 + ncols) of X (leaf rows)
                        src = x + (row0 + it.col0) * ldx + q0;
                        ld = ldx;
                        nvalid = it.ncols;
                    } else {          // ... or of T of the sibling node
                        src = tbuf + (toff[it.lv] + it.col0) * s + q0;
                        ld = s;
                        nvalid = max(0, min((int)it.ncols, tru[it.lv] - it.col0));
                    }
                    const int nkc = it.ncols >> 2;
    #pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int kc = kq + 4 * e;
    #pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int r = kc * 4 + k;
                            vals[e][k] = (colok && kc < nkc && r < nvalid) ? __ldg(src + (int64_t)r * ld + n) : 0.0f;
                        }
                    }
                };
                float nxt[2][4];
                load_item(0, nxt);
                for (int i = 0; i < nitems; ++i, ++g) {
                    const TcItem it = v.item[i];
                    const int bs = (int)(g % kTcBStages);
                    const int nkc = it.ncols >> 2;
                    float vals[2][4];
    #pragma unroll
                    for (int e = 0; e < 2; ++e)
    #pragma unroll
                        for (int k = 0; k < 4; ++k) vals[e][k] = nxt[e][k];
                    if (i + 1 < nitems) load_item(i + 1, nxt);
                    if (g >= kTcBStages) tma::mbar_wait_sleep(&b_empty[bs], (unsigned)(((g / kTcBStages) & 1) ^ 1));
                    TC_TR(trw, t == 0)
                    uint8_t* bh = bring + (size_t)bs * kTcBSlot;
                    uint8_t* bl = bh + kTcBHalf;
                    if (n < nn) {
    #pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int kc = kq + 4 * e;
                            if (kc >= nkc) break;
                            uint4 h, l;
                            tc::split_tf32(vals[e][0], h.x, l.x);
                            tc::split_tf32(vals[e][1], h.y, l.y);
                            tc::split_tf32(vals[e][2], h.z, l.z);
                            tc::split_tf32(vals[e][3], h.w, l.w);
                            const int off = kc * lbo + (n >> 3) * 128 + (n & 7) * 16;
                            *reinterpret_cast<uint4*>(bh + off) = h;
                            *reinterpret_cast<uint4*>(bl + off) = l;
                        }
                    }
                    TC_TR(tra, t == 0)
                    tma::fence_proxy_async_smem();
                    __syncwarp();
                    TC_TR(trc, t == 0)
                    if (lane == 0) tma::mbar_arrive(&b_full[bs]);
                }
            }
    }
    }
    TC_TRACE_DUMP(warp < kTcConvWarps ? 0 : warp == kTcProdWarp ? 1 : warp == kTcMmaWarp ? 2 : 3,
                  lane == 0 && (warp == 0 || warp == kTcProdWarp || warp == kTcMmaWarp || warp == kTcStageWarp0))
    tc::fence_before();
    __syncthreads();
    if (warp == kTcMmaWarp) {
        tc::fence_after();
        tc::tmem_free<512>(tbase);
    }
}

// Create time: flag set if any 32-bit word of a slab looks like an fp32 inf/NaN
// (narrow formats can only add false positives, which just keep the guarded split).
__global__ void k_scan_nonfinite(const uint32_t* __restrict__ w, int64_t n, int* flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if ((w[i] & 0x7f800000u) == 0x7f800000u) {
            *flag = 1;
            return;
        }
}

static int slab_finite(const void* slab, size_t bytes) {
    int* d = nullptr;
    if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return 0;
    int h = 0;
    cudaMemset(d, 0, sizeof(int));
    k_scan_nonfinite<<<148 * 4, 256>>>((const uint32_t*)slab, (int64_t)(bytes / 4), d);
    if (cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) h = 1;
    cudaFree(d);
    return h == 0;
}

// Item slab relayout (create time): one thread per (chunk, item, column quad, row).
__global__ void k_tc_slab(PlanView p, const __grid_constant__ TcView v, int64_t units_per_chunk, uint8_t* slab) {
    const int64_t total = units_per_chunk * p.nchunks;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int chunk = (int)(idx / units_per_chunk);
        int64_t r = idx - (int64_t)chunk * units_per_chunk;
        int i = 0;
        for (;; ++i) {
            const int64_t c = (int64_t)(v.item[i].ncols >> 2) * kTcRows;
            if (r < c) break;
            r -= c;
        }
        const TcItem it = v.item[i];
        const int kc = (int)(r / kTcRows), row = (int)(r % kTcRows);
        const int w = fmt_bytes(it.fmt);
        uint8_t* dst = slab + (int64_t)chunk * v.leaf_bytes + it.off + ((int64_t)kc * kTcRows + row) * 4 * w;
        const ChunkDesc ch = p.chunks[chunk];
        for (int k = 0; k < 4; ++k) {
            const int col = it.col0 + 4 * kc + k;
            const uint8_t* src = nullptr;
            if (it.lv < 0) {
                const LeafDesc lf = p.leaves[ch.leaf];
                src = p.arena + lf.off + ((int64_t)row * lf.ld + col) * w;
            } else {
                const NodeDesc nd = p.nodes[p.chunk_nodes[(int64_t)chunk * p.nlev + it.lv]];
                if (col < nd.ru) src = p.arena + nd.u_off + ((int64_t)col * nd.u_ld + (ch.row0 - nd.row0 + row)) * w;
            }
            for (int e = 0; e < w; ++e) dst[k * w + e] = src ? src[e] : (uint8_t)0;
        }
    }
}


// ====================================================================== phase A
// Warp roles: 0-15 converters / epilogue (warp w: M-tile w/4, TMEM lane quarter
// w%4; thread = one stacked rank row m; warp 0 polls the item's mbarriers, the
// others wait at a hardware barrier), 16 producer (A item by lane 0, the item's
// 16 X rows by bulk copy into a 4-slot ring), 17 MMA issuer + TMEM owner, 18-21 X
// stagers (warp 18 polls).  CTA b owns chunks [b*nch/nb, (b+1)*nch/nb) (the MrView
// slot layout), per chunk D = sum over 16 items.  Cross-chunk sums of a node's
// run: see the TSUM template parameter of k_tc_a; a finished row is written to
// the coefficient buffer when this CTA holds the whole node, else to the node's
// partial slot (fixed-order reduce afterwards).
constexpr int kTaConvWarps = 4 * kTcAMaxTiles;
constexpr int kTaProdWarp = kTaConvWarps;
constexpr int kTaMmaWarp = kTaConvWarps + 1;
constexpr int kTaStageWarp0 = kTaConvWarps + 2;
constexpr int kTaStageWarps = 4;
constexpr int kTaThreads = (kTaStageWarp0 + kTaStageWarps) * 32;
constexpr int kTaMaxAStages = 3;
constexpr int kTaBStages = 4;
constexpr int kTaBHalf = kTcAItemRows * kTcN * 4;  // 4 KB
constexpr int kTaBSlot = 2 * kTaBHalf;
constexpr uint32_t kTaAcc = 0;
constexpr int kTaMaxRaw = 8;
constexpr int kTaXRawSlots = 4;                          // X source rows (fp32) in flight, filled by the producer
constexpr int kTaXRawSlot = kTcAItemRows * kTcN * 4;     // 4 KB
constexpr int kTaBars = 2 * kTaMaxRaw + 2 * kTaMaxAStages + 2 * kTaBStages + 2 + 2 * kTaXRawSlots;
// TMEM: D tiles at columns t*64, then A stages of nmt*32 columns (hi 16 | lo 16
// per tile): 3 stages for <= 3 tiles (480 columns), 2 for 4 tiles (512)
__host__ __device__ inline int ta_astages(const TcAView& a) { return a.nmt <= 3 ? 3 : 2; }

__host__ __device__ inline size_t ta_raw_slot(const TcAView& a) { return ((size_t)a.item_bytes + 127) / 128 * 128; }
// Cross-chunk running sums of the accurate variant: [stacked row][64 columns + 4 pad] fp32 in
// shared memory (the pad makes the per-thread 16-byte row accesses conflict-free)
constexpr int kTaSumLd = kTcN + 4;
__host__ __device__ inline size_t ta_sum_bytes(const TcAView& a, bool tmem_sums) {
    return tmem_sums ? 0 : (size_t)((a.mtot + 31) / 32 * 32) * kTaSumLd * 4;
}
inline size_t ta_smem(const TcAView& a, int nraw, bool tmem_sums) {
    return nraw * ta_raw_slot(a) + (size_t)kTaBStages * kTaBSlot + (size_t)kTaXRawSlots * kTaXRawSlot +
           ta_sum_bytes(a, tmem_sums) + kTaBars * 8 + 16;
}
// raw ring depth: as many item slots (<= kTaMaxRaw) as fit next to the rest
inline int ta_nraw(const TcAView& a, bool tmem_sums) {
    int n = kTaMaxRaw;
    if (const char* e = getenv("HODLR_B200_TA_NRAW")) n = std::max(2, std::min(kTaMaxRaw, atoi(e)));  // (ring-depth sweeps)
    while (n > 2 && ta_smem(a, n, tmem_sums) > 227 * 1024) --n;
    return n;
}

// TSUM = true: the accumulator stays in tensor memory across a node's chunks (fastest; the
// tensor core's truncating fp32 accumulation then runs over the whole run: error ~4x larger).
// TSUM = false (default): per-chunk accumulator, cross-chunk sums added in fp32 (round to
// nearest) by the converter warps in shared memory.
template <bool TSUM>
__global__ void __launch_bounds__(kTaThreads, 1)
    k_tc_a(PlanView p, const __grid_constant__ MrView m, const __grid_constant__ TcAView a,
           const float* __restrict__ x, int64_t ldx, int64_t s, int spad, int nblk, float* __restrict__ partial,
           float* __restrict__ tbuf, int nraw, int dbg) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const size_t rslot = ta_raw_slot(a);
    uint8_t* ring = smem_raw;
    uint8_t* bring = ring + nraw * rslot;
    float* xraw = reinterpret_cast<float*>(bring + (size_t)kTaBStages * kTaBSlot);  // [4][16 rows][64] fp32 X rows
    float* sums = xraw + (size_t)kTaXRawSlots * (kTaXRawSlot / 4);  // (TSUM = false only)
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sums) + ta_sum_bytes(a, TSUM));
    uint64_t* raw_full = bars;
    uint64_t* raw_empty = raw_full + nraw;
    uint64_t* a_full = raw_empty + nraw;
    uint64_t* a_empty = a_full + kTaMaxAStages;
    uint64_t* b_full = a_empty + kTaMaxAStages;
    uint64_t* b_empty = b_full + kTaBStages;
    uint64_t* acc_full = b_empty + kTaBStages;
    uint64_t* acc_empty = acc_full + 1;
    uint64_t* xraw_full = acc_empty + 1;
    uint64_t* xraw_empty = xraw_full + kTaXRawSlots;
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(xraw_empty + kTaXRawSlots);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c_beg = (int)((int64_t)blockIdx.x * p.nchunks / gridDim.x);
    const int c_end = (int)((int64_t)(blockIdx.x + 1) * p.nchunks / gridDim.x);
    constexpr int kItems = kChunkRowsTa / kTcAItemRows;

    if (threadIdx.x == 0) {
        for (int i = 0; i < nraw; ++i) {
            tma::mbar_init(&raw_full[i], 1);
            tma::mbar_init(&raw_empty[i], kTaConvWarps);
        }
        for (int i = 0; i < kTaMaxAStages; ++i) {
            tma::mbar_init(&a_full[i], kTaConvWarps);
            tma::mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < kTaBStages; ++i) {
            tma::mbar_init(&b_full[i], kTaStageWarps);
            tma::mbar_init(&b_empty[i], 1);
        }
        tma::mbar_init(acc_full, 1);
        tma::mbar_init(acc_empty, kTaConvWarps);
        for (int i = 0; i < kTaXRawSlots; ++i) {
            tma::mbar_init(&xraw_full[i], 1);
            tma::mbar_init(&xraw_empty[i], kTaStageWarps);
        }
        tma::fence_mbar_init();
    }
    if (warp == kTaMmaWarp) tc::tmem_alloc<512>(tbase_s);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tbase_s;
    const int nas = ta_astages(a);
    const uint32_t abase = (uint32_t)a.nmt * 64, astride = (uint32_t)a.nmt * 32;
    // Aligned X: the producer warp bulk-copies every item's 16 X rows into a 4-slot ring
    // ahead of the stagers (no L2 latency or address work on their per-item chain).
    const bool xfast = ((ldx | s) & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && !(dbg & 32);

    if (warp < kTaConvWarps) {
        // ---------------------------------------------------------- converters + epilogue
        const int mt = warp >> 2, qd = warp & 3;
        const int mrow = mt * 128 + qd * 32 + lane;
        int lv = -1, c = 0, fmt = HODLR_FMT_FP32, seg = 0, r8 = 0;
        for (int l = 0; l < a.nlev; ++l)
            if (mrow >= a.lev[l].mbase && mrow < a.lev[l].mbase + a.lev[l].r8) {
                lv = l;
                c = mrow - a.lev[l].mbase;
                fmt = a.lev[l].fmt;
                seg = a.lev[l].seg;
                r8 = a.lev[l].r8;
            }
        const int w = fmt_bytes(fmt);
        const uint32_t tl = tbase + ((uint32_t)(qd * 32) << 16);
        int64_t g = 0;
        int lc = 0;  // chunks consumed (epilogues done)
        if constexpr (!TSUM) {
            if (lv >= 0)
                for (int j = 0; j < kTcN; j += 4)
                    *reinterpret_cast<float4*>(sums + (size_t)mrow * kTaSumLd + j) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        // Epilogue of chunk ci (the lc-th chunk of this CTA).  The accumulator D stays in tensor
        // memory ACROSS the chunks of a node (the MMAs keep accumulating): a warp touches D only
        // when one of its rows ends its node's run here -- it reads D, writes the finished rows
        // (to the coefficient buffer when this CTA holds the whole node, else to the node's
        // partial slot), and stores D back with those rows zeroed.
        [[maybe_unused]] int pg = 0;
        auto epilogue = [&](int ci, int q0) {
            TC_PROG(5)
            tma::mbar_wait_sleep(acc_full, (unsigned)(lc & 1));
            TC_PROG(6)
            tc::fence_after();
            bool flush = false;
            float* dst = nullptr;
            if (lv >= 0 && !(dbg & 16)) {
                const int node = p.chunk_nodes[(int64_t)ci * p.nlev + lv];
                flush = !(ci + 1 < c_end && p.chunk_nodes[(int64_t)(ci + 1) * p.nlev + lv] == node);
                if (flush) {
                    const MrSlot sl = m.slots[node];
                    const NodeDesc nd = p.nodes[node];
                    if (sl.b0 == sl.b1 && nd.ext_slot < 0) {
                        if (c < nd.rv) dst = tbuf + nd.t_off * s + (int64_t)c * s + q0;
                    } else {
                        const MrLevel L = m.lev[lv];
                        if (c < L.rv_max)
                            dst = partial + (L.part_rows + ((int64_t)blockIdx.x + sl.jrel) * L.rv_pad + c) * spad + q0;
                    }
                }
            }
            if constexpr (TSUM) {
                if (mt < a.nmt && __any_sync(0xffffffffu, flush)) {
                    const int qn = (int)min((int64_t)kTcN, s - q0);
                    const bool vec = dst && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    #pragma unroll 1
                    for (int cc = 0; cc < kTcN; cc += 16) {
                        uint32_t v[16];
                        tc::ld_x16(tl + kTaAcc + mt * 64 + cc, v);
                        tc::wait_ld();
                        if (flush) {
                            if (dst) {
                                if (vec && cc + 16 <= qn) {  // 64 contiguous bytes per row: whole sectors
    #pragma unroll
                                    for (int j = 0; j < 16; j += 4)
                                        *reinterpret_cast<float4*>(dst + cc + j) =
                                            make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                        __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
                                } else {
    #pragma unroll
                                    for (int j = 0; j < 16; ++j)
                                        if (cc + j < qn) dst[cc + j] = __uint_as_float(v[j]);
                                }
                            }
    #pragma unroll
                            for (int j = 0; j < 16; ++j) v[j] = 0u;
                        }
                        tc::st_x16(tl + kTaAcc + mt * 64 + cc, v);
                    }
                    tc::wait_st();
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tma::mbar_arrive(acc_empty);
            } else {
                // D (this chunk) -> running sums of this thread's row, 16 bytes at a time
                float* my = sums + (size_t)mrow * kTaSumLd;
                if (mt < a.nmt) {
#pragma unroll 1
                    for (int cc = 0; cc < kTcN; cc += 16) {
                        uint32_t v[16];
                        tc::ld_x16(tl + kTaAcc + mt * 64 + cc, v);
                        tc::wait_ld();
                        if (lv >= 0) {
#pragma unroll
                            for (int j = 0; j < 16; j += 4) {
                                float4 t = *reinterpret_cast<float4*>(my + cc + j);
                                t.x += __uint_as_float(v[j]), t.y += __uint_as_float(v[j + 1]);
                                t.z += __uint_as_float(v[j + 2]), t.w += __uint_as_float(v[j + 3]);
                                *reinterpret_cast<float4*>(my + cc + j) = t;
                            }
                        }
                    }
                }
                // the accumulator is free again: the MMA warp starts the next chunk while the
                // finished rows are written out
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tma::mbar_arrive(acc_empty);
                // flush a row at a time, lanes along the right-hand sides (coalesced stores)
                const int qn = (int)min((int64_t)kTcN, s - q0);
                unsigned zm = __ballot_sync(0xffffffffu, flush);
                const unsigned wm = __ballot_sync(0xffffffffu, flush && dst != nullptr);
                const unsigned long long dbits = reinterpret_cast<unsigned long long>(dst);
                while (zm) {
                    const int r = __ffs(zm) - 1;
                    zm &= zm - 1;
                    float* drow = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, dbits, r));
                    const bool wr = (wm >> r) & 1u;
                    float* srow = sums + (size_t)(mt * 128 + qd * 32 + r) * kTaSumLd;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = lane + 32 * h;
                        const float val = srow[j];
                        if (wr && j < qn) drow[j] = val;
                        srow[j] = 0.f;
                    }
                }
                __syncwarp();
            }
            ++lc;
        };
        int pend_ci = -1, pend_q0 = 0;
        int rs = 0, as = 0;
        unsigned rpar = 0, apar = 0;
        bool a_first = true;
        const bool fin = a.finite != 0;
        for (int blk = 0; blk < nblk; ++blk) {
            const int q0 = blk * kTcN;
            for (int ci = c_beg; ci < c_end; ++ci) {
                for (int it = 0; it < kItems; ++it, ++g) {
                    // only converter warp 0 polls the item's mbarriers; the others wait at a
                    // hardware barrier (their waiting takes no issue slots)
                    TC_PROG(1)
                    if (warp == 0 || (dbg & 128)) {
                        tma::mbar_wait_sleep(&raw_full[rs], rpar);
                        if (!a_first) tma::mbar_wait_sleep(&a_empty[as], apar);
                    }
                    TC_PROG(2)
                    asm volatile("bar.sync 2, %0;" ::"n"(32 * kTaConvWarps) : "memory");
                    TC_PROG(3)
                    tc::fence_after();
                    uint32_t hi[16], lo[16];
                    if (lv >= 0 && !(dbg & 4)) {
                        const uint8_t* rp = ring + (size_t)rs * rslot + seg + (size_t)c * 4 * w;
                        float f[16];
                        if (fmt == HODLR_FMT_FP32) {  // the four 16-byte loads issue back to back
#pragma unroll
                            for (int kc = 0; kc < 4; ++kc) {
                                const float4 u = *reinterpret_cast<const float4*>(rp + (size_t)kc * r8 * 16);
                                f[4 * kc] = u.x, f[4 * kc + 1] = u.y, f[4 * kc + 2] = u.z, f[4 * kc + 3] = u.w;
                            }
                        } else {
#pragma unroll
                            for (int kc = 0; kc < 4; ++kc) {
                                const float4 u = load_quad(fmt, rp + (size_t)kc * r8 * 4 * w);
                                f[4 * kc] = u.x, f[4 * kc + 1] = u.y, f[4 * kc + 2] = u.z, f[4 * kc + 3] = u.w;
                            }
                        }
                        if (fin) {
#pragma unroll
                            for (int e = 0; e < 16; ++e) tc::split_tf32_fast(f[e], hi[e], lo[e]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 16; ++e) tc::split_tf32(f[e], hi[e], lo[e]);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) hi[e] = lo[e] = 0u;
                    }
                    if (mt < a.nmt) {  // warp-uniform: warps past the last tile only keep the protocol
                        const uint32_t ah = tl + abase + as * astride + mt * 32;
                        tc::st_x16(ah, hi);
                        tc::st_x16(ah + 16, lo);
                        tc::wait_st();
                    }
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        tma::mbar_arrive(&raw_empty[rs]);
                        tma::mbar_arrive(&a_full[as]);
                    }
                    TC_PROG(4)
                    ++pg;
                    if (++rs == nraw) rs = 0, rpar ^= 1u;
                    if (++as == nas) {
                        as = 0;
                        if (a_first) a_first = false; else apar ^= 1u;
                    }
                    if (it == 0 && pend_ci >= 0) {
                        epilogue(pend_ci, pend_q0);
                        pend_ci = -1;
                    }
                }
                pend_ci = ci;
                pend_q0 = q0;
            }
        }
        if (pend_ci >= 0) epilogue(pend_ci, pend_q0);
    } else if (warp == kTaProdWarp) {
        // ---------------------------------------------------------- producer
        // (whole warp: lane 0 moves the A item; the 16 X rows go one lane each, or as one copy
        // when they are contiguous)
        const uint64_t pol = tma::policy_evict_first();
        int rs = 0, xs = 0;
        [[maybe_unused]] int pg = 0;
        unsigned rpar = 0, xpar = 0;  // parity of the *_empty waits from the second pass on
        bool r_first = true, x_first = true;
        for (int blk = 0; blk < nblk; ++blk) {
            const int q0 = blk * kTcN;
            const unsigned rowbytes = (unsigned)min((int64_t)kTcN, s - q0) * 4u;
            const bool one = (uint64_t)ldx * 4u == rowbytes && rowbytes == kTcN * 4;
            for (int ci = c_beg; ci < c_end; ++ci) {
                const uint8_t* src = a.slab + (int64_t)ci * a.chunk_bytes;
                const float* xsrc = x + (int64_t)p.chunks[ci].row0 * ldx + q0;
                for (int it = 0; it < kItems; ++it) {
                    if (lane == 0) {
                        TC_PROG(1)
                        if (!r_first) tma::mbar_wait_sleep(&raw_empty[rs], rpar);
                        TC_PROG(2)
                        tma::mbar_arrive_tx(&raw_full[rs], (unsigned)a.item_bytes);
                        tma::bulk_g2s(ring + (size_t)rs * rslot, src + (int64_t)it * a.item_bytes,
                                      (unsigned)a.item_bytes, &raw_full[rs], pol);
                    }
                    if (++rs == nraw) {
                        rs = 0;
                        if (r_first) r_first = false; else rpar ^= 1u;
                    }
                    if (xfast) {
                        // (lane 0 does every mbarrier wait of this warp: the other lanes block at the
                        // __syncwarp below instead of spinning on a divergent path next to lane 0's)
                        float* dst = xraw + (size_t)xs * (kTaXRawSlot / 4);
                        const float* xr = xsrc + (int64_t)it * kTcAItemRows * ldx;
                        const unsigned nv = ((dbg & 8) && !(dbg & 64)) ? 0u : (unsigned)kTcAItemRows;
                        if (lane == 0) {
                            TC_PROG(3)
                            if (!x_first) tma::mbar_wait_sleep(&xraw_empty[xs], xpar);
                            TC_PROG(4)
                            tma::mbar_arrive_tx(&xraw_full[xs], nv * rowbytes);
                        }
                        ++pg;
                        __syncwarp();
                        if (one) {
                            if (lane == 0 && nv) tma::bulk_g2s_plain(dst, xr, nv * rowbytes, &xraw_full[xs]);
                        } else if (lane < (int)nv) {
                            tma::bulk_g2s_plain(dst + lane * kTcN, xr + (int64_t)lane * ldx, rowbytes, &xraw_full[xs]);
                        }
                        if (++xs == kTaXRawSlots) {
                            xs = 0;
                            if (x_first) x_first = false; else xpar ^= 1u;
                        }
                    }
                }
            }
        }
    } else if (warp == kTaMmaWarp) {
        // ---------------------------------------------------------- MMA issuer
        // (whole warp, uniform control flow; the MMAs and commits are predicated on one elected lane,
        // see tc::mma_tf32_ts_u)
        const uint32_t leader = tc::elect_one();
        {
            int64_t g = 0;
            int lc = 0;
            int as = 0, bs = 0;
            [[maybe_unused]] int pg = 0;
            unsigned a_par = 0, b_par = 0;
            for (int blk = 0; blk < nblk; ++blk) {
                const int q0 = blk * kTcN;
                const int nn = (int)min((int64_t)kTcN, (s - q0 + 15) / 16 * 16);
                const uint32_t idesc = tc::idesc_tf32(128, nn);
                const uint32_t lbo = (uint32_t)(nn / 8) * 128;
                for (int ci = c_beg; ci < c_end; ++ci, ++lc) {
                    TC_PROG(1)
                    if (lc >= 1) tma::mbar_wait_sleep(acc_empty, (unsigned)((lc - 1) & 1));
                    for (int it = 0; it < kItems; ++it, ++g) {
                        // (stage indices and parities kept as counters: a 64-bit g % nas with a
                        // runtime nas takes the operands out of the uniform datapath)
                        TC_PROG(2)
                        tma::mbar_wait_sleep(&a_full[as], a_par);
                        TC_PROG(3)
                        tma::mbar_wait_sleep(&b_full[bs], b_par);
                        TC_PROG(4)
                        ++pg;
                        tc::fence_after();
                        const uint32_t bh = tc::smem_u32(bring + (size_t)bs * kTaBSlot), bl = bh + kTaBHalf;
#pragma unroll
                        for (int j = 0; j < kTcAItemRows; j += 8) {
                            const uint64_t dh = tc::smem_desc(bh + (uint32_t)(j >> 2) * lbo, lbo, 128);
                            const uint64_t dl = tc::smem_desc(bl + (uint32_t)(j >> 2) * lbo, lbo, 128);
#pragma unroll
                            for (int t = 0; t < kTcAMaxTiles; ++t) {
                                if (t >= a.nmt) break;
                                const uint32_t d = tbase + kTaAcc + t * 64;
                                const uint32_t ah = tbase + abase + as * astride + t * 32 + j;
                                if (dbg & 2) continue;
                                tc::mma_tf32_ts_u(d, ah, dh, idesc, ((TSUM ? lc : 0) | it | j) != 0, leader);
                                tc::mma_tf32_ts_u(d, ah, dl, idesc, 1, leader);
                                if (((a.tile_full >> t) & 1) && !(dbg & 1)) tc::mma_tf32_ts_u(d, ah + 16, dh, idesc, 1, leader);
                            }
                        }
                        tc::commit_u(&a_empty[as], leader);
                        tc::commit_u(&b_empty[bs], leader);
                        if (++as == nas) {
                            as = 0;
                            a_par ^= 1u;
                        }
                        if (++bs == kTaBStages) {
                            bs = 0;
                            b_par ^= 1u;
                        }
                    }
                    tc::commit_u(acc_full, leader);
                }
            }
        }
    } else {
        // ---------------------------------------------------------- X stagers
        const int t = threadIdx.x - kTaStageWarp0 * 32;
        if (xfast) {
            // stager warp 0 polls the item's two mbarriers; the others wait at a hardware barrier
            int bs = 0, xs = 0;
            [[maybe_unused]] int pg = 0;
            unsigned bpar = 0, xpar = 0;
            bool b_first = true;
            for (int blk = 0; blk < nblk; ++blk) {
                const int q0 = blk * kTcN;
                const int nn = (int)min((int64_t)kTcN, (s - q0 + 15) / 16 * 16);
                const int lbo = (nn / 8) * 128;
                const int nunits = 4 * nn;
                // this thread's two (column quad kc, right-hand side n) units, fixed for the pass
                int kcs[2], ns[2], offs[2];
                bool oks[2], lds[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int u = e * 32 * kTaStageWarps + t;
                    kcs[e] = u / nn, ns[e] = u - kcs[e] * nn;
                    oks[e] = u < nunits;
                    lds[e] = oks[e] && q0 + ns[e] < s && !(dbg & 8);
                    offs[e] = kcs[e] * lbo + (ns[e] >> 3) * 128 + (ns[e] & 7) * 16;
                }
                for (int ci = c_beg; ci < c_end; ++ci) {
                    for (int it = 0; it < kItems; ++it) {
                        TC_PROG(1)
                        if (warp == kTaStageWarp0 || (dbg & 256)) {
                            tma::mbar_wait_sleep(&xraw_full[xs], xpar);
                            TC_PROG(2)
                            if (!b_first) tma::mbar_wait_sleep(&b_empty[bs], bpar);
                        }
                        TC_PROG(3)
                        asm volatile("bar.sync 1, %0;" ::"n"(32 * kTaStageWarps) : "memory");
                        TC_PROG(4)
                        ++pg;
                        const float* rb = xraw + (size_t)xs * (kTaXRawSlot / 4);
                        uint8_t* bh = bring + (size_t)bs * kTaBSlot;
                        uint8_t* bl = bh + kTaBHalf;
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            if (!oks[e]) continue;
                            float v4[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) v4[k] = lds[e] ? rb[(kcs[e] * 4 + k) * kTcN + ns[e]] : 0.f;
                            uint4 h, l;
                            tc::split_tf32(v4[0], h.x, l.x);
                            tc::split_tf32(v4[1], h.y, l.y);
                            tc::split_tf32(v4[2], h.z, l.z);
                            tc::split_tf32(v4[3], h.w, l.w);
                            *reinterpret_cast<uint4*>(bh + offs[e]) = h;
                            *reinterpret_cast<uint4*>(bl + offs[e]) = l;
                        }
                        tma::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma::mbar_arrive(&b_full[bs]);
                            tma::mbar_arrive(&xraw_empty[xs]);
                        }
                        if (++xs == kTaXRawSlots) xs = 0, xpar ^= 1u;
                        if (++bs == kTaBStages) {
                            bs = 0;
                            if (b_first) b_first = false; else bpar ^= 1u;
                        }
                    }
                }
            }
        } else {
            int64_t g = 0;
            for (int blk = 0; blk < nblk; ++blk) {
                const int q0 = blk * kTcN;
                const int nn = (int)min((int64_t)kTcN, (s - q0 + 15) / 16 * 16);
                const int lbo = (nn / 8) * 128;
                const int nunits = 4 * nn;
                // loads of the next item are issued before the current one is split and stored
                // (and before the wait for its slot): one L2 latency per item off the critical path
                auto load_item = [&](int ci, int it, float (&vals)[2][4]) {
                    const float* src = x + ((int64_t)p.chunks[ci].row0 + it * kTcAItemRows) * ldx + q0;
    #pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int u = e * 32 * kTaStageWarps + t;
                        const int kc = u / nn, n = u - kc * nn;
                        const bool ok = u < nunits && q0 + n < s;
    #pragma unroll
                        for (int k = 0; k < 4; ++k) vals[e][k] = ok && !(dbg & 8) ? __ldg(src + (int64_t)(kc * 4 + k) * ldx + n) : 0.f;
                    }
                };
                float nxt[2][4];
                if (c_beg < c_end) load_item(c_beg, 0, nxt);
                for (int ci = c_beg; ci < c_end; ++ci) {
                    for (int it = 0; it < kItems; ++it, ++g) {
                        const int bs = (int)(g % kTaBStages);
                        float vals[2][4];
    #pragma unroll
                        for (int e = 0; e < 2; ++e)
    #pragma unroll
                            for (int k = 0; k < 4; ++k) vals[e][k] = nxt[e][k];
                        if (it + 1 < kItems)
                            load_item(ci, it + 1, nxt);
                        else if (ci + 1 < c_end)
                            load_item(ci + 1, 0, nxt);
                        if (g >= kTaBStages) tma::mbar_wait_sleep(&b_empty[bs], (unsigned)(((g / kTaBStages) & 1) ^ 1));
                        uint8_t* bh = bring + (size_t)bs * kTaBSlot;
                        uint8_t* bl = bh + kTaBHalf;
    #pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int u = e * 32 * kTaStageWarps + t;
                            if (u >= nunits) continue;
                            const int kc = u / nn, n = u - kc * nn;
                            uint4 h, l;
                            tc::split_tf32(vals[e][0], h.x, l.x);
                            tc::split_tf32(vals[e][1], h.y, l.y);
                            tc::split_tf32(vals[e][2], h.z, l.z);
                            tc::split_tf32(vals[e][3], h.w, l.w);
                            const int off = kc * lbo + (n >> 3) * 128 + (n & 7) * 16;
                            *reinterpret_cast<uint4*>(bh + off) = h;
                            *reinterpret_cast<uint4*>(bl + off) = l;
                        }
                        tma::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) tma::mbar_arrive(&b_full[bs]);
                    }
                }
            }
    }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == kTaMmaWarp) {
        tc::fence_after();
        tc::tmem_free<512>(tbase);
    }
}

// A slab relayout (create time): one thread per (chunk, item, level, column quad kc, c).
__global__ void k_tca_slab(PlanView p, const __grid_constant__ TcAView a, int64_t units_per_item, uint8_t* slab) {
    constexpr int kItems = kChunkRowsTa / kTcAItemRows;
    const int64_t total = units_per_item * kItems * p.nchunks;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ci_it = idx / units_per_item;
        int64_t r = idx - ci_it * units_per_item;
        const int chunk = (int)(ci_it / kItems), it = (int)(ci_it % kItems);
        int l = 0;
        for (;; ++l) {
            const int64_t cnt = 4LL * a.lev[l].r8;
            if (r < cnt) break;
            r -= cnt;
        }
        const TcALevel L = a.lev[l];
        const int kc = (int)(r / L.r8), c = (int)(r % L.r8);
        const int w = fmt_bytes(L.fmt);
        uint8_t* dst = slab + (int64_t)chunk * a.chunk_bytes + (int64_t)it * a.item_bytes + L.seg +
                       ((int64_t)kc * L.r8 + c) * 4 * w;
        const ChunkDesc ch = p.chunks[chunk];
        const NodeDesc nd = p.nodes[p.chunk_nodes[(int64_t)chunk * p.nlev + l]];
        const int row = ch.row0 - nd.row0 + it * kTcAItemRows + 4 * kc;
        const uint8_t* src = c < nd.rv ? p.arena + nd.v_off + ((int64_t)c * nd.v_ld + row) * w : nullptr;
        for (int e = 0; e < 4 * w; ++e) dst[e] = src ? src[e] : (uint8_t)0;
    }
}

}  // namespace

static hodlr_status tca_prepare(const MrInput& in, MrPlan& mr);

hodlr_status tc_prepare(const MrInput& in, MrPlan& mr) {
    if (in.leaf_fmt != HODLR_FMT_FP32 || !mr.ok || mr.has_fp64_operand || getenv("HODLR_B200_NO_TC"))
        return HODLR_OK;
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, in.device);
    if (major != 10) return HODLR_OK;
    const auto& nodes = *in.nodes;
    const auto& chunks = *in.chunks;
    const auto& leaves = *in.leaves;
    for (const ChunkDesc& c : chunks) {
        const LeafDesc& l = leaves[c.leaf];
        if (c.nrows != kTcRows || l.m != kTcRows || l.row0 != c.row0 || l.fmt != HODLR_FMT_FP32) return HODLR_OK;
    }
    TcView& v = mr.tcv;
    v = TcView{};
    v.nlev = in.nlev;
    int64_t off = 0;
    auto add = [&](int fmt, int ncols, int lv, int col0) {
        if (v.nitems >= kTcMaxItems) return false;
        TcItem& it = v.item[v.nitems++];
        it.off = (int32_t)off;
        it.bytes = kTcRows * ncols * fmt_bytes(fmt);
        it.fmt = (int16_t)fmt;
        it.ncols = (int16_t)ncols;
        it.lv = (int16_t)lv;
        it.col0 = (int16_t)col0;
        off += it.bytes;
        return true;
    };
    for (int c = 0; c < kTcRows; c += kTcItemCols)
        if (!add(HODLR_FMT_FP32, kTcItemCols, -1, c)) return HODLR_OK;
    for (int lv = 0; lv < in.nlev; ++lv) {
        const MrLevel& L = mr.view.lev[lv];
        int fmt = -1;
        for (int id = L.node0; id < L.node0 + L.nnodes; ++id) {
            const NodeDesc& nd = nodes[id];
            if (nd.ru <= 0) continue;
            if (fmt >= 0 && fmt != nd.u_fmt) return HODLR_OK;  // one storage format per level
            fmt = nd.u_fmt;
        }
        if (fmt < 0) continue;
        if (fmt == HODLR_FMT_FP64) return HODLR_OK;
        const int R = (L.ru_max + 7) / 8 * 8;
        for (int c = 0; c < R; c += kTcItemCols)
            if (!add(fmt, std::min(kTcItemCols, R - c), lv, c)) return HODLR_OK;
    }
    v.leaf_bytes = (off + 127) / 128 * 128;
    if (v.leaf_bytes >= (1LL << 31)) return HODLR_OK;
    int64_t upc = 0;
    for (int i = 0; i < v.nitems; ++i) upc += (int64_t)(v.item[i].ncols >> 2) * kTcRows;
    const size_t bytes = (size_t)v.leaf_bytes * chunks.size();
    void* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) {
        cudaGetLastError();
        return HODLR_OK;  // no room: the fragment-slab kernels serve
    }
    cudaError_t e = cudaMemset(d, 0, bytes);
    if (e == cudaSuccess) {
        k_tc_slab<<<148 * 8, 256>>>(*in.view, v, upc, (uint8_t*)d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(d);
        return HODLR_ERR_CUDA;
    }
    v.slab = (const uint8_t*)d;
    v.finite = slab_finite(d, bytes);
    mr.tc_dev = d;
    mr.tc_ok = true;
    (void)nodes;
    if (mr.tca_cand) return tca_prepare(in, mr);
    return HODLR_OK;
}


bool tc_a_candidate(const MrInput& in, const MrView& v) {
    if (in.leaf_fmt != HODLR_FMT_FP32 || getenv("HODLR_B200_NO_TC")) return false;
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, in.device);
    if (major != 10) return false;
    for (const ChunkDesc& c : *in.chunks) {
        const LeafDesc& l = (*in.leaves)[c.leaf];
        if (c.nrows != kTcRows || l.m != kTcRows || l.row0 != c.row0) return false;
    }
    int mtot = 0;
    for (int lv = 0; lv < in.nlev; ++lv) {
        const MrLevel& L = v.lev[lv];
        int fmt = -1;
        for (int id = L.node0; id < L.node0 + L.nnodes; ++id) {
            const NodeDesc& nd = (*in.nodes)[id];
            if (nd.rv <= 0) continue;
            if ((fmt >= 0 && fmt != nd.v_fmt) || nd.v_fmt == HODLR_FMT_FP64) return false;
            fmt = nd.v_fmt;
        }
        mtot += L.rv_max;
    }
    return mtot > 0 && mtot <= 128 * kTcAMaxTiles;
}

static hodlr_status tca_prepare(const MrInput& in, MrPlan& mr) {
    TcAView& a = mr.tcav;
    a = TcAView{};
    a.nlev = in.nlev;
    int mb = 0, seg = 0;
    for (int lv = 0; lv < in.nlev; ++lv) {
        const MrLevel& L = mr.view.lev[lv];
        int fmt = HODLR_FMT_FP32;
        for (int id = L.node0; id < L.node0 + L.nnodes; ++id)
            if ((*in.nodes)[id].rv > 0) fmt = (*in.nodes)[id].v_fmt;
        TcALevel& T = a.lev[lv];
        T.mbase = mb;
        T.r8 = L.rv_max;  // rows stacked without padding (any row -> TMEM lane mapping works)
        T.fmt = fmt;
        T.seg = seg;
        if (fmt == HODLR_FMT_FP32)
            for (int t = mb / 128; t <= (mb + std::max(T.r8, 1) - 1) / 128; ++t) a.tile_full |= 1u << t;
        mb += T.r8;
        seg += kTcAItemRows * T.r8 * fmt_bytes(fmt);
    }
    a.mtot = mb;
    a.nmt = (mb + 127) / 128;
    a.item_bytes = seg;
    a.chunk_bytes = (int64_t)seg * (kChunkRowsTa / kTcAItemRows);
    if (ta_smem(a, 2, false) > 227 * 1024) return HODLR_OK;
    const size_t bytes = (size_t)a.chunk_bytes * in.chunks->size();
    void* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) {
        cudaGetLastError();
        return HODLR_OK;
    }
    k_tca_slab<<<148 * 8, 256>>>(*in.view, a, 4LL * mb, (uint8_t*)d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(d);
        return HODLR_ERR_CUDA;
    }
    a.slab = (const uint8_t*)d;
    a.finite = slab_finite(d, bytes);
    mr.tca_dev = d;
    mr.tca_ok = true;
    return HODLR_OK;
}

bool tca_usable(const MrPlan& mr, int64_t s) {
    return mr.tca_ok && s > 1 && !getenv("HODLR_B200_NO_TC") && !getenv("HODLR_B200_NO_TCA");
}

cudaError_t tc_phase_a(const PlanView& p, const MrPlan& mr, const float* x, int64_t ldx, int64_t s, float* partial,
                       float* tbuf, cudaStream_t st) {
    if (p.nchunks == 0) return cudaSuccess;
    // HODLR_B200_TC_SUMS=tmem: keep a node's running sums in tensor memory (faster, ~4x the
    // rounding error: the tensor core accumulates with truncation); default: fp32 sums in smem
    const char* sums_env = getenv("HODLR_B200_TC_SUMS");
    const bool tsum = sums_env && sums_env[0] == 't';
    const int nraw = ta_nraw(mr.tcav, tsum);
    const size_t sm = ta_smem(mr.tcav, nraw, tsum);
    auto kern = tsum ? k_tc_a<true> : k_tc_a<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int nblk = (int)((s + kTcN - 1) / kTcN);
#ifdef HODLR_TC_PROGRESS
    {
        static int* host = nullptr;
        if (!host) {
            cudaHostAlloc(&host, 64 * sizeof(int), cudaHostAllocMapped);
            int* dev = nullptr;
            cudaHostGetDevicePointer(&dev, host, 0);
            cudaMemcpyToSymbol(g_progress, &dev, sizeof(dev));
        }
        for (int i = 0; i < 64; ++i) host[i] = -1;
        std::thread([] {
            std::this_thread::sleep_for(std::chrono::seconds(3));
            fprintf(stderr, "PROGRESS");
            for (int i = 0; i < kTaThreads / 32; ++i) fprintf(stderr, " w%d:%d.%d", i, host[i] >> 8, host[i] & 255);
            fprintf(stderr, "\n");
        }).detach();
    }
#endif
    kern<<<mr.view.nb, kTaThreads, sm, st>>>(p, mr.view, mr.tcav, x, ldx, s, (int)mr_spad(s), nblk, partial,
                                                tbuf, nraw, getenv("HODLR_TC_DBG") ? atoi(getenv("HODLR_TC_DBG")) : 0);
    return cudaGetLastError();
}

bool tc_usable(const MrPlan& mr, int64_t s) {
    return mr.tc_ok && s > 1 && !getenv("HODLR_B200_NO_TC") && !getenv("HODLR_B200_NO_TCB");
}

cudaError_t tc_phase_b(const PlanView& p, const MrPlan& mr, const float* x, int64_t ldx, float* b, int64_t ldb,
                       int64_t s, const float* tbuf, cudaStream_t st) {
    if (p.nchunks == 0) return cudaSuccess;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_tc_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int nblk = (int)((s + kTcN - 1) / kTcN);
    const int nwork = p.nchunks * nblk;
    const int grid = std::min(nwork, sms);
    k_tc_b<<<grid, kTcThreads, kTcSmem, st>>>(p, mr.tcv, x, ldx, tbuf, b, ldb, s, nblk,
                                               getenv("HODLR_TC_DBG") ? atoi(getenv("HODLR_TC_DBG")) : 0);
    return cudaGetLastError();
}

}  // namespace hodlr
