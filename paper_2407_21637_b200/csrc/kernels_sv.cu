// Single-vector (s = 1) fast path: ONE persistent cooperative kernel per matvec.
//
// Work list (dynamic, one atomic queue):
//   items [0, A)    phase A, one per leaf-chunk of M rows: partial V'^T x of every
//                   level's V' column restricted to the chunk (16-byte loads of the
//                   narrow factor, in-register up-conversion, warp-shuffle reduce);
//                   the last chunk of a node to finish reduces the node's partials
//                   in chunk order (deterministic) into t and publishes a flag.
//   items [A, A+B)  phase B, one per RB-row block of a leaf: y = D x first (no
//                   dependency; 16-byte loads of the dense leaf), then wait for the
//                   t of every ancestor level (flags), then
//                   b = sum_k U_k t_{k,sib} + y, written once (rows are disjoint: no
//                   atomics on b).
// Phase-A items are handed out before any phase-B item and never wait, so with all
// CTAs co-resident (cooperative launch) the flag waits always make progress.  The
// leaf product of the first phase-B items hides the reduction latency, so the
// grid-wide dependency of Alg. 3's level-1 inner product costs no barrier.
// Per-call state (queue, counters, flags, epoch) lives in the zero-initialised
// workspace; the last CTA to finish resets it and bumps the epoch.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "sv.h"

namespace hodlr {

namespace {

constexpr int kM = 256;        // rows per phase-A chunk (= leaf size of the fast path)
constexpr int kRB = 32;        // rows per phase-B item
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLev = 24;

struct SvSync {
    unsigned epoch, queue, done, pad;
};

struct SvDev {
    int32_t* sib;  // [nnodes] node whose t the U of this node consumes
};

template <typename W>
struct SvArgs {
    const W* x;
    W* b;
    W* partial;
    W* tbuf;
    SvSync* sync;
    unsigned* counters;  // [nnodes]
    unsigned* flags;     // [nnodes]
    const int32_t* sib;
    int num_a, num_b, items_per_leaf;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 16-byte streaming load (read-once data: do not pollute L1).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Unpack a 16-byte vector of format FMT into E = 16/bytes(FMT) values and
// accumulate dot with xs[0..E).
template <int FMT, typename W>
__device__ __forceinline__ W dot16_word(uint32_t w, const W* xs, W acc) {
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
    } else {  // q52 (e5m2): byte b -> binary16 bits b << 8
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

// Unpack a 16-byte vector of format FMT into E = 16/bytes(FMT) values and
// accumulate their dot product with xs[0..E).
template <int FMT, typename W>
__device__ __forceinline__ W dot16(const uint4& v, const W* xs, W acc) {
    if constexpr (FMT == HODLR_FMT_FP64) {
        acc = dot_f64<W>(v.x, v.y, xs[0], acc);
        acc = dot_f64<W>(v.z, v.w, xs[1], acc);
    } else {
        constexpr int PW = FMT == HODLR_FMT_FP32 ? 1 : FMT == HODLR_FMT_Q52 ? 4 : 2;
        acc = dot16_word<FMT, W>(v.x, xs + 0 * PW, acc);
        acc = dot16_word<FMT, W>(v.y, xs + 1 * PW, acc);
        acc = dot16_word<FMT, W>(v.z, xs + 2 * PW, acc);
        acc = dot16_word<FMT, W>(v.w, xs + 3 * PW, acc);
    }
    return acc;
}

// Up to 4 columns (same node => same format) dotted with the chunk's x over kM
// rows: all loads of the group are issued before the math.
template <int FMT, typename W>
__device__ __forceinline__ void dot_cols(const uint8_t* col0, int64_t cstride, int ncols,
                                         const W* xs, int lane, W out[4]) {
    constexpr int E = 16 / (FMT == HODLR_FMT_FP64 ? 8 : FMT == HODLR_FMT_FP32 ? 4
                            : FMT == HODLR_FMT_Q52 ? 1 : 2);
    constexpr int NV = kM / E;                   // 16-byte vectors per column
    constexpr int PER = NV >= 32 ? NV / 32 : 1;  // per lane
    const bool active = NV >= 32 || lane < NV;
    uint4 v[4][PER];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < PER; ++i)
            if (c < ncols && active) v[c][i] = ldg_stream(col0 + c * cstride + (int64_t)(lane + 32 * i) * 16);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        W acc = W(0);
        if (c < ncols && active) {
#pragma unroll
            for (int i = 0; i < PER; ++i) acc = dot16<FMT, W>(v[c][i], xs + (lane + 32 * i) * E, acc);
        }
        out[c] = acc;
    }
}

template <typename W>
__device__ __forceinline__ void dot_cols_any(int fmt, const uint8_t* col0, int64_t cstride, int ncols,
                                             const W* xs, int lane, W out[4]) {
    switch (fmt) {
        case HODLR_FMT_FP64: dot_cols<HODLR_FMT_FP64, W>(col0, cstride, ncols, xs, lane, out); break;
        case HODLR_FMT_FP32: dot_cols<HODLR_FMT_FP32, W>(col0, cstride, ncols, xs, lane, out); break;
        case HODLR_FMT_FP16: dot_cols<HODLR_FMT_FP16, W>(col0, cstride, ncols, xs, lane, out); break;
        case HODLR_FMT_BF16: dot_cols<HODLR_FMT_BF16, W>(col0, cstride, ncols, xs, lane, out); break;
        default: dot_cols<HODLR_FMT_Q52, W>(col0, cstride, ncols, xs, lane, out); break;
    }
}

template <typename W>
__device__ __forceinline__ W load_elem(int fmt, const uint8_t* col, int i) {
    switch (fmt) {
        case HODLR_FMT_FP64: return (W)__ldg((const double*)col + i);
        case HODLR_FMT_FP32: return (W)__ldg((const float*)col + i);
        case HODLR_FMT_FP16: return (W)dec_fp16(__ldg((const unsigned short*)col + i));
        case HODLR_FMT_BF16: return (W)dec_bf16(__ldg((const unsigned short*)col + i));
        default: return (W)dec_q52(__ldg(col + i));
    }
}

struct __align__(16) SmemA {
    int lev_node[kMaxLev];
    int lev_groups[kMaxLev + 1];  // prefix sums of ceil(rv/4)
    int last[kMaxLev];
};

template <typename W>
__global__ void __launch_bounds__(kThreads, 1) k_sv_fused(PlanView p, SvArgs<W> a) {
    __shared__ __align__(16) W xs[kM];
    __shared__ __align__(16) W ts[512];          // phase-B coefficients (sum of ranks <= 512)
    __shared__ W red[kWarps][kRB];
    __shared__ W yrow[kRB];
    __shared__ SmemA sa;
    __shared__ int s_item;
    __shared__ unsigned s_epoch;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nlev = p.nlev;
    const int total = a.num_a + a.num_b;

    if (threadIdx.x == 0) s_epoch = ld_acquire(&a.sync->epoch);
    __syncthreads();
    const unsigned target = s_epoch + 1;

    for (;;) {
        if (threadIdx.x == 0) s_item = (int)atomicAdd(&a.sync->queue, 1u);
        __syncthreads();
        const int item = s_item;
        if (item >= total) break;
        if (item < a.num_a) {
            // ------------------------------------------------ phase A
            const int chunk = item;
            const ChunkDesc ch = p.chunks[chunk];
            for (int i = threadIdx.x; i < kM; i += kThreads) xs[i] = a.x[ch.row0 + i];
            if (threadIdx.x == 0) {
                int g = 0;
                for (int lv = 0; lv < nlev; ++lv) {
                    int id = p.chunk_nodes[chunk * nlev + lv];
                    sa.lev_node[lv] = id;
                    sa.lev_groups[lv] = g;
                    g += (p.nodes[id].rv + 3) >> 2;
                }
                sa.lev_groups[nlev] = g;
            }
            __syncthreads();
            const int ngroups = sa.lev_groups[nlev];
            for (int gi = warp; gi < ngroups; gi += kWarps) {
                int lv = 0;
                while (sa.lev_groups[lv + 1] <= gi) ++lv;
                const NodeDesc& nd = p.nodes[sa.lev_node[lv]];
                const int c0 = (gi - sa.lev_groups[lv]) * 4;
                const int nc = min(4, nd.rv - c0);
                const int64_t cstride = (int64_t)nd.v_ld * fmt_bytes(nd.v_fmt);
                const uint8_t* col0 = p.arena + nd.v_off + c0 * cstride +
                                      (int64_t)(ch.row0 - nd.row0) * fmt_bytes(nd.v_fmt);
                W out[4];
                dot_cols_any<W>(nd.v_fmt, col0, cstride, nc, xs, lane, out);
#pragma unroll
                for (int c = 0; c < 4; ++c) out[c] = warp_sum(out[c]);
                if (lane < nc) {
                    W v = lane == 0 ? out[0] : lane == 1 ? out[1] : lane == 2 ? out[2] : out[3];
                    a.partial[nd.part_off + (int64_t)(c0 + lane) * nd.nchunk + (chunk - nd.chunk0)] = v;
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                for (int lv = 0; lv < nlev; ++lv) {
                    const int id = sa.lev_node[lv];
                    const NodeDesc& nd = p.nodes[id];
                    unsigned old = atomicAdd(&a.counters[id], 1u);
                    sa.last[lv] = (old == (unsigned)nd.nchunk - 1) ? 1 : 0;
                }
                __threadfence();
            }
            __syncthreads();
            // last arriver of a node: fixed-order reduction over its chunks
            for (int lv = 0; lv < nlev; ++lv) {
                if (!sa.last[lv]) continue;
                const int id = sa.lev_node[lv];
                const NodeDesc& nd = p.nodes[id];
                for (int c = warp; c < nd.rv; c += kWarps) {
                    const W* src = a.partial + nd.part_off + (int64_t)c * nd.nchunk;
                    // lane-strided in chunk order, then a fixed shuffle tree
                    W acc = W(0);
                    for (int j = lane; j < nd.nchunk; j += 32) acc += __ldcg(src + j);
                    acc = warp_sum(acc);
                    if (lane == 0) a.tbuf[nd.t_off + c] = acc;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    a.counters[id] = 0;
                    __threadfence();
                    st_release(&a.flags[id], target);
                }
            }
        } else {
            // ------------------------------------------------ phase B
            const int j = item - a.num_a;
            const int leaf = j / a.items_per_leaf;
            const int r0 = (j % a.items_per_leaf) * kRB;  // row offset inside the leaf
            const LeafDesc lf = p.leaves[leaf];
            for (int i = threadIdx.x; i < kM; i += kThreads) xs[i] = a.x[lf.row0 + i];
            __syncthreads();
            // y = D[r0:r0+RB, :] x_leaf  (warp: RB/kWarps rows; 16-B vectors)
            {
                constexpr int RPW = kRB / kWarps;
                const int wb = fmt_bytes(lf.fmt);
                const uint8_t* d0 = p.arena + lf.off + (int64_t)(r0 + warp * RPW) * lf.ld * wb;
                const int64_t rstride = (int64_t)lf.ld * wb;
                W acc[RPW];
                if (lf.fmt == HODLR_FMT_FP64) {
                    constexpr int PER = kM / 2 / 32;
                    uint4 v[RPW][PER];
#pragma unroll
                    for (int r = 0; r < RPW; ++r)
#pragma unroll
                        for (int i = 0; i < PER; ++i) v[r][i] = ldg_stream(d0 + r * rstride + (lane + 32 * i) * 16);
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        W s = W(0);
#pragma unroll
                        for (int i = 0; i < PER; ++i) s = dot16<HODLR_FMT_FP64, W>(v[r][i], xs + (lane + 32 * i) * 2, s);
                        acc[r] = s;
                    }
                } else {
                    constexpr int PER = kM / 4 / 32;
                    uint4 v[RPW][PER];
#pragma unroll
                    for (int r = 0; r < RPW; ++r)
#pragma unroll
                        for (int i = 0; i < PER; ++i) v[r][i] = ldg_stream(d0 + r * rstride + (lane + 32 * i) * 16);
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        W s = W(0);
#pragma unroll
                        for (int i = 0; i < PER; ++i) s = dot16<HODLR_FMT_FP32, W>(v[r][i], xs + (lane + 32 * i) * 4, s);
                        acc[r] = s;
                    }
                }
#pragma unroll
                for (int r = 0; r < RPW; ++r) {
                    W s = warp_sum(acc[r]);
                    if (lane == 0) yrow[warp * RPW + r] = s;
                }
            }
            // wait for the coefficients of every level, stage them in smem
            if (threadIdx.x == 0) {
                const int chunk = leaf;  // one chunk per leaf on this path
                int off = 0;
                for (int lv = 0; lv < nlev; ++lv) {
                    const int id = p.chunk_nodes[chunk * nlev + lv];
                    const int src = a.sib[id];
                    sa.lev_node[lv] = id;
                    sa.lev_groups[lv] = off;
                    off += p.nodes[id].ru;
                    if (ld_acquire(&a.flags[src]) != target) {
                        unsigned ns = 32;
                        while (ld_acquire(&a.flags[src]) != target) {
                            __nanosleep(ns);
                            ns = min(ns * 2, 256u);
                        }
                    }
                }
                sa.lev_groups[nlev] = off;
            }
            __syncthreads();
            const int ncoef = sa.lev_groups[nlev];
            for (int i = threadIdx.x; i < ncoef; i += kThreads) {
                int lv = 0;
                while (sa.lev_groups[lv + 1] <= i) ++lv;
                const NodeDesc& nd = p.nodes[sa.lev_node[lv]];
                ts[i] = __ldcg(a.tbuf + nd.tsrc_off + (i - sa.lev_groups[lv]));
            }
            __syncthreads();
            // U part: warp w takes coefficients w, w+8, ...; lane = row
            {
                W acc = W(0);
                const int row_in_leaf = r0 + lane;
                for (int i = warp; i < ncoef; i += kWarps) {
                    int lv = 0;
                    while (sa.lev_groups[lv + 1] <= i) ++lv;
                    const NodeDesc& nd = p.nodes[sa.lev_node[lv]];
                    const int c = i - sa.lev_groups[lv];
                    const int64_t cstride = (int64_t)nd.u_ld * fmt_bytes(nd.u_fmt);
                    const uint8_t* col = p.arena + nd.u_off + c * cstride;
                    const int r = lf.row0 + row_in_leaf - nd.row0;
                    acc = fma(load_elem<W>(nd.u_fmt, col, r), ts[i], acc);
                }
                red[warp][lane] = acc;
            }
            __syncthreads();
            if (warp == 0) {
                W s = W(0);
#pragma unroll
                for (int w = 0; w < kWarps; ++w) s += red[w][lane];
                a.b[lf.row0 + r0 + lane] = s + yrow[lane];
            }
        }
        __syncthreads();
    }
    // ---- teardown: the last CTA resets the queue and publishes the next epoch
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned old = atomicAdd(&a.sync->done, 1u);
        if (old == gridDim.x - 1) {
            a.sync->queue = 0;
            a.sync->done = 0;
            __threadfence();
            st_release(&a.sync->epoch, target);
        }
    }
}

}  // namespace

hodlr_status sv_prepare(const std::vector<NodeDesc>& nodes, const std::vector<ChunkDesc>& chunks,
                        const std::vector<LeafDesc>& leaves, const std::vector<int32_t>& chunk_nodes,
                        int nlev, SvPlan& sv, bool* ok) {
    sv = SvPlan{};
    *ok = false;
    if (nlev > kMaxLev || leaves.empty()) return HODLR_OK;
    for (const LeafDesc& l : leaves)
        if (l.m != kM || (l.fmt != HODLR_FMT_FP64 && l.fmt != HODLR_FMT_FP32)) return HODLR_OK;
    if (chunks.size() != leaves.size()) return HODLR_OK;
    for (const NodeDesc& nd : nodes)
        if (nd.ext_slot >= 0) return HODLR_OK;
    // sum of ranks a leaf consumes must fit the shared coefficient buffer
    std::vector<int32_t> sib(nodes.size(), -1);
    for (size_t c = 0; c < chunks.size(); ++c) {
        int tot = 0;
        for (int lv = 0; lv < nlev; ++lv) tot += nodes[chunk_nodes[c * nlev + lv]].ru;
        if (tot > 512) return HODLR_OK;
    }
    // sibling lookup: node whose t_off equals our tsrc_off
    for (size_t i = 0; i < nodes.size(); ++i) {
        for (size_t j = 0; j < nodes.size(); ++j) {
            if (nodes[j].level == nodes[i].level && nodes[j].t_off == nodes[i].tsrc_off && j != i) {
                sib[i] = (int32_t)j;
                break;
            }
        }
        if (sib[i] < 0 && nodes[i].ru > 0) return HODLR_OK;
        if (sib[i] < 0) sib[i] = (int32_t)i;  // rank-0 U: any published flag works
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HODLR_OK;
    int sms = 0, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (!coop || sms <= 0) return HODLR_OK;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sv_fused<double>, kThreads, 0) != cudaSuccess ||
        occ < 1)
        return HODLR_OK;
    int occf = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf, k_sv_fused<float>, kThreads, 0);
    occ = std::min(occ, std::max(occf, 1));
    void* d = nullptr;
    if (cudaMalloc(&d, sib.size() * sizeof(int32_t) + 16) != cudaSuccess) return HODLR_OK;
    cudaMemcpy(d, sib.data(), sib.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    sv.dev = d;
    sv.num_items_a = (int)chunks.size();
    sv.num_items_b = (int)leaves.size() * (kM / kRB);
    sv.grid = std::min(sms * std::min(occ, 2), sv.num_items_a + sv.num_items_b);
    sv.launches = 1;
    sv.extra_ws = sizeof(SvSync) + 2 * nodes.size() * sizeof(unsigned) + 256;
    *ok = true;
    return HODLR_OK;
}

void sv_release(SvPlan& sv) {
    if (sv.dev) cudaFree(sv.dev);
    sv = SvPlan{};
}
size_t sv_extra_ws(const SvPlan& sv, int64_t) { return sv.extra_ws; }
int sv_launches(const SvPlan& sv) { return sv.launches; }

template <typename W>
cudaError_t sv_matvec(const PlanView& p, const SvPlan& sv, const W* x, W* b, W* partial, W* tbuf,
                      void* extra, cudaStream_t st) {
    SvArgs<W> a;
    a.x = x;
    a.b = b;
    a.partial = partial;
    a.tbuf = tbuf;
    a.sync = (SvSync*)extra;
    a.counters = (unsigned*)((uint8_t*)extra + sizeof(SvSync));
    a.flags = a.counters + p.nnodes;
    a.sib = (const int32_t*)sv.dev;
    a.num_a = sv.num_items_a;
    a.num_b = sv.num_items_b;
    a.items_per_leaf = kM / kRB;
    PlanView pv = p;
    void* args[] = {&pv, &a};
    return cudaLaunchCooperativeKernel((const void*)k_sv_fused<W>, dim3(sv.grid), dim3(kThreads), args, 0, st);
}

template cudaError_t sv_matvec<double>(const PlanView&, const SvPlan&, const double*, double*,
                                       double*, double*, void*, cudaStream_t);
template cudaError_t sv_matvec<float>(const PlanView&, const SvPlan&, const float*, float*, float*,
                                      float*, void*, cudaStream_t);

}  // namespace hodlr
