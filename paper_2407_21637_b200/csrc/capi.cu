// C-ABI entry points (include/hodlr_b200.h): host-side packing of a HODLR
// matrix into the device layout of plan.h, and the stream-ordered matvec.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hodlr_b200.h"
#include "formats.cuh"
#include "kernels.h"
#include "mrhs.h"
#include "plan.h"
#include "sv.h"

using namespace hodlr;

namespace {

thread_local std::string g_err;

hodlr_status fail(hodlr_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return fail(HODLR_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)

constexpr int kChunkRows = 256;  // row tile: one leaf in the BASELINE configs
constexpr size_t kAlign = 256;

inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }
inline int elems_per_16B(int fmt) { return 16 / fmt_bytes(fmt); }
inline bool valid_fmt(int f) { return f >= HODLR_FMT_Q52 && f <= HODLR_FMT_FP64; }

struct DeviceBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    cudaError_t ensure(size_t want) {
        if (bytes >= want && p) return cudaSuccess;
        release();
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
};

}  // namespace

struct hodlr_handle {
    int device = 0;
    int depth = 0, L = 0, rank = 0, nranks = 1;
    int leaf_fmt = HODLR_FMT_FP64;
    int64_t n_global = 0, n_local = 0, row0 = 0;
    int64_t matrix_bytes = 0;
    int max_chunk_rows = 0;
    std::vector<NodeDesc> nodes;
    std::vector<ChunkDesc> chunks;
    std::vector<int32_t> chunk_nodes;
    std::vector<LeafDesc> leaves;
    std::vector<ExtDesc> ext;
    // (level k, node j) -> node id; only local nodes are present
    std::vector<std::vector<int>> node_id;
    std::vector<int64_t> factor_rows;  // for unpack: rows of U / V of each desc factor
    int64_t part_count = 0, t_count = 0, ext_count = 0;
    DeviceBuf arena, tables;
    // Host-buffer calls (hodlr_matvec_host): kHostCtx staging contexts, so calls from
    // different host threads (on different streams) overlap -- one call's device-to-host
    // copy runs under the next call's host-to-device copy (PCIe is full duplex).  A call
    // holds one context from entry to return; further callers wait for a free one.
    struct HostCtx {
        DeviceBuf e2e;                       // x / b staging (binary64 and working copies)
        cudaStream_t copy_stream = nullptr;  // device-to-host copies of finished row ranges
        std::vector<cudaEvent_t> slice_ev;
        cudaEvent_t h2d_ev = nullptr;        // this context's last host-to-device copy
        bool busy = false;
    };
    // Host-to-device copies of concurrent calls run one after the other (each waits for the
    // previous call's copy): two calls that start together then do not share the H2D
    // direction and finish it together -- the second call's copy runs under the first
    // call's kernels and device-to-host copy instead.
    cudaEvent_t last_h2d = nullptr;
    std::mutex h2d_mu;
    static constexpr int kHostCtx = 2;
    HostCtx hctx[kHostCtx];
    std::condition_variable hcv;
    // NULL-workspace calls: one zero-initialised workspace per CUDA stream, so
    // concurrent calls on different streams never share the fused kernel's
    // synchronisation state (matvec is safe to call concurrently)
    struct StreamWs {
        void* stream;
        DeviceBuf buf;
    };
    std::vector<StreamWs> ws;
    std::mutex ws_mu;
    size_t arena_bytes = 0;
    PlanView view{};
    bool sv_ok = false;  // single-vector fast path usable
    SvPlan sv{};
    MrPlan mr{};  // multi-RHS tensor-core path
    std::mutex mu;
};

namespace {

// Sequential writer of one arena segment: values are staged in binary64 on the
// host, copied to the device and quantised by K0 into the segment's format.
struct SegmentWriter {
    int fmt;
    uint8_t* dst;  // device, start of segment
    std::vector<double> host;
    double* dev_stage;
    int64_t flushed = 0;  // elements already written to the device
    size_t cap;
    cudaError_t err = cudaSuccess;

    SegmentWriter(int f, uint8_t* d, double* stage, size_t capacity)
        : fmt(f), dst(d), dev_stage(stage), cap(capacity) {
        host.reserve(cap);
    }
    void flush() {
        if (host.empty() || err != cudaSuccess) return;
        err = cudaMemcpy(dev_stage, host.data(), host.size() * sizeof(double),
                         cudaMemcpyHostToDevice);
        if (err == cudaSuccess)
            err = launch_quantize(fmt, dev_stage, dst + flushed * fmt_bytes(fmt),
                                  (int64_t)host.size(), 0);
        if (err == cudaSuccess) err = cudaStreamSynchronize(0);
        flushed += (int64_t)host.size();
        host.clear();
    }
    inline void put(double v) {
        host.push_back(v);
        if (host.size() == cap) flush();
    }
    int64_t position() const { return flushed + (int64_t)host.size(); }
};

struct ColumnSrc {  // a factor restricted to rows [r0, r0+nrows)
    const double* base;
    int64_t rs, cs, r0;
};

// element i of a payload: binary64, or (container v2) the narrow encoding of `enc`
inline double payload_at(const void* base, int enc, int64_t i) {
    return enc == HODLR_FMT_FP64 ? ((const double*)base)[i] : dec_any(enc, base, i);
}

hodlr_status build(const hodlr_desc* d, int device, hodlr_shard shard, hodlr_handle** out) {
    if (!d || !out) return fail(HODLR_ERR_INVALID, "null descriptor or output pointer");
    *out = nullptr;
    if (d->depth < 0 || d->depth > 30) return fail(HODLR_ERR_INVALID, "depth out of range");
    if (d->n < 1) return fail(HODLR_ERR_INVALID, "dimension must be positive");
    if (!valid_fmt(d->leaf_fmt)) return fail(HODLR_ERR_UNSUPPORTED, "unsupported leaf format");
    if (d->payload_encoded != 0 && d->payload_encoded != 1)
        return fail(HODLR_ERR_INVALID, "payload_encoded must be 0 or 1");
    const bool enc = d->payload_encoded == 1;
    const int depth = d->depth;
    const int64_t nleaf = int64_t(1) << depth;
    if (nleaf > d->n) return fail(HODLR_ERR_INVALID, "tree too deep for dimension");
    if (!d->leaf_bounds || !d->leaves || !d->leaf_ld || (depth > 0 && !d->factors))
        return fail(HODLR_ERR_INVALID, "missing descriptor arrays");
    const int64_t* bd = d->leaf_bounds;
    if (bd[0] != 0 || bd[nleaf] != d->n) return fail(HODLR_ERR_INVALID, "leaf bounds must span [0, n)");
    for (int64_t i = 0; i < nleaf; ++i)
        if (bd[i + 1] <= bd[i]) return fail(HODLR_ERR_INVALID, "leaf bounds must increase");
    if (d->n > (int64_t(1) << 31) - 1) return fail(HODLR_ERR_UNSUPPORTED, "n must fit in int32");
    int P = shard.nranks, g = shard.rank;
    if (P < 1 || (P & (P - 1)) || g < 0 || g >= P)
        return fail(HODLR_ERR_INVALID, "nranks must be a power of two and 0 <= rank < nranks");
    int L = 0;
    while ((1 << L) < P) ++L;
    if (L > depth) return fail(HODLR_ERR_INVALID, "more ranks than level-depth nodes (nranks > 2^depth)");

    auto node_rows = [&](int k, int64_t j, int64_t* a, int64_t* b) {
        int64_t span = int64_t(1) << (depth - k);
        *a = bd[j * span];
        *b = bd[(j + 1) * span];
    };
    // factors: level k (1-based), pair i -> index 2*(2^(k-1)-1) + 2i + {0 upper, 1 lower}
    auto fidx = [&](int k, int64_t i, int lower) {
        return 2 * ((int64_t(1) << (k - 1)) - 1) + 2 * i + lower;
    };
    // validate every factor's shape against the tree
    for (int k = 1; k <= depth; ++k) {
        for (int64_t i = 0; i < (int64_t(1) << (k - 1)); ++i) {
            int64_t a1, b1, a2, b2;
            node_rows(k, 2 * i, &a1, &b1);
            node_rows(k, 2 * i + 1, &a2, &b2);
            for (int lo = 0; lo < 2; ++lo) {
                const hodlr_factor_in& f = d->factors[fidx(k, i, lo)];
                int64_t want_r = lo ? b2 - a2 : b1 - a1, want_c = lo ? b1 - a1 : b2 - a2;
                if (!valid_fmt(f.fmt)) return fail(HODLR_ERR_UNSUPPORTED, "unsupported factor format");
                if (f.rank < 0 || f.rows != want_r || f.cols != want_c)
                    return fail(HODLR_ERR_INVALID, "factor shape does not match the cluster tree (level " +
                                                       std::to_string(k) + ", pair " + std::to_string(i) + ")");
                if (f.rank > 0 && (!f.U || !f.V)) return fail(HODLR_ERR_INVALID, "null factor data");
            }
        }
    }

    auto* h = new hodlr_handle();
    h->device = device;
    h->depth = depth;
    h->L = L;
    h->rank = g;
    h->nranks = P;
    h->leaf_fmt = d->leaf_fmt;
    h->n_global = d->n;
    const int64_t lf0 = (int64_t)g << (depth - L), lf1 = (int64_t)(g + 1) << (depth - L);
    h->row0 = bd[lf0];
    h->n_local = bd[lf1] - bd[lf0];

    // ---- leaves and chunks
    struct Col { int fmt; ColumnSrc src; int c; int64_t nrows; };
    int64_t seg_elems[kNumFormats] = {0, 0, 0, 0, 0};
    int64_t leaf_elems = 0;
    for (int64_t lf = lf0; lf < lf1; ++lf) {
        LeafDesc L_{};
        L_.row0 = (int32_t)(bd[lf] - h->row0);
        L_.m = (int32_t)(bd[lf + 1] - bd[lf]);
        L_.ld = (int32_t)round_up(L_.m, elems_per_16B(d->leaf_fmt));
        L_.fmt = d->leaf_fmt;
        L_.off = leaf_elems;  // elements for now
        leaf_elems += (int64_t)L_.m * L_.ld;
        h->leaves.push_back(L_);
        h->matrix_bytes += (int64_t)L_.m * L_.m * fmt_bytes(d->leaf_fmt);
        for (int r = 0; r < L_.m; r += kChunkRows) {
            ChunkDesc c{};
            c.row0 = L_.row0 + r;
            c.nrows = std::min(kChunkRows, L_.m - r);
            c.leaf = (int32_t)(lf - lf0);
            h->chunks.push_back(c);
            h->max_chunk_rows = std::max(h->max_chunk_rows, c.nrows);
        }
    }
    // ---- nodes
    std::vector<Col> cols_u, cols_v;  // per node: first column index
    std::vector<int64_t> node_ucol0, node_vcol0;
    std::vector<Col> columns;  // all factor columns in layout order
    h->node_id.assign(depth + 1, {});
    std::vector<int64_t> ext_slot_of_level(depth + 1, -1);
    int64_t ext_count = 0;
    std::vector<int64_t> node_j;  // tree index j of every node
    for (int k = 1; k <= L; ++k) {  // external levels: slot per level, max rank over nodes
        int64_t rmax = 0;
        for (int64_t i = 0; i < (int64_t(1) << (k - 1)); ++i)
            for (int lo = 0; lo < 2; ++lo) rmax = std::max<int64_t>(rmax, d->factors[fidx(k, i, lo)].rank);
        ext_slot_of_level[k] = ext_count;
        ext_count += rmax;
    }
    h->ext_count = ext_count;

    for (int k = 1; k <= depth; ++k) {
        h->node_id[k].assign(size_t(1) << k, -1);
        int64_t j0, j1;
        if (k <= L) {
            j0 = (int64_t)g >> (L - k);
            j1 = j0 + 1;
        } else {
            j0 = lf0 >> (depth - k);
            j1 = ((lf1 - 1) >> (depth - k)) + 1;
        }
        for (int64_t j = j0; j < j1; ++j) {
            int64_t a, b;
            node_rows(k, j, &a, &b);
            int64_t sa = std::max(a, h->row0), sb = std::min(b, h->row0 + h->n_local);
            int64_t i = j >> 1;
            bool first = (j & 1) == 0;
            // U of the block whose rows are node j; V' of the block whose cols are node j
            const hodlr_factor_in& fu = d->factors[fidx(k, i, first ? 0 : 1)];
            const hodlr_factor_in& fv = d->factors[fidx(k, i, first ? 1 : 0)];
            NodeDesc nd{};
            nd.level = k;
            nd.ru = fu.rank;
            nd.rv = fv.rank;
            nd.u_fmt = fu.fmt;
            nd.v_fmt = fv.fmt;
            nd.row0 = (int32_t)(sa - h->row0);
            nd.nrows = (int32_t)(sb - sa);
            nd.u_ld = (int32_t)round_up(nd.nrows, elems_per_16B(fu.fmt));
            nd.v_ld = (int32_t)round_up(nd.nrows, elems_per_16B(fv.fmt));
            nd.u_off = seg_elems[fu.fmt];
            seg_elems[fu.fmt] += (int64_t)nd.ru * nd.u_ld;
            nd.v_off = seg_elems[fv.fmt];
            seg_elems[fv.fmt] += (int64_t)nd.rv * nd.v_ld;
            for (int c = 0; c < nd.ru; ++c)
                columns.push_back({fu.fmt, {fu.U, fu.u_rs, fu.u_cs, sa - a}, c, nd.nrows});
            for (int c = 0; c < nd.rv; ++c)
                columns.push_back({fv.fmt, {fv.V, fv.v_rs, fv.v_cs, sa - a}, c, nd.nrows});
            nd.ext_slot = k <= L ? (int32_t)ext_slot_of_level[k] : -1;
            h->node_id[k][j] = (int)h->nodes.size();
            h->nodes.push_back(nd);
            node_j.push_back(j);
        }
    }
    // storage_bits restricted to local rows: every factor element belongs to
    // exactly one (node, row) of U or V'.
    for (const NodeDesc& nd : h->nodes)
        h->matrix_bytes += (int64_t)nd.nrows * ((int64_t)nd.ru * fmt_bytes(nd.u_fmt) +
                                                (int64_t)nd.rv * fmt_bytes(nd.v_fmt));
    // chunk ranges per node, partial / coefficient offsets
    const int nlev = depth;
    h->chunk_nodes.assign(h->chunks.size() * (size_t)nlev, -1);
    for (size_t ci = 0; ci < h->chunks.size(); ++ci) {
        int64_t grow = h->row0 + h->chunks[ci].row0;
        for (int k = 1; k <= depth; ++k) {
            // node containing this row at level k
            int64_t lf = lf0 + h->chunks[ci].leaf;
            int64_t j = lf >> (depth - k);
            int id = h->node_id[k][j];
            (void)grow;
            h->chunk_nodes[ci * nlev + (k - 1)] = id;
            NodeDesc& nd = h->nodes[id];
            if (nd.nchunk == 0) nd.chunk0 = (int32_t)ci;
            nd.nchunk++;
        }
    }
    int64_t part = 0, tcount = 0;
    for (NodeDesc& nd : h->nodes) {
        nd.part_off = part;
        part += (int64_t)nd.rv * nd.nchunk;
        if (nd.ext_slot < 0) {
            nd.t_off = tcount;
            tcount += nd.rv;
        } else {
            nd.t_off = -1;
        }
    }
    for (size_t id = 0; id < h->nodes.size(); ++id) {
        NodeDesc& nd = h->nodes[id];
        if (nd.ext_slot < 0) {
            // sibling is local (levels > L stay inside this rank's subtree)
            int k = nd.level;
            int sib = h->node_id[k][node_j[id] ^ 1];
            nd.tsrc_off = h->nodes[sib].t_off;
        } else {
            int k = nd.level;
            int64_t j = (int64_t)g >> (L - k);
            int64_t sib = j ^ 1;
            ExtDesc e{};
            e.slot = (int32_t)nd.ext_slot;
            e.rank = nd.ru;
            e.g0 = (int32_t)(sib << (L - k));
            e.g1 = (int32_t)((sib + 1) << (L - k));
            e.tdst = tcount;
            nd.tsrc_off = tcount;
            tcount += nd.ru;
            h->ext.push_back(e);
        }
    }
    h->part_count = part;
    h->t_count = tcount;
    for (int k = 1; k <= L; ++k)  // kernels_shard.cu relies on external nodes being ids 0..L-1
        if (h->nodes[k - 1].level != k || h->nodes[k - 1].ext_slot < 0) {
            delete h;
            return fail(HODLR_ERR_INVALID, "internal: external node order");
        }

    // ---- arena layout: [leaves][q52][bf16][fp16][fp32][fp64], 256-B aligned
    int64_t seg_byte_off[kNumFormats];
    size_t off = round_up(leaf_elems * fmt_bytes(d->leaf_fmt), kAlign);
    for (int f = 0; f < kNumFormats; ++f) {
        seg_byte_off[f] = (int64_t)off;
        off += round_up(seg_elems[f] * fmt_bytes(f), kAlign);
    }
    // + slack: 4-element vector loads at a column's ragged end may touch up to
    // 15 elements past it (the values are masked, the addresses must be valid)
    h->arena_bytes = std::max<size_t>(off, kAlign) + kAlign;
    for (LeafDesc& l : h->leaves) l.off *= fmt_bytes(d->leaf_fmt);
    for (NodeDesc& nd : h->nodes) {
        nd.u_off = seg_byte_off[nd.u_fmt] + nd.u_off * fmt_bytes(nd.u_fmt);
        nd.v_off = seg_byte_off[nd.v_fmt] + nd.v_off * fmt_bytes(nd.v_fmt);
    }

    // ---- device allocation and packing
    auto cleanup = [&](hodlr_status st) {
        h->arena.release();
        h->tables.release();
        delete h;
        return st;
    };
    cudaError_t ce = cudaSetDevice(device);
    if (ce != cudaSuccess) return cleanup(fail(HODLR_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(ce)));
    ce = h->arena.ensure(h->arena_bytes);
    if (ce != cudaSuccess) return cleanup(fail(HODLR_ERR_CUDA, std::string("arena allocation: ") + cudaGetErrorString(ce)));
    ce = cudaMemset(h->arena.p, 0, h->arena_bytes);
    if (ce != cudaSuccess) return cleanup(fail(HODLR_ERR_CUDA, cudaGetErrorString(ce)));
    const size_t cap = size_t(1) << 24;  // 16 M doubles staged per flush
    double* stage = nullptr;
    ce = cudaMalloc(&stage, cap * sizeof(double));
    if (ce != cudaSuccess) return cleanup(fail(HODLR_ERR_CUDA, std::string("staging allocation: ") + cudaGetErrorString(ce)));
    uint8_t* A = (uint8_t*)h->arena.p;
    {
        SegmentWriter w(d->leaf_fmt, A, stage, cap);
        for (size_t li = 0; li < h->leaves.size(); ++li) {
            const LeafDesc& l = h->leaves[li];
            const double* src = d->leaves[lf0 + li];
            int64_t ld = d->leaf_ld[lf0 + li];
            if (!src || ld < l.m) {
                cudaFree(stage);
                return cleanup(fail(HODLR_ERR_INVALID, "bad leaf pointer or stride"));
            }
            for (int r = 0; r < l.m; ++r) {
                for (int c = 0; c < l.m; ++c)
                    w.put(payload_at(src, enc ? d->leaf_fmt : HODLR_FMT_FP64, (int64_t)r * ld + c));
                for (int c = l.m; c < l.ld; ++c) w.put(0.0);
            }
        }
        w.flush();
        if (w.err != cudaSuccess) {
            cudaFree(stage);
            return cleanup(fail(HODLR_ERR_CUDA, std::string("leaf packing: ") + cudaGetErrorString(w.err)));
        }
    }
    for (int f = 0; f < kNumFormats; ++f) {
        if (seg_elems[f] == 0) continue;
        SegmentWriter w(f, A + seg_byte_off[f], stage, cap);
        // columns of format f in the order their offsets were assigned
        for (const Col& col : columns) {
            if (col.fmt != f) continue;
            int64_t ld = round_up(col.nrows, elems_per_16B(f));
            for (int64_t r = 0; r < col.nrows; ++r)
                w.put(payload_at(col.src.base, enc ? f : HODLR_FMT_FP64,
                                 (col.src.r0 + r) * col.src.rs + (int64_t)col.c * col.src.cs));
            for (int64_t r = col.nrows; r < ld; ++r) w.put(0.0);
        }
        w.flush();
        if (w.err != cudaSuccess) {
            cudaFree(stage);
            return cleanup(fail(HODLR_ERR_CUDA, std::string("factor packing: ") + cudaGetErrorString(w.err)));
        }
        if (w.position() != seg_elems[f]) {
            cudaFree(stage);
            return cleanup(fail(HODLR_ERR_INVALID, "internal: segment size mismatch"));
        }
    }
    cudaFree(stage);

    // ---- tables
    size_t tb = 0;
    auto place = [&](size_t bytes) { size_t o = tb; tb = round_up(tb + bytes, 64); return o; };
    size_t o_nodes = place(h->nodes.size() * sizeof(NodeDesc));
    size_t o_chunks = place(h->chunks.size() * sizeof(ChunkDesc));
    size_t o_cn = place(h->chunk_nodes.size() * sizeof(int32_t));
    size_t o_leaves = place(h->leaves.size() * sizeof(LeafDesc));
    size_t o_ext = place(h->ext.size() * sizeof(ExtDesc));
    ce = h->tables.ensure(std::max<size_t>(tb, 64));
    if (ce != cudaSuccess) return cleanup(fail(HODLR_ERR_CUDA, cudaGetErrorString(ce)));
    uint8_t* T = (uint8_t*)h->tables.p;
    auto up = [&](size_t o, const void* src, size_t bytes) {
        return bytes ? cudaMemcpy(T + o, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    ce = up(o_nodes, h->nodes.data(), h->nodes.size() * sizeof(NodeDesc));
    if (ce == cudaSuccess) ce = up(o_chunks, h->chunks.data(), h->chunks.size() * sizeof(ChunkDesc));
    if (ce == cudaSuccess) ce = up(o_cn, h->chunk_nodes.data(), h->chunk_nodes.size() * sizeof(int32_t));
    if (ce == cudaSuccess) ce = up(o_leaves, h->leaves.data(), h->leaves.size() * sizeof(LeafDesc));
    if (ce == cudaSuccess) ce = up(o_ext, h->ext.data(), h->ext.size() * sizeof(ExtDesc));
    if (ce != cudaSuccess) return cleanup(fail(HODLR_ERR_CUDA, cudaGetErrorString(ce)));

    PlanView& v = h->view;
    v.arena = A;
    v.nodes = (const NodeDesc*)(T + o_nodes);
    v.chunks = (const ChunkDesc*)(T + o_chunks);
    v.chunk_nodes = (const int32_t*)(T + o_cn);
    v.leaves = (const LeafDesc*)(T + o_leaves);
    v.ext = (const ExtDesc*)(T + o_ext);
    v.nnodes = (int32_t)h->nodes.size();
    v.nchunks = (int32_t)h->chunks.size();
    v.nlev = nlev;
    v.nleaves = (int32_t)h->leaves.size();
    v.next = (int32_t)h->ext.size();
    v.n_local = (int32_t)h->n_local;
    v.part_count = h->part_count;
    v.t_count = h->t_count;
    v.ext_count = h->ext_count;

    {
        MrInput mi{&h->view, (const uint8_t*)h->arena.p, L, &h->nodes, &h->chunks, &h->leaves, &h->chunk_nodes, nlev,
                   d->leaf_fmt, device, h->ext_count};
        if (mr_prepare(mi, h->mr) != HODLR_OK) return cleanup(fail(HODLR_ERR_CUDA, "multi-RHS plan upload failed"));
        const char* no_mr = getenv("HODLR_B200_DISABLE_MRHS");
        if (no_mr && no_mr[0] == '1') mr_release(h->mr);
    }
    const char* no_sv = getenv("HODLR_B200_DISABLE_FUSED");
    if (!(no_sv && no_sv[0] == '1')) {
        // sharded handles: the fused kernel runs the rank's subtree (levels
        // L+1..l renumbered 1..l-L); external levels run in kernels_shard.cu
        std::vector<NodeDesc> sub;
        for (const NodeDesc& nd : h->nodes)
            if (nd.level > L) {
                sub.push_back(nd);
                sub.back().level -= L;
            }
        // geometry 1 (4 CTAs per SM) for binary32-working matrices; HODLR_B200_SV_GEO=0/1 overrides
        int geo = h->leaf_fmt == HODLR_FMT_FP32 ? 1 : 0;
        if (const char* g = getenv("HODLR_B200_SV_GEO")) geo = atoi(g) == 1 ? 1 : 0;
        SvInput si{&sub, &h->chunks, &h->leaves, &h->chunk_nodes, depth - L, (const uint8_t*)h->arena.p,
                   h->arena_bytes, geo};
        hodlr_status st = sv_prepare(si, h->sv, &h->sv_ok);
        if (st != HODLR_OK) return cleanup(st);
        if (h->sv_ok && P > 1) {
            // leave a few SMs to the all-gather kernel that overlaps the
            // subtree (the persistent kernel would otherwise hold every SM)
            int sms = 148, reserve = 4;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
            if (const char* r = getenv("HODLR_B200_SHARD_RESERVE_SMS")) reserve = atoi(r);
            reserve = std::max(0, std::min(reserve, sms - 1));
            sv_set_grid(h->sv, h->sv.ctas_per_sm * (sms - reserve));
        }
    }
    *out = h;
    return HODLR_OK;
}

// Workspace: [fused-path sync state (fixed offset 0, must start zeroed)]
//            [partials: part_count*s][coefficients: t_count*s]
//            [sharded only: k_ext_v per-block partials | discarded send | ticket]
// partial sums: the generic layout or the multi-RHS slot layout, whichever is larger
int64_t part_elems(const hodlr_handle* h, int64_t s) {
    return std::max<int64_t>(h->part_count * s, h->mr.ok ? mr_part_elems(h->mr, s) : 0);
}
template <typename W>
size_t ext_ws_bytes(const hodlr_handle* h, int64_t s) {
    if (h->nranks == 1 || h->ext_count == 0) return 0;
    return (size_t)round_up((int64_t)ext_v_blocks(h->n_local) * h->ext_count * s * sizeof(W), kAlign) +
           (size_t)round_up(h->ext_count * s * sizeof(W), kAlign) + kAlign;
}
template <typename W>
size_t ws_bytes_for(const hodlr_handle* h, int64_t s) {
    return (size_t)round_up((int64_t)sv_extra_ws(h->sv, s), kAlign) +
           (size_t)round_up(part_elems(h, s) * sizeof(W), kAlign) +
           (size_t)round_up((h->t_count * s) * sizeof(W), kAlign) + ext_ws_bytes<W>(h, s);
}

// narrow working formats (q52 / bf16 / fp16) run the strict-order kernels
// (kernels_seq.cu) on binary64 carriers
bool narrow_working(int working) { return working >= HODLR_FMT_Q52 && working <= HODLR_FMT_FP16; }
int working_bytes(int working) { return working == HODLR_FMT_FP32 ? 4 : 8; }
// workspace of a strict-order call: coefficients + the rounded copy of x
size_t seq_ws_bytes(const hodlr_handle* h, int64_t s) {
    return (size_t)round_up(h->t_count * s * 8, kAlign) + (size_t)round_up(h->n_local * s * 8, kAlign);
}

template <typename W>
void carve(const hodlr_handle* h, int64_t s, void* ws, W** partial, W** tbuf, void** extra) {
    uint8_t* p = (uint8_t*)ws;
    *extra = p;
    p += round_up((int64_t)sv_extra_ws(h->sv, s), kAlign);
    *partial = (W*)p;
    p += round_up(part_elems(h, s) * sizeof(W), kAlign);
    *tbuf = (W*)p;
}

template <typename W>
struct ExtWs {
    W* scratch;
    W* dummy_send;
    unsigned* ticket;
};
template <typename W>
ExtWs<W> carve_ext(const hodlr_handle* h, int64_t s, void* ws) {
    uint8_t* p = (uint8_t*)ws + ws_bytes_for<W>(h, s) - ext_ws_bytes<W>(h, s);
    ExtWs<W> e;
    e.scratch = (W*)p;
    p += round_up((int64_t)ext_v_blocks(h->n_local) * h->ext_count * s * sizeof(W), kAlign);
    e.dummy_send = (W*)p;
    p += round_up(h->ext_count * s * sizeof(W), kAlign);
    e.ticket = (unsigned*)p;
    return e;
}

hodlr_status check_working(int working, bool allow_narrow = false) {
    if (working == HODLR_FMT_FP64 || working == HODLR_FMT_FP32) return HODLR_OK;
    if (narrow_working(working)) {
        if (allow_narrow) return HODLR_OK;
        return fail(HODLR_ERR_UNSUPPORTED,
                    "sharded matvec: working precision must be fp64 or fp32 (bf16/fp16/q52 working run unsharded)");
    }
    return fail(HODLR_ERR_INVALID, "unknown working format code");
}

hodlr_status resolve_ws(hodlr_handle* h, int working, int64_t s, void** ws, size_t ws_bytes, void* stream,
                        bool strict = false) {
    size_t need = working == HODLR_FMT_FP32 ? ws_bytes_for<float>(h, s) : ws_bytes_for<double>(h, s);
    // strict-order calls: the fused kernel's sync header stays untouched at the
    // front (the workspace may be shared with fast calls on the same stream)
    if (strict || narrow_working(working))
        need = (size_t)round_up((int64_t)sv_extra_ws(h->sv, s), kAlign) + seq_ws_bytes(h, s);
    if (*ws) {
        if (ws_bytes < need) return fail(HODLR_ERR_INVALID, "workspace too small");
        return HODLR_OK;
    }
    std::lock_guard<std::mutex> lock(h->ws_mu);
    hodlr_handle::StreamWs* w = nullptr;
    for (auto& e : h->ws)
        if (e.stream == stream) w = &e;
    if (!w) {
        h->ws.push_back(hodlr_handle::StreamWs{stream, DeviceBuf{}});
        w = &h->ws.back();
    }
    if (w->buf.bytes < need) {
        // (growing: cudaFree waits for the device, so earlier calls on this
        // stream are done with the old buffer; the zeroing is ordered on the
        // caller's stream before the call's kernels)
        CUDA_TRY(cudaSetDevice(h->device));
        cudaError_t e = w->buf.ensure(std::max<size_t>(need, kAlign));
        if (e == cudaSuccess) e = cudaMemsetAsync(w->buf.p, 0, w->buf.bytes, (cudaStream_t)stream);
        if (e != cudaSuccess) return fail(HODLR_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(e));
    }
    *ws = w->buf.p;
    return HODLR_OK;
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <typename W>
hodlr_status run_local(hodlr_handle* h, const W* x, int64_t ldx, W* b, int64_t ldb, int64_t s,
                       void* ws, cudaStream_t st) {
    W *partial, *tbuf;
    void* extra;
    carve<W>(h, s, ws, &partial, &tbuf, &extra);
    cudaError_t e;
    if (h->sv_ok && s == 1 && ldx == 1 && ldb == 1 && h->nranks == 1 && aligned16(x) && aligned16(b)) {
        e = sv_matvec<W>(h->view, h->sv, x, b, partial, tbuf, extra, st);
    } else if (h->nranks == 1 && mr_usable(h->mr, sizeof(W) == 8 ? HODLR_FMT_FP64 : HODLR_FMT_FP32)) {
        e = mr_matvec<W>(h->view, h->mr, 0, x, ldx, b, ldb, s, partial, tbuf, st);
    } else {
        e = gen_begin<W>(h->view, x, ldx, s, partial, tbuf, nullptr, st);
        if (e == cudaSuccess) e = gen_end<W>(h->view, x, ldx, tbuf, b, ldb, s, h->max_chunk_rows, st);
    }
    if (e != cudaSuccess) return fail(HODLR_ERR_CUDA, std::string("matvec launch: ") + cudaGetErrorString(e));
    return HODLR_OK;
}

// Strict-order path (kernels_seq.cu): x and b are binary64 carriers; x is
// rounded to `working` into the workspace first.
hodlr_status run_seq(hodlr_handle* h, int working, const double* x, int64_t ldx, double* b, int64_t ldb, int64_t s,
                     void* ws, cudaStream_t st) {
    uint8_t* p = (uint8_t*)ws + round_up((int64_t)sv_extra_ws(h->sv, s), kAlign);
    double* tbuf = (double*)p;
    double* xr = (double*)(p + round_up(h->t_count * s * 8, kAlign));
    cudaError_t e = cudaSuccess;
    if (working != HODLR_FMT_FP64) {
        e = seq_round(working, x, xr, h->n_local, s, ldx, s, st);
        x = xr;
        ldx = s;
    }
    if (e == cudaSuccess) e = seq_matvec(working, h->view, x, ldx, b, ldb, s, tbuf, st);
    if (e != cudaSuccess) return fail(HODLR_ERR_CUDA, std::string("strict matvec launch: ") + cudaGetErrorString(e));
    return HODLR_OK;
}

// the single-vector fused kernel runs a rank's subtree (its own phase A)
bool shard_sv_local(const hodlr_handle* h, int64_t s, int64_t ldx) { return h->sv_ok && s == 1 && ldx == 1; }
// (shard_local falls back to the generic kernels for unaligned single vectors:
// the same choice as run_local)

template <typename W>
cudaError_t shard_local_impl(hodlr_handle* h, const W* x, int64_t ldx, W* b, int64_t ldb, int64_t s, void* ws,
                             cudaStream_t st) {
    W *partial, *tbuf;
    void* extra;
    carve<W>(h, s, ws, &partial, &tbuf, &extra);
    if (h->sv_ok && s == 1 && ldx == 1 && ldb == 1 && aligned16(x) && aligned16(b))
        return sv_matvec<W>(h->view, h->sv, x, b, partial, tbuf, extra, st);
    // multi-RHS kernels over the subtree levels (L+1..l) and the leaves; the
    // external levels are added by shard_end.  With fragment slabs, shard_begin
    // already ran phase A (all levels): only phase B is left.
    const int wf = sizeof(W) == 8 ? HODLR_FMT_FP64 : HODLR_FMT_FP32;
    if (!shard_sv_local(h, s, ldx) && mr_slab_begin_usable(h->mr, wf))
        return cudaSuccess;  // slab path: phase B (every level) runs in shard_end, after the exchange
    if (mr_usable(h->mr, wf)) return mr_matvec<W>(h->view, h->mr, h->L, x, ldx, b, ldb, s, partial, tbuf, st);
    // generic: the whole local plan with the external coefficients set to 0
    // (their products add exact zeros); the external partials go to a
    // discarded buffer, shard_begin owns the real ones.
    W* dummy = h->ext_count ? carve_ext<W>(h, s, ws).dummy_send : nullptr;
    cudaError_t e = gen_begin<W>(h->view, x, ldx, s, partial, tbuf, dummy, st);
    for (const ExtDesc& x_ : h->ext)
        if (e == cudaSuccess && x_.rank > 0)
            e = cudaMemsetAsync(tbuf + x_.tdst * s, 0, (size_t)x_.rank * s * sizeof(W), st);
    if (e == cudaSuccess) e = gen_end<W>(h->view, x, ldx, tbuf, b, ldb, s, h->max_chunk_rows, st);
    return e;
}

}  // namespace

extern "C" {

int32_t hodlr_abi_version(void) { return HODLR_B200_ABI_VERSION; }
const char* hodlr_last_error(void) { return g_err.c_str(); }

hodlr_status hodlr_create(const hodlr_desc* d, int32_t device, hodlr_handle** out) {
    return build(d, device, hodlr_shard{0, 1}, out);
}
hodlr_status hodlr_create_sharded(const hodlr_desc* d, int32_t device, hodlr_shard shard,
                                  hodlr_handle** out) {
    return build(d, device, shard, out);
}

hodlr_status hodlr_destroy(hodlr_handle* h) {
    if (!h) return HODLR_OK;
    cudaSetDevice(h->device);
    h->arena.release();
    h->tables.release();
    for (auto& w : h->ws) w.buf.release();
    for (auto& c : h->hctx) {
        c.e2e.release();
        if (c.copy_stream) cudaStreamDestroy(c.copy_stream);
        for (cudaEvent_t e : c.slice_ev) cudaEventDestroy(e);
        if (c.h2d_ev) cudaEventDestroy(c.h2d_ev);
    }
    sv_release(h->sv);
    mr_release(h->mr);
    delete h;
    return HODLR_OK;
}

hodlr_status hodlr_matvec_path(const hodlr_handle* h, int32_t working, int64_t s, int32_t* path,
                               int32_t* launches) {
    if (!h || !path || !launches || s < 1) return fail(HODLR_ERR_INVALID, "bad arguments");
    hodlr_status st = check_working(working, true);
    if (st != HODLR_OK) return st;
    if (narrow_working(working)) {
        *path = HODLR_PATH_STRICT;
        *launches = 3;
    } else if (h->sv_ok && s == 1) {
        *path = HODLR_PATH_FUSED_SV;
        *launches = sv_launches(h->sv);
    } else if (mr_usable(h->mr, working)) {
        const bool slab = h->nranks > 1 ? mr_slab_begin_usable(h->mr, working) : mr_slab_used(h->mr, working, h->L);
        *path = slab ? HODLR_PATH_MRHS_SLAB : HODLR_PATH_MRHS;
        if (slab && working == HODLR_FMT_FP32 && tc_usable(h->mr, s)) *path = HODLR_PATH_MRHS_TC;
        *launches = mr_launches();
    } else {
        *path = HODLR_PATH_GENERIC;
        *launches = 3;
    }
    return HODLR_OK;
}

hodlr_status hodlr_workspace_size(const hodlr_handle* h, int64_t s, size_t* bytes) {
    if (!h || !bytes || s < 1) return fail(HODLR_ERR_INVALID, "bad arguments");
    *bytes = ws_bytes_for<double>(h, s);
    return HODLR_OK;
}

hodlr_status hodlr_matvec(hodlr_handle* h, int32_t working, const void* x, int64_t ldx, void* b,
                          int64_t ldb, int64_t s, void* ws, size_t ws_bytes, void* stream) {
    if (!h) return fail(HODLR_ERR_INVALID, "null handle");
    if (h->nranks != 1) return fail(HODLR_ERR_INVALID, "sharded handle: use hodlr_matvec_shard_begin/end");
    hodlr_status stc = check_working(working, true);
    if (stc != HODLR_OK) return stc;
    if (s < 1 || ldx < s || ldb < s) return fail(HODLR_ERR_INVALID, "need s >= 1, ldx >= s, ldb >= s");
    if (!x || !b) return fail(HODLR_ERR_INVALID, "null x or b");
    hodlr_status r = resolve_ws(h, working, s, &ws, ws_bytes, stream);
    if (r != HODLR_OK) return r;
    cudaStream_t st = (cudaStream_t)stream;
    if (narrow_working(working)) return run_seq(h, working, (const double*)x, ldx, (double*)b, ldb, s, ws, st);
    if (working == HODLR_FMT_FP64)
        return run_local<double>(h, (const double*)x, ldx, (double*)b, ldb, s, ws, st);
    return run_local<float>(h, (const float*)x, ldx, (float*)b, ldb, s, ws, st);
}

hodlr_status hodlr_matvec_strict(hodlr_handle* h, int32_t working, const double* x, int64_t ldx, double* b,
                                 int64_t ldb, int64_t s, void* ws, size_t ws_bytes, void* stream) {
    if (!h) return fail(HODLR_ERR_INVALID, "null handle");
    if (h->nranks != 1) return fail(HODLR_ERR_INVALID, "strict-order matvec needs an unsharded handle");
    hodlr_status stc = check_working(working, true);
    if (stc != HODLR_OK) return stc;
    if (s < 1 || ldx < s || ldb < s) return fail(HODLR_ERR_INVALID, "need s >= 1, ldx >= s, ldb >= s");
    if (!x || !b) return fail(HODLR_ERR_INVALID, "null x or b");
    hodlr_status r = resolve_ws(h, working, s, &ws, ws_bytes, stream, true);
    if (r != HODLR_OK) return r;
    return run_seq(h, working, x, ldx, b, ldb, s, ws, (cudaStream_t)stream);
}

hodlr_status hodlr_workspace_size_for(const hodlr_handle* h, int32_t working, int32_t strict, int64_t s,
                                      size_t* bytes) {
    if (!h || !bytes || s < 1) return fail(HODLR_ERR_INVALID, "bad arguments");
    hodlr_status stc = check_working(working, true);
    if (stc != HODLR_OK) return stc;
    if (strict || narrow_working(working))
        *bytes = (size_t)round_up((int64_t)sv_extra_ws(h->sv, s), kAlign) + seq_ws_bytes(h, s);
    else
        *bytes = working == HODLR_FMT_FP32 ? ws_bytes_for<float>(h, s) : ws_bytes_for<double>(h, s);
    return HODLR_OK;
}

hodlr_status hodlr_matvec_host(hodlr_handle* h, int32_t working, const double* x_host,
                               double* b_host, int64_t s, void* stream) {
    if (!h) return fail(HODLR_ERR_INVALID, "null handle");
    if (h->nranks != 1) return fail(HODLR_ERR_INVALID, "host-buffer matvec needs an unsharded handle");
    hodlr_status stc = check_working(working, true);
    if (stc != HODLR_OK) return stc;
    if (s < 1 || !x_host || !b_host) return fail(HODLR_ERR_INVALID, "bad arguments");
    // take a free staging context (released on every return path)
    struct CtxLease {
        hodlr_handle* h;
        hodlr_handle::HostCtx* c = nullptr;
        bool contended = false;  // another host-buffer call is in flight on this handle
        explicit CtxLease(hodlr_handle* hh) : h(hh) {
            std::unique_lock<std::mutex> lk(h->mu);
            h->hcv.wait(lk, [&] {
                for (auto& x : h->hctx)
                    if (!x.busy) return true;
                return false;
            });
            for (auto& x : h->hctx)
                if (!x.busy) {
                    c = &x;
                    break;
                }
            c->busy = true;
            for (auto& x : h->hctx)
                if (x.busy && &x != c) contended = true;
        }
        ~CtxLease() {
            {
                std::lock_guard<std::mutex> lk(h->mu);
                c->busy = false;
            }
            h->hcv.notify_one();
        }
    } lease(h);
    hodlr_handle::HostCtx& hc = *lease.c;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = h->n_local;
    const int wb = working_bytes(working);
    size_t xb = round_up(n * s * 8, kAlign), wbytes = round_up(n * s * wb, kAlign);
    size_t need = 2 * xb + 2 * wbytes;
    CUDA_TRY(cudaSetDevice(h->device));
    CUDA_TRY(hc.e2e.ensure(need));
    uint8_t* base = (uint8_t*)hc.e2e.p;
    double* xd = (double*)base;
    double* bd = (double*)(base + xb);
    void* xw = base + 2 * xb;
    void* bw = base + 2 * xb + wbytes;
    void* ws = nullptr;
    hodlr_status r = resolve_ws(h, working, s, &ws, 0, stream);
    if (r != HODLR_OK) return r;
    // A pinned (page-locked, UVA-mapped) host b is written by the kernels
    // directly where each element is stored once: the widening kernel (fp32
    // working) and the fused single-vector kernel (fp64 working, b rows written
    // once as the U pieces finish, so the PCIe writes overlap the kernel's tail).
    // Saves the D2H copy-engine pass (cfg2 e2e 78 -> 68 us); pageable buffers go
    // through the staging copy.
    auto mapped = [](const void* hp) -> void* {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, hp) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
    };
    // x in: ordered after the previous call's host-to-device copy (see hodlr_handle::last_h2d)
    // (a lone caller needs no ordering and records no event)
    auto copy_x_in = [&](double* dst) -> cudaError_t {
        std::lock_guard<std::mutex> lk(h->h2d_mu);
        if (!lease.contended) {
            h->last_h2d = nullptr;
            return cudaMemcpyAsync(dst, x_host, n * s * 8, cudaMemcpyHostToDevice, st);
        }
        cudaError_t e = cudaSuccess;
        if (!hc.h2d_ev) e = cudaEventCreateWithFlags(&hc.h2d_ev, cudaEventDisableTiming);
        if (e == cudaSuccess && h->last_h2d && h->last_h2d != hc.h2d_ev) e = cudaStreamWaitEvent(st, h->last_h2d, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dst, x_host, n * s * 8, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(hc.h2d_ev, st);
        if (e == cudaSuccess) h->last_h2d = hc.h2d_ev;
        return e;
    };
    const bool zc = !getenv("HODLR_B200_NO_ZEROCOPY");
    double* b_map = zc ? (double*)mapped(b_host) : nullptr;
    if (narrow_working(working)) {
        CUDA_TRY(copy_x_in(xd));
        r = run_seq(h, working, xd, s, bd, s, s, ws, st);
        if (r != HODLR_OK) return r;
        b_map = nullptr;
    } else if (working == HODLR_FMT_FP64 && mr_sliceable(h->mr, working, s) && !(h->sv_ok && s == 1) &&
               n * s * 8 >= (int64_t(8) << 20) && !getenv("HODLR_B200_NO_E2E_PIPELINE")) {
        // Multi-RHS slab path with a large result (cfg4: 134 MB each way): phase A +
        // reduce once, then phase B over row ranges; each finished range is copied out
        // on a second stream while the next ranges are computed, so only the first
        // range's kernel time stays in front of the 2.4 ms device-to-host copy.
        CUDA_TRY(copy_x_in(xd));
        double *partial, *tbuf;
        void* extra;
        carve<double>(h, s, ws, &partial, &tbuf, &extra);
        CUDA_TRY(mr_phase_a(h->view, h->mr, xd, s, s, partial, tbuf, st));
        const int nch = h->view.nchunks;
        const int nsl = std::max(1, std::min(8, nch / 64));
        if (!hc.copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&hc.copy_stream, cudaStreamNonBlocking));
        while ((int)hc.slice_ev.size() < nsl) {
            cudaEvent_t ev;
            CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            hc.slice_ev.push_back(ev);
        }
        for (int i = 0; i < nsl; ++i) {
            const int c0 = (int)((int64_t)i * nch / nsl), c1 = (int)((int64_t)(i + 1) * nch / nsl);
            CUDA_TRY(mr_phase_b_range(h->view, h->mr, xd, s, bd, s, s, tbuf, c0, c1, st));
            CUDA_TRY(cudaEventRecord(hc.slice_ev[i], st));
            CUDA_TRY(cudaStreamWaitEvent(hc.copy_stream, hc.slice_ev[i], 0));
            const int64_t r0 = h->chunks[c0].row0, r1 = c1 < nch ? h->chunks[c1].row0 : n;
            CUDA_TRY(cudaMemcpyAsync(b_host + r0 * s, bd + r0 * s, (size_t)(r1 - r0) * s * 8, cudaMemcpyDeviceToHost,
                                     hc.copy_stream));
        }
        CUDA_TRY(cudaStreamSynchronize(hc.copy_stream));
        CUDA_TRY(cudaStreamSynchronize(st));
        return HODLR_OK;
    } else if (working == HODLR_FMT_FP64) {
        CUDA_TRY(copy_x_in(xd));
        if (!(h->sv_ok && s == 1) || ((uintptr_t)b_map & 15)) b_map = nullptr;  // multi-pass writers / unaligned: stage in HBM
        r = run_local<double>(h, xd, s, b_map ? b_map : bd, s, s, ws, st);
        if (r != HODLR_OK) return r;
    } else {
        // (x is still staged by the copy engine: one kernel reading 2 MB of mapped
        // host memory measured slower than the copy, cfg5 eps=1e-2 e2e 180 -> 247 us)
        CUDA_TRY(copy_x_in(xd));
        CUDA_TRY(launch_round_in<float>(xd, (float*)xw, n, s, s, s, st));
        r = run_local<float>(h, (const float*)xw, s, (float*)bw, s, s, ws, st);
        if (r != HODLR_OK) return r;
        CUDA_TRY(launch_widen_out<float>((const float*)bw, b_map ? b_map : bd, n, s, s, s, st));
    }
    if (!b_map) CUDA_TRY(cudaMemcpyAsync(b_host, bd, n * s * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return HODLR_OK;
}

hodlr_status hodlr_shard_exchange_count(const hodlr_handle* h, int64_t s, int64_t* count) {
    if (!h || !count || s < 1) return fail(HODLR_ERR_INVALID, "bad arguments");
    *count = h->ext_count * s;
    return HODLR_OK;
}

hodlr_status hodlr_matvec_shard_begin(hodlr_handle* h, int32_t working, const void* x_local,
                                      int64_t ldx, int64_t s, void* send, void* ws,
                                      size_t ws_bytes, void* stream) {
    if (!h) return fail(HODLR_ERR_INVALID, "null handle");
    hodlr_status stc = check_working(working);
    if (stc != HODLR_OK) return stc;
    if (s < 1 || ldx < s || !x_local) return fail(HODLR_ERR_INVALID, "bad x / s");
    if (h->ext_count > 0 && !send) return fail(HODLR_ERR_INVALID, "null send buffer");
    hodlr_status r = resolve_ws(h, working, s, &ws, ws_bytes, stream);
    if (r != HODLR_OK) return r;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if (!shard_sv_local(h, s, ldx) && mr_slab_begin_usable(h->mr, working)) {
        // phase A over every level on the tensor cores: external partials -> send
        if (working == HODLR_FMT_FP64) {
            double *partial, *tbuf;
            void* extra;
            carve<double>(h, s, ws, &partial, &tbuf, &extra);
            e = mr_shard_begin<double>(h->view, h->mr, (const double*)x_local, ldx, s, partial, tbuf, (double*)send, st);
        } else {
            float *partial, *tbuf;
            void* extra;
            carve<float>(h, s, ws, &partial, &tbuf, &extra);
            e = mr_shard_begin<float>(h->view, h->mr, (const float*)x_local, ldx, s, partial, tbuf, (float*)send, st);
        }
    } else if (working == HODLR_FMT_FP64) {
        ExtWs<double> x = carve_ext<double>(h, s, ws);
        e = ext_begin<double>(h->view, (const double*)x_local, ldx, s, x.scratch, x.ticket, (double*)send, st);
    } else {
        ExtWs<float> x = carve_ext<float>(h, s, ws);
        e = ext_begin<float>(h->view, (const float*)x_local, ldx, s, x.scratch, x.ticket, (float*)send, st);
    }
    if (e != cudaSuccess) return fail(HODLR_ERR_CUDA, std::string("shard_begin: ") + cudaGetErrorString(e));
    return HODLR_OK;
}

hodlr_status hodlr_matvec_shard_local(hodlr_handle* h, int32_t working, const void* x_local,
                                      int64_t ldx, void* b_local, int64_t ldb, int64_t s,
                                      void* ws, size_t ws_bytes, void* stream) {
    if (!h) return fail(HODLR_ERR_INVALID, "null handle");
    hodlr_status stc = check_working(working);
    if (stc != HODLR_OK) return stc;
    if (s < 1 || ldx < s || ldb < s || !x_local || !b_local) return fail(HODLR_ERR_INVALID, "bad x / b / s");
    hodlr_status r = resolve_ws(h, working, s, &ws, ws_bytes, stream);
    if (r != HODLR_OK) return r;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = working == HODLR_FMT_FP64
                        ? shard_local_impl<double>(h, (const double*)x_local, ldx, (double*)b_local, ldb, s, ws, st)
                        : shard_local_impl<float>(h, (const float*)x_local, ldx, (float*)b_local, ldb, s, ws, st);
    if (e != cudaSuccess) return fail(HODLR_ERR_CUDA, std::string("shard_local: ") + cudaGetErrorString(e));
    return HODLR_OK;
}

hodlr_status hodlr_matvec_shard_end(hodlr_handle* h, int32_t working, const void* x_local,
                                    int64_t ldx, const void* recv, void* b_local, int64_t ldb,
                                    int64_t s, void* ws, size_t ws_bytes, void* stream) {
    if (!h) return fail(HODLR_ERR_INVALID, "null handle");
    hodlr_status stc = check_working(working);
    if (stc != HODLR_OK) return stc;
    if (s < 1 || ldx < s || ldb < s || !x_local || !b_local) return fail(HODLR_ERR_INVALID, "bad x / b / s");
    if (h->ext_count > 0 && !recv) return fail(HODLR_ERR_INVALID, "null recv buffer");
    hodlr_status r = resolve_ws(h, working, s, &ws, ws_bytes, stream);
    if (r != HODLR_OK) return r;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    const bool slab = !shard_sv_local(h, s, ldx) && mr_slab_begin_usable(h->mr, working);
    if (working == HODLR_FMT_FP64) {
        double *partial, *tbuf;
        void* extra;
        carve<double>(h, s, ws, &partial, &tbuf, &extra);
        if (slab) {
            e = gen_ext<double>(h->view, s, (const double*)recv, tbuf, st);
            if (e == cudaSuccess)
                e = mr_slab_phase_b<double>(h->view, h->mr, (const double*)x_local, ldx, (double*)b_local, ldb, s,
                                            tbuf, st);
        } else {
            e = ext_finish<double>(h->view, s, (const double*)recv, tbuf, (double*)b_local, ldb, st);
        }
    } else {
        float *partial, *tbuf;
        void* extra;
        carve<float>(h, s, ws, &partial, &tbuf, &extra);
        if (slab) {
            e = gen_ext<float>(h->view, s, (const float*)recv, tbuf, st);
            if (e == cudaSuccess)
                e = mr_slab_phase_b<float>(h->view, h->mr, (const float*)x_local, ldx, (float*)b_local, ldb, s,
                                           tbuf, st);
        } else {
            e = ext_finish<float>(h->view, s, (const float*)recv, tbuf, (float*)b_local, ldb, st);
        }
    }
    if (e != cudaSuccess) return fail(HODLR_ERR_CUDA, std::string("shard_end: ") + cudaGetErrorString(e));
    return HODLR_OK;
}

hodlr_status hodlr_quantize(int32_t fmt, const double* src, void* dst, int64_t count, void* stream) {
    if (!valid_fmt(fmt)) return fail(HODLR_ERR_UNSUPPORTED, "unsupported format");
    if (count < 0 || (count > 0 && (!src || !dst))) return fail(HODLR_ERR_INVALID, "bad arguments");
    CUDA_TRY(launch_quantize(fmt, src, dst, count, (cudaStream_t)stream));
    return HODLR_OK;
}
hodlr_status hodlr_dequantize(int32_t fmt, const void* src, double* dst, int64_t count, void* stream) {
    if (!valid_fmt(fmt)) return fail(HODLR_ERR_UNSUPPORTED, "unsupported format");
    if (count < 0 || (count > 0 && (!src || !dst))) return fail(HODLR_ERR_INVALID, "bad arguments");
    CUDA_TRY(launch_dequantize(fmt, src, dst, count, (cudaStream_t)stream));
    return HODLR_OK;
}
hodlr_status hodlr_quantize_host(int32_t fmt, const double* src, void* dst, int64_t count) {
    if (!valid_fmt(fmt)) return fail(HODLR_ERR_UNSUPPORTED, "unsupported format");
    if (count < 0 || (count > 0 && (!src || !dst))) return fail(HODLR_ERR_INVALID, "bad arguments");
    for (int64_t i = 0; i < count; ++i) enc_any(fmt, src[i], dst, i);
    return HODLR_OK;
}
hodlr_status hodlr_dequantize_host(int32_t fmt, const void* src, double* dst, int64_t count) {
    if (!valid_fmt(fmt)) return fail(HODLR_ERR_UNSUPPORTED, "unsupported format");
    if (count < 0 || (count > 0 && (!src || !dst))) return fail(HODLR_ERR_INVALID, "bad arguments");
    for (int64_t i = 0; i < count; ++i) dst[i] = dec_any(fmt, src, i);
    return HODLR_OK;
}

static hodlr_status copy_cols_back(const hodlr_handle* h, int64_t off, int fmt, int ld, int rank,
                                   int64_t rows, double* out) {
    std::vector<uint8_t> raw((size_t)ld * rank * fmt_bytes(fmt) + 16);
    if (rank > 0) {
        cudaError_t e = cudaMemcpy(raw.data(), (const uint8_t*)h->arena.p + off,
                                   (size_t)ld * rank * fmt_bytes(fmt), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return fail(HODLR_ERR_CUDA, cudaGetErrorString(e));
    }
    for (int64_t r = 0; r < rows; ++r)
        for (int c = 0; c < rank; ++c) out[r * rank + c] = dec_any(fmt, raw.data(), (int64_t)c * ld + r);
    return HODLR_OK;
}

hodlr_status hodlr_unpack_factor(const hodlr_handle* h, int64_t index, double* U, double* V) {
    if (!h) return fail(HODLR_ERR_INVALID, "null handle");
    if (h->nranks != 1) return fail(HODLR_ERR_INVALID, "unpack needs an unsharded handle");
    int64_t nf = 2 * ((int64_t(1) << h->depth) - 1);
    if (index < 0 || index >= nf) return fail(HODLR_ERR_INVALID, "factor index out of range");
    // invert fidx: level k with 2*(2^(k-1)-1) <= index < 2*(2^k-1)
    int k = 1;
    while (2 * ((int64_t(1) << k) - 1) <= index) ++k;
    int64_t rel = index - 2 * ((int64_t(1) << (k - 1)) - 1);
    int64_t i = rel / 2;
    int lower = (int)(rel % 2);
    // upper: U in node 2i, V in node 2i+1; lower: U in node 2i+1, V in node 2i
    const NodeDesc& nu = h->nodes[h->node_id[k][2 * i + lower]];
    const NodeDesc& nv = h->nodes[h->node_id[k][2 * i + 1 - lower]];
    CUDA_TRY(cudaSetDevice(h->device));
    hodlr_status r = copy_cols_back(h, nu.u_off, nu.u_fmt, nu.u_ld, nu.ru, nu.nrows, U);
    if (r != HODLR_OK) return r;
    return copy_cols_back(h, nv.v_off, nv.v_fmt, nv.v_ld, nv.rv, nv.nrows, V);
}

hodlr_status hodlr_unpack_leaf(const hodlr_handle* h, int64_t leaf, double* D) {
    if (!h) return fail(HODLR_ERR_INVALID, "null handle");
    if (leaf < 0 || leaf >= (int64_t)h->leaves.size()) return fail(HODLR_ERR_INVALID, "leaf index out of range");
    const LeafDesc& l = h->leaves[leaf];
    std::vector<uint8_t> raw((size_t)l.m * l.ld * fmt_bytes(l.fmt));
    CUDA_TRY(cudaSetDevice(h->device));
    CUDA_TRY(cudaMemcpy(raw.data(), (const uint8_t*)h->arena.p + l.off, raw.size(), cudaMemcpyDeviceToHost));
    for (int r = 0; r < l.m; ++r)
        for (int c = 0; c < l.m; ++c) D[(int64_t)r * l.m + c] = dec_any(l.fmt, raw.data(), (int64_t)r * l.ld + c);
    return HODLR_OK;
}

hodlr_status hodlr_info(const hodlr_handle* h, hodlr_info_t* info) {
    if (!h || !info) return fail(HODLR_ERR_INVALID, "bad arguments");
    info->n_local = h->n_local;
    info->row0 = h->row0;
    info->matrix_bytes = h->matrix_bytes;
    info->device_bytes = (int64_t)h->arena_bytes;
    info->depth = h->depth;
    info->leaf_fmt = h->leaf_fmt;
    info->launches_per_matvec = (h->sv_ok ? sv_launches(h->sv) : 3) + (h->nranks > 1 && h->ext_count ? 3 : 0);
    info->num_levels_external = h->L;
    return HODLR_OK;
}

}  // extern "C"
