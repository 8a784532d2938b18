// Multi-right-hand-side (s > 1) path: the batched U/V application and the
// leaf products as dense contractions on the tensor cores (SURVEY.md §7.1
// step 5; north star "tensor cores only in the multi-RHS mode").
//
// Three stream-ordered launches per matvec over the level-batched arena of
// plan.h (no separate layout):
//   MA  persistent-range phase A: CTA b owns a contiguous run of chunks (row
//       tiles) and accumulates V'_k[rows]^T X[rows] for every level k in
//       shared memory while consecutive chunks stay inside one level-k node;
//       a node boundary (or the end of the run) flushes the tile to a partial
//       slot (level k, slot = b + index of the node in its level).
//   MR  fixed-order reduction of a node's slots (CTA order) -> T_k
//       (deterministic; no atomics anywhere).
//   MB  one CTA per chunk: b[rows] = [D | U_1 .. U_l] [X_leaf ; T_1 .. T_l],
//       i.e. the leaf product and every level's U T as ONE contraction with
//       K = m + sum_k r_k, written once (disjoint rows).
// Tensor-core kinds: fp64 working -> DMMA (mma.sync m8n8k4 f64, the B200's
// FP64 tensor path); fp32 working -> TF32 with a hi/lo split of both operands
// (3 products, "3xTF32"), which keeps fp32-level accuracy.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "../../include/hodlr_b200.h"
#include "plan.h"
#include "tcb.h"

namespace hodlr {

constexpr int kMrMaxLevels = 31;
constexpr int kMr2MaxTasks = 64;           // 16 compute warps x <= 4 tasks
constexpr int kMr2MaxRows = 1024;          // kMr2MaxTasks x MR (16 for TF32)

struct MrLevel {
    int32_t node0, nnodes;   // node ids of the level: [node0, node0 + nnodes)
    int32_t rv_max, ru_max;  // max ranks over the level's nodes
    int32_t rv_pad;          // rv_max rounded up to 8: rows of one partial slot
    int32_t ext_w;           // external level of a sharded handle: its send-slot width (else 0)
    int64_t part_rows;       // first partial row of the level (a row holds spad values)
};

// Per node id: the phase-A CTAs whose chunk runs intersect the node, its index
// within its level, and its level (0-based).
struct MrSlot {
    int32_t b0, b1, jrel, lv;
};

// Phase-A flush table (k_mr3_a), per (chunk, level): does the level's node end at
// this chunk of its run, and where do its rows go.
struct MrFlush {
    int64_t row;             // direct: t_off of the node; else the partial row of its (run, node) slot
    int32_t clim;            // stored columns: c < clim
    int32_t direct;          // 1: the run holds the whole node, its sum IS the coefficient
};

struct MrView {
    int32_t nlev;            // levels 0..nlev-1 = tree levels 1..nlev
    int32_t nb;              // phase-A CTAs; slots per level = nb + nnodes
    int64_t part_rows;       // total partial rows (x spad values)
    const MrSlot* slots;     // device, indexed by node id
    const MrFlush* flush;    // device, [nchunks][nlev]
    const uint32_t* flush_mask;  // device, [nchunks]: bit lv = level lv's node ends at this chunk of its run
    MrLevel lev[kMrMaxLevels];
};

// Fragment slabs (uniform trees: every leaf one 256-row chunk, one storage
// format per level): the quantised factors and leaves re-ordered, per chunk,
// into exactly the sequence of MMA operand fragments the kernels consume, so
// each warp streams contiguous bytes with cp.async.bulk into a private ring.
//   A region (phase A), per chunk: 16 k-steps, each holding one k-block of
//     every task (level-major, m-tile-major; one k-block = 32 lanes x AR rows
//     x 4 consecutive rows of V'), so any run of k-steps is one contiguous stage.
//   B region (phase B), per chunk and warp (rows 32w..32w+31): 16 D items
//     (one per 16-column k step: MT m-tiles x 32 lanes x AR x 4 values), then
//     the U items of every level (one per KU-column step).
struct Mr2Level {
    int32_t nmt;      // phase-A m-tiles (ceil(rv_max / MR))
    int32_t vfmt;     // V' storage format of the level
    int32_t ablk;     // bytes of one A k-block
    int32_t steps;    // U steps (ceil(ru_max / KU))
    int32_t ufmt;     // U storage format of the level
    int32_t usz;      // bytes of one U item
    int64_t aoff;     // offset of the level's first task block inside one k-step of the A region
    int64_t uoff;     // offset of the level's first U item in a warp's B region
    int32_t ulo;      // the same, relative to the start of the U area (after the 16 D items)
    int32_t unext;    // U-area offset of the next level with steps, -1 if none
};
struct Mr2View {
    int32_t nlev, lev_lo;      // levels lev_lo..nlev-1 are in the B region (phase B)
    int32_t alev_lo;           // levels alev_lo..nlev-1 are in the A region (0: incl. external levels)
    int32_t ntasks;            // phase-A tasks (m-tiles) per chunk
    int32_t nu_items;          // U items per warp per chunk
    int64_t a_chunk_bytes, b_chunk_bytes;
    int32_t warp_bytes;        // B bytes per warp per chunk
    int32_t d_item;            // bytes of one D item (a power of two: the ring slot)
    int32_t lslot;             // log2(d_item)
    int32_t leaf_fmt;
    int32_t max_ablk;
    int32_t arow;              // A bytes of one k-step, all tasks ([kb][task] layout)
    int32_t widen_fast;        // the slabs hold no fp32 subnormal / inf / nan (integer fp32 -> fp64 widening is exact)
    // Stacked U (every level's U in one storage format): the levels' U columns are
    // concatenated (no per-level padding) and cut into nku 16-column k-blocks laid
    // out exactly like the D items ([k-block][warp][m-tile][lane][4 columns]), so
    // the U part of phase B is nku more iterations of the D loop.
    int32_t ustack;            // 1: stacked U layout (else per-level U steps)
    int32_t nku;               // 16-column U k-blocks per chunk
    int32_t ufmt_all;          // the common U storage format
    int32_t u_item;            // bytes of one warp's block of one U k-block
    int16_t urow_lv[kMr2MaxRows];  // stacked U column -> level (-1: padding)
    int16_t urow_c[kMr2MaxRows];   //                  -> rank column
    // Phase-A tasks stack the levels' V' columns along M (a run of levels with
    // one storage format shares m-tiles; a format change starts a new tile):
    // stacked row m -> (level, column), level -1 = padding.
    int32_t task_fmt[kMr2MaxTasks];
    int32_t task_off[kMr2MaxTasks];   // byte offset of the task's block inside one k-step
    int16_t row_lv[kMr2MaxRows];
    int16_t row_c[kMr2MaxRows];
    const uint8_t* slab_a;
    const uint8_t* slab_b;
    Mr2Level lev[kMrMaxLevels];
};

struct MrPlan {
    bool ok = false;
    bool slab_ok = false;      // fragment slabs built (for the working precision slab_fmt)
    bool sharded = false;      // handle of a sharded tree (external levels 1..L)
    int slab_fmt = -1;
    Mr2View v2{};
    void* slab_dev = nullptr;
    bool has_fp64_operand = false;  // an fp64 factor or leaf: the TF32 kind cannot take it
    int leaf_fmt = HODLR_FMT_FP64;
    MrView view{};
    void* dev = nullptr;
    void* flush_dev = nullptr; // device: MrFlush table + masks
    int32_t* multi = nullptr;  // device: ids of nodes summed over several phase-A CTAs (or external)
    int nmulti = 0;
    int nbig = 0;              // the first nbig listed nodes sum more than 32 slots
    int rmax_big = 0, rmax_small = 0;
    int max_leaf_m = 0;
    bool tc_ok = false;        // tcgen05 phase B (fp32 working, uniform 256-row leaves)
    void* tc_dev = nullptr;
    TcView tcv{};
    bool tca_cand = false;     // tcgen05 phase A eligible (decided before the slot layout: nb = SMs)
    bool tca_ok = false;
    void* tca_dev = nullptr;
    TcAView tcav{};
};

struct MrInput {
    const PlanView* view;      // device tables of the handle (for the relayout kernels)
    const uint8_t* d_arena;    // quantised level-batched arena (device)
    int lev_lo;                // first level handled by the multi-RHS kernels
    const std::vector<NodeDesc>* nodes;
    const std::vector<ChunkDesc>* chunks;
    const std::vector<LeafDesc>* leaves;
    const std::vector<int32_t>* chunk_nodes;
    int nlev;
    int leaf_fmt;
    int device;
    int64_t ext_count;         // sharded: send slots per unit s (external levels)
};

hodlr_status mr_prepare(const MrInput& in, MrPlan& mr);
void mr_release(MrPlan& mr);
inline int64_t mr_spad(int64_t s) { return (s + 7) / 8 * 8; }
// partial elements needed for s right-hand sides
inline int64_t mr_part_elems(const MrPlan& mr, int64_t s) { return mr.view.part_rows * mr_spad(s); }
// true if the multi-RHS kernels take this call
bool mr_usable(const MrPlan& mr, int working_fmt);
// true if such a call runs the fragment-slab kernels
bool mr_slab_used(const MrPlan& mr, int working_fmt, int lev_lo);
int mr_launches();
// Levels lev_lo..nlev-1 only (lev_lo = L on a sharded handle: the external
// levels run in kernels_shard.cu).  `send` receives external-level sums when
// lev_lo = 0 on a sharded handle (unused otherwise).
template <typename W>
cudaError_t mr_matvec(const PlanView& p, const MrPlan& mr, int lev_lo, const W* x, int64_t ldx, W* b,
                      int64_t ldb, int64_t s, W* partial, W* tbuf, cudaStream_t st);
// Sharded handles with fragment slabs: shard_begin runs phase A over ALL levels
// (external partials -> send, subtree coefficients -> tbuf); shard_local does
// nothing; shard_end reduces the gathered external coefficients and runs phase
// B over ALL levels (mr_slab_phase_b): b is written once, no read-modify-write.
bool mr_slab_begin_usable(const MrPlan& mr, int working_fmt);
template <typename W>
cudaError_t mr_shard_begin(const PlanView& p, const MrPlan& mr, const W* x, int64_t ldx, int64_t s, W* partial,
                           W* tbuf, W* send, cudaStream_t st);
template <typename W>
cudaError_t mr_slab_phase_b(const PlanView& p, const MrPlan& mr, const W* x, int64_t ldx, W* b, int64_t ldb,
                            int64_t s, const W* tbuf, cudaStream_t st);

// Host-buffer pipeline: phase A + reduce, then phase B over chunk ranges [chunk0, chunk1)
// (256-row chunks, in row order), so the copies of finished ranges overlap later kernels.
bool mr_sliceable(const MrPlan& mr, int working_fmt, int64_t s);
cudaError_t mr_phase_a(const PlanView& p, const MrPlan& mr, const double* x, int64_t ldx, int64_t s, double* partial,
                       double* tbuf, cudaStream_t st);
cudaError_t mr_phase_b_range(const PlanView& p, const MrPlan& mr, const double* x, int64_t ldx, double* b, int64_t ldb,
                             int64_t s, double* tbuf, int chunk0, int chunk1, cudaStream_t st);

// tcgen05 phase A / B (kernels_tc.cu)
bool tc_a_candidate(const MrInput& in, const MrView& v);
bool tca_usable(const MrPlan& mr, int64_t s);
cudaError_t tc_phase_a(const PlanView& p, const MrPlan& mr, const float* x, int64_t ldx, int64_t s, float* partial,
                       float* tbuf, cudaStream_t st);
hodlr_status tc_prepare(const MrInput& in, MrPlan& mr);
bool tc_usable(const MrPlan& mr, int64_t s);
cudaError_t tc_phase_b(const PlanView& p, const MrPlan& mr, const float* x, int64_t ldx, float* b, int64_t ldb,
                       int64_t s, const float* tbuf, cudaStream_t st);

}  // namespace hodlr
