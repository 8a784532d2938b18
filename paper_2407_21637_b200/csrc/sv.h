// Single-vector (s = 1) streaming fast path: one persistent kernel per matvec,
// fed by cp.async.bulk (TMA bulk copies) from a leaf-slab layout.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "../../include/hodlr_b200.h"
#include "plan.h"

namespace hodlr {

struct SvPlan {
    void* dev = nullptr;     // slab arena (device)
    size_t dev_bytes = 0;
    const uint8_t* slab = nullptr;
    void* params = nullptr;  // host copy of the kernel parameter block
    int nleaves = 0, nnodes = 0, depth = 0;
    int rb = 0;                 // rows per phase-B item
    int num_items_a = 0, num_items_b = 0;
    int grid = 0;
    int launches = 1;
    int split = 0;              // 1: A-only launch + PDL-dependent R/BC launch
    int64_t tfast_count = 0;    // padded coefficient buffer (elements)
    int64_t part_count = 0;     // fast-path partial buffer (elements)
    size_t extra_ws = 0;        // bytes of workspace for sync state + coefficients
    int leaf_fmt = 4;
    int geo = 0;                // kernel geometry of this plan (SvInput::geo)
    int ctas_per_sm = 2;        // pipelines per SM of that geometry
};

struct SvInput {
    const std::vector<NodeDesc>* nodes;
    const std::vector<ChunkDesc>* chunks;
    const std::vector<LeafDesc>* leaves;
    const std::vector<int32_t>* chunk_nodes;
    int nlev;
    const uint8_t* d_arena;     // generic (level-batched) arena, already quantised
    size_t arena_bytes;
    // Kernel geometry (kernels_sv.cu is compiled twice): 0 = 2 CTAs per SM x 8 consumer
    // warps, ring of 3 x 32.5 KB (binary64 working: cfg2 and the fp64 half of cfg5);
    // 1 = 4 CTAs per SM x 4 consumer warps, ring of 2 x 20.3 KB (binary32 working: twice
    // the elements per byte, so more pieces are consumed concurrently; cfg5 eps = 1e-2:
    // 76.1 -> 68.4 us, and 45.7 vs 39.7 us on cfg2, which is why it is not the default).
    int geo = 0;
};

hodlr_status sv_prepare(const SvInput& in, SvPlan& sv, bool* ok);
void sv_release(SvPlan& sv);
size_t sv_extra_ws(const SvPlan& sv, int64_t s);
int sv_launches(const SvPlan& sv);
// shrink the persistent grid (e.g. to leave SMs to a concurrent all-gather);
// keeps the R-piece queue position within what that grid can reach
void sv_set_grid(SvPlan& sv, int grid);
template <typename W>
cudaError_t sv_matvec(const PlanView& p, const SvPlan& sv, const W* x, W* b, W* partial, W* tbuf,
                      void* extra, cudaStream_t st);

}  // namespace hodlr
