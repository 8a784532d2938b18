// Single-vector (s = 1) fast path: one persistent kernel per matvec.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "../../include/hodlr_b200.h"
#include "plan.h"

namespace hodlr {

struct SvPlan {
    void* dev = nullptr;   // device-side work lists
    int num_items_a = 0;   // phase-A work items
    int num_items_b = 0;   // phase-B work items
    int grid = 0;          // persistent CTAs
    int launches = 1;
    size_t extra_ws = 0;   // bytes of workspace beyond partials/coefficients (per s=1)
    const void* items = nullptr;
    const void* sync = nullptr;
};

hodlr_status sv_prepare(const std::vector<NodeDesc>& nodes, const std::vector<ChunkDesc>& chunks,
                        const std::vector<LeafDesc>& leaves, const std::vector<int32_t>& chunk_nodes,
                        int nlev, SvPlan& sv, bool* ok);
void sv_release(SvPlan& sv);
size_t sv_extra_ws(const SvPlan& sv, int64_t s);
int sv_launches(const SvPlan& sv);
template <typename W>
cudaError_t sv_matvec(const PlanView& p, const SvPlan& sv, const W* x, W* b, W* partial, W* tbuf,
                      void* extra, cudaStream_t st);

}  // namespace hodlr
