// Single-vector fast path (placeholder: disabled until the fused kernel lands).
#include "sv.h"

namespace hodlr {

hodlr_status sv_prepare(const std::vector<NodeDesc>&, const std::vector<ChunkDesc>&,
                        const std::vector<LeafDesc>&, const std::vector<int32_t>&, int, SvPlan& sv,
                        bool* ok) {
    sv = SvPlan{};
    *ok = false;
    return HODLR_OK;
}
void sv_release(SvPlan& sv) { sv = SvPlan{}; }
size_t sv_extra_ws(const SvPlan& sv, int64_t) { return sv.extra_ws; }
int sv_launches(const SvPlan& sv) { return sv.launches; }

template <typename W>
cudaError_t sv_matvec(const PlanView&, const SvPlan&, const W*, W*, W*, W*, void*, cudaStream_t) {
    return cudaErrorNotSupported;
}
template cudaError_t sv_matvec<double>(const PlanView&, const SvPlan&, const double*, double*,
                                       double*, double*, void*, cudaStream_t);
template cudaError_t sv_matvec<float>(const PlanView&, const SvPlan&, const float*, float*, float*,
                                      float*, void*, cudaStream_t);

}  // namespace hodlr
