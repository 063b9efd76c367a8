// Explicit instantiations of the fused kernel (split for parallel builds).
#include "gram_mi_sm100.cuh"

namespace mib200 {
template cudaError_t launch_impl<2, MI_OUT_F64, MI_MODE_EXACT, 6, 8, false, false>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
template cudaError_t launch_impl<2, MI_OUT_F64, MI_MODE_EXACT, 6, 8, true, false>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
template cudaError_t launch_impl<2, MI_OUT_F64, MI_MODE_EPSILON, 6, 8, false, false>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
template cudaError_t launch_impl<2, MI_OUT_F64, MI_MODE_EPSILON, 6, 8, true, false>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
}  // namespace mib200
