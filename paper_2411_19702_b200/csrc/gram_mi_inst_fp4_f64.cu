// Explicit instantiations of the fused kernel, e2m1 (kind::mxf4) operands.
#include "gram_mi_sm100.cuh"

namespace mib200 {
template cudaError_t launch_impl<2, MI_OUT_F64, MI_MODE_EXACT, 6, 8, false, true>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
template cudaError_t launch_impl<2, MI_OUT_F64, MI_MODE_EXACT, 6, 8, true, true>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
template cudaError_t launch_impl<2, MI_OUT_F64, MI_MODE_EPSILON, 6, 8, false, true>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
template cudaError_t launch_impl<2, MI_OUT_F64, MI_MODE_EPSILON, 6, 8, true, true>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
template cudaError_t launch_impl<2, MI_OUT_COUNTS, MI_MODE_EXACT, 6, 8, false, true>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
template cudaError_t launch_impl<2, MI_OUT_COUNTS, MI_MODE_EXACT, 6, 8, true, true>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
}  // namespace mib200
