// Explicit instantiations of the fused kernel's word-operand build (XP): e2m1
// operands expanded from the packed words inside the producer, 4 epilogue
// warps, unpaced (gram_mi_sm100.cuh).
#include "gram_mi_sm100.cuh"

namespace mib200 {
#define MI_XP_INST(OV, MV)                                                                                  \
    template cudaError_t launch_impl<2, OV, MV, kXpStages, kXpEpiWarps, false, true, true>(const CUtensorMap&,    \
                                                                                  const GramMiParams&, int, \
                                                                                  cudaStream_t);
MI_XP_INST(MI_OUT_F64, MI_MODE_EXACT)
MI_XP_INST(MI_OUT_F64, MI_MODE_EPSILON)
MI_XP_INST(MI_OUT_F32, MI_MODE_EXACT)
MI_XP_INST(MI_OUT_F32, MI_MODE_EPSILON)
MI_XP_INST(MI_OUT_COUNTS, MI_MODE_EXACT)
#undef MI_XP_INST
}  // namespace mib200
