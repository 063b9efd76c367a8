// Kernel 2+3 dispatch: picks the instantiation (gram_mi_inst_*.cu) of the
// fused Gram + MI kernel (gram_mi_sm100.cuh) for the launch's knobs.
#include "gram_mi_sm100.cuh"

namespace mib200 {

#define MI_EXTERN(CGV, OV, MV, PV) \
    extern template cudaError_t launch_impl<CGV, OV, MV, 6, 8, PV>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
MI_EXTERN(2, MI_OUT_F64, MI_MODE_EXACT, false)
MI_EXTERN(2, MI_OUT_F64, MI_MODE_EPSILON, false)
MI_EXTERN(2, MI_OUT_F32, MI_MODE_EXACT, false)
MI_EXTERN(2, MI_OUT_F32, MI_MODE_EPSILON, false)
MI_EXTERN(2, MI_OUT_COUNTS, MI_MODE_EXACT, false)
MI_EXTERN(2, MI_OUT_F64, MI_MODE_EXACT, true)
MI_EXTERN(2, MI_OUT_F64, MI_MODE_EPSILON, true)
MI_EXTERN(2, MI_OUT_F32, MI_MODE_EXACT, true)
MI_EXTERN(2, MI_OUT_F32, MI_MODE_EPSILON, true)
MI_EXTERN(2, MI_OUT_COUNTS, MI_MODE_EXACT, true)
MI_EXTERN(1, MI_OUT_F64, MI_MODE_EXACT, false)
MI_EXTERN(1, MI_OUT_F64, MI_MODE_EPSILON, false)
MI_EXTERN(1, MI_OUT_F32, MI_MODE_EXACT, false)
MI_EXTERN(1, MI_OUT_F32, MI_MODE_EPSILON, false)
MI_EXTERN(1, MI_OUT_COUNTS, MI_MODE_EXACT, false)
#undef MI_EXTERN

cudaError_t launch_gram_mi(int cg, int out_kind, int mode, int stages, int epi_warps, const CUtensorMap& tmap,
                           const GramMiParams& p, int num_sms, cudaStream_t stream) {
    const bool pace = p.pace != nullptr && p.pace_window > 0;
#define MI_DISPATCH_P(CGV, OV, MV, STV, EWV, PV)                                                               \
    if (cg == CGV && out_kind == OV && mode == MV && stages == STV && epi_warps == EWV && pace == PV) \
        return launch_impl<CGV, OV, MV, STV, EWV, PV>(tmap, p, num_sms, stream);
#define MI_DISPATCH(CGV, OV, MV, STV, EWV) MI_DISPATCH_P(CGV, OV, MV, STV, EWV, false)
    MI_DISPATCH(2, MI_OUT_F64, MI_MODE_EXACT, 6, 8)
    MI_DISPATCH(2, MI_OUT_F64, MI_MODE_EPSILON, 6, 8)
    MI_DISPATCH(2, MI_OUT_F32, MI_MODE_EXACT, 6, 8)
    MI_DISPATCH(2, MI_OUT_F32, MI_MODE_EPSILON, 6, 8)
    MI_DISPATCH(2, MI_OUT_COUNTS, MI_MODE_EXACT, 6, 8)
    MI_DISPATCH_P(2, MI_OUT_F64, MI_MODE_EXACT, 6, 8, true)
    MI_DISPATCH_P(2, MI_OUT_F64, MI_MODE_EPSILON, 6, 8, true)
    MI_DISPATCH_P(2, MI_OUT_F32, MI_MODE_EXACT, 6, 8, true)
    MI_DISPATCH_P(2, MI_OUT_F32, MI_MODE_EPSILON, 6, 8, true)
    MI_DISPATCH_P(2, MI_OUT_COUNTS, MI_MODE_EXACT, 6, 8, true)
    MI_DISPATCH(1, MI_OUT_F64, MI_MODE_EXACT, 6, 8)
    MI_DISPATCH(1, MI_OUT_F64, MI_MODE_EPSILON, 6, 8)
    MI_DISPATCH(1, MI_OUT_F32, MI_MODE_EXACT, 6, 8)
    MI_DISPATCH(1, MI_OUT_F32, MI_MODE_EPSILON, 6, 8)
    MI_DISPATCH(1, MI_OUT_COUNTS, MI_MODE_EXACT, 6, 8)
#undef MI_DISPATCH
#undef MI_DISPATCH_P
    // knob combinations without a dedicated build fall back to the default build of the variant
    if (stages != 6 || epi_warps != 8) return launch_gram_mi(cg, out_kind, mode, 6, 8, tmap, p, num_sms, stream);
    if (pace) {  // no paced build of this variant (CG == 1)
        GramMiParams q = p;
        q.pace = nullptr;
        return launch_gram_mi(cg, out_kind, mode, stages, epi_warps, tmap, q, num_sms, stream);
    }
    return cudaErrorInvalidValue;
}

int gram_mi_tile_size(int cg) { return 128 * cg; }

}  // namespace mib200
