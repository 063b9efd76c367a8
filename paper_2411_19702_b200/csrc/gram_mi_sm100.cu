// Kernel 2+3 dispatch: picks the instantiation (gram_mi_inst_*.cu) of the
// fused Gram + MI kernel (gram_mi_sm100.cuh) for the launch's knobs.
#include "gram_mi_sm100.cuh"

namespace mib200 {

#define MI_EXTERN4(CGV, OV, MV, PV, FV) \
    extern template cudaError_t launch_impl<CGV, OV, MV, 6, 8, PV, FV>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
#define MI_EXTERN(CGV, OV, MV, PV) MI_EXTERN4(CGV, OV, MV, PV, false)
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
MI_EXTERN4(2, MI_OUT_F64, MI_MODE_EXACT, false, true)
MI_EXTERN4(2, MI_OUT_F64, MI_MODE_EPSILON, false, true)
MI_EXTERN4(2, MI_OUT_F32, MI_MODE_EXACT, false, true)
MI_EXTERN4(2, MI_OUT_F32, MI_MODE_EPSILON, false, true)
MI_EXTERN4(2, MI_OUT_COUNTS, MI_MODE_EXACT, false, true)
MI_EXTERN4(2, MI_OUT_F64, MI_MODE_EXACT, true, true)
MI_EXTERN4(2, MI_OUT_F64, MI_MODE_EPSILON, true, true)
MI_EXTERN4(2, MI_OUT_F32, MI_MODE_EXACT, true, true)
MI_EXTERN4(2, MI_OUT_F32, MI_MODE_EPSILON, true, true)
MI_EXTERN4(2, MI_OUT_COUNTS, MI_MODE_EXACT, true, true)
#undef MI_EXTERN
#undef MI_EXTERN4

cudaError_t launch_gram_mi(int cg, bool fp4, int out_kind, int mode, int stages, int epi_warps,
                           const CUtensorMap& tmap, const GramMiParams& p, int num_sms, cudaStream_t stream) {
    const bool pace = p.pace != nullptr && p.pace_window > 0;
#define MI_DISPATCH_PF(CGV, OV, MV, STV, EWV, PV, FV)                                                            \
    if (cg == CGV && out_kind == OV && mode == MV && stages == STV && epi_warps == EWV && pace == PV && fp4 == FV) \
        return launch_impl<CGV, OV, MV, STV, EWV, PV, FV>(tmap, p, num_sms, stream);
#define MI_DISPATCH_P(CGV, OV, MV, STV, EWV, PV) \
    MI_DISPATCH_PF(CGV, OV, MV, STV, EWV, PV, false) MI_DISPATCH_PF(CGV, OV, MV, STV, EWV, PV, true)
#define MI_DISPATCH(CGV, OV, MV, STV, EWV) MI_DISPATCH_PF(CGV, OV, MV, STV, EWV, false, false)
    MI_DISPATCH_P(2, MI_OUT_F64, MI_MODE_EXACT, 6, 8, false)
    MI_DISPATCH_P(2, MI_OUT_F64, MI_MODE_EPSILON, 6, 8, false)
    MI_DISPATCH_P(2, MI_OUT_F32, MI_MODE_EXACT, 6, 8, false)
    MI_DISPATCH_P(2, MI_OUT_F32, MI_MODE_EPSILON, 6, 8, false)
    MI_DISPATCH_P(2, MI_OUT_COUNTS, MI_MODE_EXACT, 6, 8, false)
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
#undef MI_DISPATCH_PF
    if (fp4 && cg != 2) return cudaErrorInvalidValue;  // e2m1 operands: SM-pair builds only
    // knob combinations without a dedicated build fall back to the default build of the variant
    if (stages != 6 || epi_warps != 8) return launch_gram_mi(cg, fp4, out_kind, mode, 6, 8, tmap, p, num_sms, stream);
    if (pace) {  // no paced build of this variant (CG == 1)
        GramMiParams q = p;
        q.pace = nullptr;
        return launch_gram_mi(cg, fp4, out_kind, mode, stages, epi_warps, tmap, q, num_sms, stream);
    }
    return cudaErrorInvalidValue;
}

#define MI_XP_EXTERN(OV, MV) \
    extern template cudaError_t launch_impl<2, OV, MV, kXpStages, kXpEpiWarps, false, true, true>(const CUtensorMap&, const GramMiParams&, int, cudaStream_t);
MI_XP_EXTERN(MI_OUT_F64, MI_MODE_EXACT)
MI_XP_EXTERN(MI_OUT_F64, MI_MODE_EPSILON)
MI_XP_EXTERN(MI_OUT_F32, MI_MODE_EXACT)
MI_XP_EXTERN(MI_OUT_F32, MI_MODE_EPSILON)
MI_XP_EXTERN(MI_OUT_COUNTS, MI_MODE_EXACT)
#undef MI_XP_EXTERN

cudaError_t launch_gram_mi_words(int out_kind, int mode, const CUtensorMap& tmap, const GramMiParams& p, int num_sms,
                                 cudaStream_t stream) {
#define MI_XP_DISPATCH(OV, MV) \
    if (out_kind == OV && mode == MV) return launch_impl<2, OV, MV, kXpStages, kXpEpiWarps, false, true, true>(tmap, p, num_sms, stream);
    MI_XP_DISPATCH(MI_OUT_F64, MI_MODE_EXACT)
    MI_XP_DISPATCH(MI_OUT_F64, MI_MODE_EPSILON)
    MI_XP_DISPATCH(MI_OUT_F32, MI_MODE_EXACT)
    MI_XP_DISPATCH(MI_OUT_F32, MI_MODE_EPSILON)
    MI_XP_DISPATCH(MI_OUT_COUNTS, MI_MODE_EXACT)
#undef MI_XP_DISPATCH
    return cudaErrorInvalidValue;
}

int gram_mi_tile_size(int cg) { return 128 * cg; }

}  // namespace mib200
