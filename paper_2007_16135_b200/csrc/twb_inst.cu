// One translation unit per (kind, R, Z, D), selected by -D flags from the
// Makefile: TWB_KIND_BATCH or TWB_KIND_WAVE, TWB_R, TWB_Z, TWB_D.
// P (degree): 1, 2, or 0 = runtime degree (always with the NaN-exact min).
// E: NaN-exact compare chain; N1: nu == 1.0 (nu * x == x exactly).
#include "twb_dispatch.h"

namespace twb {

#define TWB_SWITCH                                                                   \
    if constexpr (TWB_D == 1) {                                                      \
        if (E) return CALL(2, true, false);                                          \
        return N1 ? CALL(2, false, true) : CALL(2, false, false);                    \
    } else {                                                                         \
        if (P == 0) return CALL(0, true, false);                                     \
        if (P == 1) {                                                                \
            if (E) return CALL(1, true, false);                                      \
            return N1 ? CALL(1, false, true) : CALL(1, false, false);                \
        }                                                                            \
        if (E) return CALL(2, true, false);                                          \
        return N1 ? CALL(2, false, true) : CALL(2, false, false);                    \
    }

#if defined(TWB_KIND_BATCH)
template <>
cudaError_t batch_d<TWB_D, TWB_R, TWB_Z>(int P, bool E, bool N1, const BatchArgs<TWB_R, TWB_Z>& a,
                                         int64_t max_rows, const Alloc& alloc, cudaStream_t st,
                                         LaunchCtx* ctx) {
#define CALL(p, e, n) run_batch<TWB_D, p, e, n, TWB_R, TWB_Z>(a, max_rows, alloc, st, ctx)
    TWB_SWITCH
#undef CALL
}
#elif defined(TWB_KIND_WAVE)
template <>
cudaError_t wave_d<TWB_D, TWB_R, TWB_Z>(int P, bool E, bool N1, const WaveProblem<TWB_R, TWB_Z>& pr,
                                        const Alloc& alloc, cudaStream_t st, LaunchCtx* ctx) {
#define CALL(p, e, n) run_wave<TWB_D, p, e, n, TWB_R, TWB_Z>(pr, alloc, st, ctx)
    TWB_SWITCH
#undef CALL
}
#else
#error "define TWB_KIND_BATCH or TWB_KIND_WAVE"
#endif

}  // namespace twb
