// Per-D / per-precision dispatch entry points, defined in twb_inst.cu (compiled
// once per (kind, R, Z, D) combination by the Makefile).
#pragma once

#include "twb_launch.cuh"

namespace twb {

template <int D, typename R, typename Z>
cudaError_t batch_d(int P, bool E, bool N1, const BatchArgs<R, Z>& a, int64_t max_rows,
                    const Alloc& alloc, cudaStream_t st, LaunchCtx* ctx);

template <int D, typename R, typename Z>
cudaError_t wave_d(int P, bool E, bool N1, const WaveProblem<R, Z>& pr, const Alloc& alloc,
                   cudaStream_t st, LaunchCtx* ctx);

}  // namespace twb
