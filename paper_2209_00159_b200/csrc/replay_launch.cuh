// replay_launch.cuh — template dispatch of replay_kernel<BPL, RATE, ALG1, MODE>;
// each MODE is instantiated in its own translation unit (replay_m<MODE>.cu) so
// the library builds in parallel.
#pragma once
#include <cuda_runtime.h>

#include "replay_kernel.cuh"

namespace orloj {

template <int MODE>
cudaError_t launch_replay(const ReplayParams &p, int bpl, bool rate, bool alg1, unsigned blocks, size_t smem,
                          cudaStream_t s);

#ifdef ORLOJ_REPLAY_INSTANTIATE
template <int MODE>
cudaError_t launch_replay(const ReplayParams &p, int bpl, bool rate, bool alg1, unsigned blocks, size_t smem,
                          cudaStream_t s) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (bpl * 4 + (rate ? 1 : 0) + (alg1 ? 2 : 0)) {
#define ORLOJ_REPLAY_CASE(BPL_, RATE_, ALG1_)                                                                   \
  case BPL_ * 4 + (RATE_ ? 1 : 0) + (ALG1_ ? 2 : 0):                                                            \
    e = cudaFuncSetAttribute(replay_kernel<BPL_, RATE_, ALG1_, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                                        \
    if (e == cudaSuccess) replay_kernel<BPL_, RATE_, ALG1_, MODE><<<blocks, REPLAY_WARPS * 32, smem, s>>>(p);   \
    break;
    ORLOJ_REPLAY_CASE(1, false, false)
    ORLOJ_REPLAY_CASE(1, true, false)
    ORLOJ_REPLAY_CASE(1, false, true)
    ORLOJ_REPLAY_CASE(2, false, false)
    ORLOJ_REPLAY_CASE(2, true, false)
    ORLOJ_REPLAY_CASE(2, false, true)
    ORLOJ_REPLAY_CASE(4, false, false)
    ORLOJ_REPLAY_CASE(4, true, false)
    ORLOJ_REPLAY_CASE(4, false, true)
#undef ORLOJ_REPLAY_CASE
    default:
      break;
  }
  return e;
}
template cudaError_t launch_replay<ORLOJ_REPLAY_INSTANTIATE>(const ReplayParams &, int, bool, bool, unsigned,
                                                             size_t, cudaStream_t);
#endif

}  // namespace orloj
