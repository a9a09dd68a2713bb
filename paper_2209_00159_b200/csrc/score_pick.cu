// score_pick.cu — instantiates score_kernel<..., PICK = true, ...> (see score_launch.cuh).
#include "score_launch.cuh"

namespace orloj {
namespace host {
cudaError_t launch_score_pick(const ScoreParams &p, RowSrc src, cudaStream_t s) {
  return launch_score_b<true>(p, src, s);
}
}  // namespace host
}  // namespace orloj
