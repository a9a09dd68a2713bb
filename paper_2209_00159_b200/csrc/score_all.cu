// score_all.cu — instantiates score_kernel<..., PICK = false, ...> (see score_launch.cuh).
#include "score_launch.cuh"

namespace orloj {
namespace host {
cudaError_t launch_score_all(const ScoreParams &p, RowSrc src, cudaStream_t s) {
  return launch_score_b<false>(p, src, s);
}
}  // namespace host
}  // namespace orloj
