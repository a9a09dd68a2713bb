// host_util.h — host-side helpers shared by the translation units of
// liborloj.so (defined in orloj.cu): status / last-error plumbing, O(1)
// argument checks and the profile compilation (division magic, A3, A14).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/orloj.h"
#include "common.cuh"

namespace orloj {
namespace host {

orloj_status fail(orloj_status st, const char *fmt, ...);
orloj_status cuda_fail(cudaError_t e, const char *where);
orloj_status ok();
bool aligned16(const void *p);
orloj_status check_store(const orloj_store *st, int max_bins);
orloj_status compile_profile(const orloj_latency_profile *pr, int32_t B, int kcap, ProfileDev *out);
orloj_status check_queues(const orloj_queues *q);
int bins_per_lane(int B);
int slots_for(int kmax);

}  // namespace host
}  // namespace orloj
