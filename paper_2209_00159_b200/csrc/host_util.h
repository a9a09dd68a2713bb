// host_util.h — host-side helpers shared by the translation units of
// liborloj.so (defined in orloj.cu): status / last-error plumbing, O(1)
// argument checks and the profile compilation (division magic, A3, A14).
#pragma once
#include <cuda_runtime.h>

#include <atomic>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a tool (nsys, ncu) injects
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
// x[0..n) = v on `stream` (async)
cudaError_t fill_i64(int64_t *x, int64_t n, int64_t v, cudaStream_t s);
int bins_per_lane(int B);
int slots_for(int kmax);

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device property of a
// kernel: set it once per (kernel, device) — `done` is one bit per device id
// (ids >= 64 set it on every call).  Idempotent, so a race only repeats it.
template <class K>
cudaError_t ensure_max_dyn_smem(K kernel, int bytes, std::atomic<uint64_t> &done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// One NVTX range per C-ABI call (push at entry, pop at return), so nsys / ncu
// timelines attribute the multi-stream replay and the e2e copy pipelines to
// the library calls that enqueued them.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
#define ORLOJ_NVTX(name) ::orloj::host::NvtxRange orloj_nvtx_range_(name)

// Resident blocks per SM x SM count (one wave) of a kernel at a block size and
// dynamic shared memory, cached per device for the last smem size asked (the
// occupancy query costs microseconds: not on every launch).  Races only
// repeat the query.
struct WaveCache {
  std::atomic<int64_t> key[64];   // smem bytes + 1 (0: empty)
  std::atomic<int64_t> wave[64];
};
template <class K>
cudaError_t one_wave(K kernel, int threads, size_t smem, WaveCache &c, int64_t *out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && c.key[dev].load(std::memory_order_acquire) == (int64_t)smem + 1) {
    *out = c.wave[dev].load(std::memory_order_relaxed);
    return cudaSuccess;
  }
  int sms = 148, occ = 1;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem)) != cudaSuccess) return e;
  *out = (int64_t)sms * (occ < 1 ? 1 : occ);
  if (dev < 64) {
    c.wave[dev].store(*out, std::memory_order_relaxed);
    c.key[dev].store((int64_t)smem + 1, std::memory_order_release);
  }
  return cudaSuccess;
}

}  // namespace host
}  // namespace orloj
