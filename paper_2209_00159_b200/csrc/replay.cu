// replay.cu — C ABI of the trace replay (include/orloj.h): argument checks,
// policy / profile compilation, launch of replay_kernel (plain, or the exact
// segmented form: speculative segments + stitch).
#include <cuda_runtime.h>

#include <cstring>

#include "../../include/orloj.h"
#include "host_util.h"
#include "replay_launch.cuh"

using namespace orloj;
using namespace orloj::host;

namespace {

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
size_t seg_state_bytes(int64_t S, int32_t G) { return align256((size_t)S * G * sizeof(ReplaySeg)); }
constexpr size_t SEG_STATS_BYTES = 256;  // workspace head: stitch statistics (include/orloj.h)

orloj_status replay_impl(const orloj_store *store, const orloj_latency_profile *profile, const orloj_trace *tr,
                         const orloj_replay_policy *policy, int32_t G, int64_t N, void *ws, size_t ws_bytes,
                         orloj_counters *per_bucket, int32_t *log, void *stream,
                         const orloj_replay_epoch *ep = nullptr) {
  orloj_status st;
  if ((st = check_store(store, ORLOJ_REPLAY_MAX_BINS))) return st;
  if (!policy || (policy->objective != ORLOJ_OBJ_EXPECTED_FINISH && policy->objective != ORLOJ_OBJ_FINISH_RATE &&
                  policy->objective != ORLOJ_OBJ_ALG1))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay policy: objective must be EXPECTED_FINISH, FINISH_RATE or ALG1");
  const bool rate = policy->objective == ORLOJ_OBJ_FINISH_RATE;
  const bool alg1 = policy->objective == ORLOJ_OBJ_ALG1;
  if (alg1 && (!policy->size_threshold_ticks || !policy->priority_table || !policy->priority_log_expected ||
               !(policy->priority_b_per_tick > 0.0) || policy->drop_threshold_ticks))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT,
                "replay policy ALG1: needs size thresholds, priority tables for sizes 1..kmax and b > 0, "
                "and no drop thresholds (Alg. 1 drops by the bs = 1 threshold)");
  if (!tr || tr->num_scenarios < 0 || tr->num_buckets < 1)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "trace: need num_scenarios >= 0 and num_buckets >= 1");
  if (tr->num_scenarios > 0 && (!tr->arrival_offsets || !tr->arrival_ticks || !tr->dist_id || !tr->true_bin ||
                                !tr->slo_ticks || !tr->bucket || !per_bucket))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "trace arrays / per_bucket must be non-NULL device pointers");
  if (ep && (ep->num_epochs < 1 || ep->epoch < 0 || ep->epoch >= ep->num_epochs))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay epoch: need 0 <= epoch < num_epochs");
  if (G < 1 || G > ORLOJ_REPLAY_MAX_SEGMENTS)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay: segments=%d outside 1..%d", G, ORLOJ_REPLAY_MAX_SEGMENTS);
  if (G > 1) {
    const size_t need = orloj_replay_seg_workspace(tr->num_scenarios, N, G, log != nullptr);
    if (N < 0)
      return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay: num_arrivals=%lld must be arrival_offsets[S]", (long long)N);
    if (need > 0 && (!ws || ((uintptr_t)ws & 255u) || ws_bytes < need))
      return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay: segments=%d need a 256-byte aligned device workspace of "
                  "%zu bytes (got %zu)", G, need, ws_bytes);
  }
  ReplayParams p;
  std::memset(&p, 0, sizeof(p));
  if ((st = compile_profile(profile, store->num_bins, ORLOJ_REPLAY_MAX_KMAX, &p.prof))) return st;
  const int B = store->num_bins, D = store->num_dists;
  const int bpl = bins_per_lane(B);
  const size_t store_b = (size_t)D * B * 4;
  if (store_b > (64u << 10))
    return fail(ORLOJ_ERR_CAPACITY, "replay: store of %zu bytes exceeds the 64 KiB shared-memory budget", store_b);
  const size_t warp_b = rate ? (bpl == 1 ? ReplayWarpSmem<1, true>::bytes()
                                         : bpl == 2 ? ReplayWarpSmem<2, true>::bytes() : ReplayWarpSmem<4, true>::bytes())
                             : (bpl == 1 ? ReplayWarpSmem<1>::bytes()
                                         : bpl == 2 ? ReplayWarpSmem<2>::bytes() : ReplayWarpSmem<4>::bytes());
  const size_t smem = replay_head_bytes(D, B) + REPLAY_WARPS * warp_b;
  p.log2F = store->log2_cdf;
  p.D = D;
  p.B = B;
  p.S = tr->num_scenarios;
  p.arr_off = tr->arrival_offsets;
  p.arrival = tr->arrival_ticks;
  p.dist = tr->dist_id;
  p.true_bin = tr->true_bin;
  p.slo = tr->slo_ticks;
  p.bucket = tr->bucket;
  p.counters = reinterpret_cast<unsigned long long *>(per_bucket);
  p.log = log;
  p.drop_thr = policy->drop_threshold_ticks;
  p.num_epochs = 1;
  if (ep) {
    p.epoch = ep->epoch;
    p.num_epochs = ep->num_epochs;
    p.t_carry = ep->worker_free_ticks;
    p.outcome = ep->outcome;
  }
  if (alg1) {
    p.size_thr = policy->size_threshold_ticks;
    p.prio_table = policy->priority_table;
    p.prio_logEL = policy->priority_log_expected;
    p.prio_b = policy->priority_b_per_tick;
  }
  if (p.S == 0) return ok();
  const unsigned blocks = (unsigned)((p.S + REPLAY_WARPS - 1) / REPLAY_WARPS);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (G == 1) {
    e = launch_replay<0>(p, bpl, rate, alg1, blocks, smem, s);
  } else {
    // segmented (exact, replay_kernel.cuh): speculative segments, then the stitch
    p.G = G;
    p.seg_stats = reinterpret_cast<unsigned long long *>(ws);
    p.seg = reinterpret_cast<ReplaySeg *>(reinterpret_cast<char *>(ws) + SEG_STATS_BYTES);
    p.seg_log = log ? reinterpret_cast<int32_t *>(reinterpret_cast<char *>(ws) + SEG_STATS_BYTES +
                                                  seg_state_bytes(p.S, G))
                    : nullptr;
    p.num_arrivals = N;
    const unsigned blocks_a = (unsigned)((p.S * G + REPLAY_WARPS - 1) / REPLAY_WARPS);
    e = cudaMemsetAsync(ws, 0, 32 * sizeof(unsigned long long), s);  // diagnostics head (read after the call)
    if (e == cudaSuccess) e = launch_replay<1>(p, bpl, rate, alg1, blocks_a, smem, s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = launch_replay<2>(p, bpl, rate, alg1, blocks, smem, s);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay_trace launch");
  return ok();
}


}  // namespace

extern "C" {

size_t orloj_replay_seg_workspace(int64_t num_scenarios, int64_t num_arrivals, int32_t segments,
                                  int32_t with_log) {
  if (num_scenarios <= 0 || segments <= 1) return 0;
  size_t b = SEG_STATS_BYTES + seg_state_bytes(num_scenarios, segments);
  if (with_log) b += align256((size_t)(2 * num_arrivals + num_scenarios * (int64_t)segments * 34) * sizeof(int32_t));
  return b;
}

orloj_status orloj_replay_trace(const orloj_store *store, const orloj_latency_profile *profile,
                                const orloj_trace *tr, orloj_counters *per_bucket, int32_t *log, void *stream) {
  ORLOJ_NVTX("orloj_replay_trace");
  const orloj_replay_policy def{ORLOJ_OBJ_EXPECTED_FINISH, nullptr, nullptr, nullptr, nullptr, 0.0};
  return orloj_replay_trace_ex(store, profile, tr, &def, per_bucket, log, stream);
}

orloj_status orloj_replay_trace_ex(const orloj_store *store, const orloj_latency_profile *profile,
                                   const orloj_trace *tr, const orloj_replay_policy *policy,
                                   orloj_counters *per_bucket, int32_t *log, void *stream) {
  ORLOJ_NVTX("orloj_replay_trace_ex");
  return replay_impl(store, profile, tr, policy, 1, 0, nullptr, 0, per_bucket, log, stream);
}

orloj_status orloj_replay_trace_seg(const orloj_store *store, const orloj_latency_profile *profile,
                                    const orloj_trace *tr, const orloj_replay_policy *policy, int32_t segments,
                                    int64_t num_arrivals, void *workspace, size_t workspace_bytes, orloj_counters *per_bucket,
                                    int32_t *log, void *stream) {
  ORLOJ_NVTX("orloj_replay_trace_seg");
  const orloj_replay_policy def{ORLOJ_OBJ_EXPECTED_FINISH, nullptr, nullptr, nullptr, nullptr, 0.0};
  return replay_impl(store, profile, tr, policy ? policy : &def, segments, num_arrivals, workspace, workspace_bytes, per_bucket,
                     log, stream);
}

orloj_status orloj_replay_trace_epoch(const orloj_store *store, const orloj_latency_profile *profile,
                                      const orloj_trace *tr, const orloj_replay_policy *policy,
                                      const orloj_replay_epoch *epoch, orloj_counters *per_bucket, int32_t *log,
                                      void *stream) {
  ORLOJ_NVTX("orloj_replay_trace_epoch");
  const orloj_replay_policy def{ORLOJ_OBJ_EXPECTED_FINISH, nullptr, nullptr, nullptr, nullptr, 0.0};
  if (!epoch) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay_trace_epoch: epoch descriptor is NULL");
  return replay_impl(store, profile, tr, policy ? policy : &def, 1, 0, nullptr, 0, per_bucket, log, stream, epoch);
}

size_t orloj_replay_feedback_workspace(int64_t num_scenarios, int64_t num_arrivals, int32_t num_dists,
                                       int32_t num_bins) {
  if (num_scenarios < 0 || num_arrivals < 0 || num_dists < 1 || num_bins < 1) return 0;
  return align256((size_t)num_scenarios * 8) + align256((size_t)num_arrivals) +
         align256((size_t)num_dists * num_bins * 4);
}

orloj_status orloj_replay_feedback(const orloj_store *store, const orloj_latency_profile *profile,
                                   const orloj_trace *tr, const orloj_replay_policy *policy,
                                   const orloj_feedback *fb, void *workspace, size_t workspace_bytes,
                                   orloj_counters *per_epoch_bucket, uint32_t *window_counts_out,
                                   int32_t *decision_logs, void *stream) {
  ORLOJ_NVTX("orloj_replay_feedback");
  orloj_status st;
  if ((st = check_store(store, ORLOJ_REPLAY_MAX_BINS))) return st;
  if (!fb || fb->num_epochs < 1 || fb->window_epochs < 1 || fb->min_samples < 1)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay_feedback: need num_epochs >= 1, window_epochs >= 1, "
                "min_samples >= 1");
  if (!tr || !per_epoch_bucket)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay_feedback: trace / per_epoch_bucket NULL");
  const int64_t S = tr->num_scenarios;
  const int32_t D = store->num_dists, B = store->num_bins;
  if (S < 0) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay_feedback: num_scenarios < 0");
  cudaStream_t s = (cudaStream_t)stream;
  // the arrival count sizes the outcome buffer: read arrival_offsets[S] (synchronous; off the hot path)
  int64_t N = 0;
  if (S > 0) {
    if (!tr->arrival_offsets) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay_feedback: arrival_offsets NULL");
    cudaError_t e = cudaMemcpyAsync(&N, tr->arrival_offsets + S, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "replay_feedback: reading arrival_offsets[S]");
  }
  const size_t need = orloj_replay_feedback_workspace(S, N, D, B);
  if (!workspace || ((uintptr_t)workspace & 255u) || workspace_bytes < need)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "replay_feedback: need a 256-byte aligned device workspace of %zu "
                "bytes (got %zu)", need, workspace_bytes);
  char *w = reinterpret_cast<char *>(workspace);
  int64_t *t_carry = reinterpret_cast<int64_t *>(w);
  uint8_t *outcome = reinterpret_cast<uint8_t *>(w + align256((size_t)S * 8));
  uint32_t *counts = reinterpret_cast<uint32_t *>(w + align256((size_t)S * 8) + align256((size_t)N));
  cudaError_t e = fill_i64(t_carry, S, INT64_MIN, s);  // the worker starts free
  if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, (size_t)D * B * 4, s);
  if (e != cudaSuccess) return cuda_fail(e, "replay_feedback: memset");
  float *rows = const_cast<float *>(store->log2_cdf);  // rewritten in place at every refresh (header)
  for (int32_t ep = 0; ep < fb->num_epochs; ++ep) {
    // (1) replay epoch ep with the current store (static during the epoch, A18)
    if (N > 0 && (e = cudaMemsetAsync(outcome, 0, (size_t)N, s)) != cudaSuccess)
      return cuda_fail(e, "replay_feedback: memset");
    const orloj_replay_epoch rep{ep, fb->num_epochs, t_carry, outcome};
    st = orloj_replay_trace_epoch(store, profile, tr, policy, &rep, per_epoch_bucket + (int64_t)ep * tr->num_buckets,
                                  decision_logs ? decision_logs + (int64_t)ep * (N + S) : nullptr, stream);
    if (st) return st;
    // (2) the profiler evaluates the sampled completed requests solo
    if ((st = orloj_profile_outcomes(tr->dist_id, tr->true_bin, outcome, fb->sample_mask, N, counts, D, B, stream)))
      return st;
    // (3) the scheduler picks the window up: rows with enough samples are rebuilt
    if ((st = orloj_store_refresh(counts, D, B, fb->min_samples, rows, stream))) return st;
    // (4) the profiling memory is reset every window_epochs epochs
    if (window_counts_out && ep == fb->num_epochs - 1 &&
        (e = cudaMemcpyAsync(window_counts_out, counts, (size_t)D * B * 4, cudaMemcpyDeviceToDevice, s)) !=
            cudaSuccess)
      return cuda_fail(e, "replay_feedback: copy of the window counts");
    if ((ep + 1) % fb->window_epochs == 0 && (e = cudaMemsetAsync(counts, 0, (size_t)D * B * 4, s)) != cudaSuccess)
      return cuda_fail(e, "replay_feedback: window reset");
  }
  return ok();
}

}  // extern "C"
