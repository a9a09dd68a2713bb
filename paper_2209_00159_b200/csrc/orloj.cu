// orloj.cu — liborloj.so: the C ABI declared in include/orloj.h.
//
// Host side: O(1) argument validation, profile compilation (division magic),
// template dispatch on (bins per lane, member slots), launches on the caller's
// stream.  No allocation and no global mutable state in the hot calls.
#include "../../include/orloj.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "host_util.h"
#include "score_launch.cuh"
#include "score_kernel.cuh"
#include "model_kernel.cuh"
#include "priority_kernel.cuh"
#include "store_kernel.cuh"

using namespace orloj;

namespace orloj {
namespace host {

thread_local std::string g_last_error;

orloj_status fail(orloj_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

orloj_status cuda_fail(cudaError_t e, const char *where) {
  return fail(ORLOJ_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

orloj_status ok() {
  g_last_error.clear();
  return ORLOJ_OK;
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

orloj_status check_store(const orloj_store *st, int max_bins) {
  if (!st) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store is NULL");
  if (st->num_dists < 1) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store.num_dists=%d < 1", st->num_dists);
  if (st->num_bins < 4 || st->num_bins % 4)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store.num_bins=%d must be a positive multiple of 4", st->num_bins);
  if (st->num_bins > max_bins)
    return fail(ORLOJ_ERR_CAPACITY, "store.num_bins=%d > %d", st->num_bins, max_bins);
  if (!st->log2_cdf || !aligned16(st->log2_cdf))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store.log2_cdf must be a 16-byte aligned device pointer");
  return ORLOJ_OK;
}

// Compile the profile into kernel parameters (A3, A14, horizon check).
orloj_status compile_profile(const orloj_latency_profile *pr, int32_t B, int kcap, ProfileDev *out) {
  if (!pr || !pr->offset_ticks || !pr->ticks_per_bin)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "profile or its arrays are NULL");
  if (pr->kmax < 1) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "profile.kmax=%d < 1", pr->kmax);
  if (pr->kmax > kcap) return fail(ORLOJ_ERR_CAPACITY, "profile.kmax=%d > %d", pr->kmax, kcap);
  std::memset(out, 0, sizeof(*out));
  out->kmax = pr->kmax;
  out->B = B;
  for (int k = 0; k < pr->kmax; ++k) {
    const int64_t a = pr->offset_ticks[k], w = pr->ticks_per_bin[k];
    if (a < 0 || w < 1)
      return fail(ORLOJ_ERR_INVALID_ARGUMENT, "profile k=%d: need a_k >= 0 and w_k >= 1 (got %lld, %lld)", k + 1,
                  (long long)a, (long long)w);
    if (k > 0 && (a < pr->offset_ticks[k - 1] || w < pr->ticks_per_bin[k - 1]))
      return fail(ORLOJ_ERR_INVALID_ARGUMENT, "profile must be non-decreasing in k (A14); violated at k=%d", k + 1);
    if (a > 0x3fffffffLL || w > 0x3fffffffLL || a + w * (int64_t)B > 0x3fffffffLL)
      return fail(ORLOJ_ERR_CAPACITY, "profile horizon a_k + w_k*B = %lld ticks exceeds 2^30-1 at k=%d",
                  (long long)(a + w * (int64_t)B), k + 1);
    uint32_t c = 0;
    while ((1ull << c) < (uint64_t)w) ++c;
    const uint64_t num = 1ull << (31 + c);
    const uint64_t m = (num + (uint64_t)w - 1) / (uint64_t)w;
    out->a[k] = (int32_t)a;
    out->w[k] = (int32_t)w;
    out->a2[k] = (int32_t)(2 * a);
    out->wB2[k] = (int32_t)(2 * w * B);
    out->mag[k] = (uint32_t)m;
    out->sh[k] = c;
  }
  return ORLOJ_OK;
}

orloj_status check_queues(const orloj_queues *q) {
  if (!q) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "queues is NULL");
  if (q->num_queues < 0) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "num_queues < 0");
  if (q->num_queues > 0 && (!q->queue_offsets || !q->deadline_ticks || !q->dist_id || !q->now_ticks))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "queue arrays must be non-NULL device pointers");
  return ORLOJ_OK;
}

cudaError_t fill_i64(int64_t *x, int64_t n, int64_t v, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t want = (n + 255) / 256;
  fill_i64_kernel<<<(unsigned)(want < 148 * 8 ? want : 148 * 8), 256, 0, s>>>(x, n, v);
  return cudaGetLastError();
}

int bins_per_lane(int B) { return B <= 32 ? 1 : B <= 64 ? 2 : B <= 128 ? 4 : 8; }
int slots_for(int kmax) {
  const int c = (kmax + 31) / 32;
  return c <= 1 ? 1 : c <= 2 ? 2 : c <= 4 ? 4 : 8;
}

}  // namespace host
}  // namespace orloj

using namespace orloj::host;

namespace {

cudaError_t launch_score(const ScoreParams &p, bool pick, int64_t store_bytes, cudaStream_t s) {
  const RowSrc src = store_bytes <= SMEM_STORE_BYTES ? RowSrc::Smem
                     : store_bytes > STREAM_STORE_BYTES ? RowSrc::TmaStream
                                                        : RowSrc::Tma;
  return pick ? launch_score_pick(p, src, s) : launch_score_all(p, src, s);
}

orloj_status prepare_score(const orloj_store *store, const orloj_latency_profile *profile,
                           const orloj_queues *queues, ScoreParams *p) {
  orloj_status st;
  if ((st = check_store(store, ORLOJ_MAX_BINS))) return st;
  if ((st = check_queues(queues))) return st;
  std::memset(p, 0, sizeof(*p));
  if ((st = compile_profile(profile, store->num_bins, ORLOJ_MAX_KMAX, &p->prof))) return st;
  p->log2F = store->log2_cdf;
  p->D = store->num_dists;
  p->B = store->num_bins;
  p->kmax = profile->kmax;
  p->Q = queues->num_queues;
  p->offsets = queues->queue_offsets;
  p->deadline = queues->deadline_ticks;
  p->dist = queues->dist_id;
  p->now = queues->now_ticks;
  return ORLOJ_OK;
}

int64_t store_bytes(const orloj_store *st) { return (int64_t)st->num_dists * st->num_bins * 4; }

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

orloj_status run_flag_check(unsigned int *dflag, cudaStream_t s, unsigned int *host_flag) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(host_flag, dflag, sizeof(unsigned), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(dflag, s);
  cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "validation");
  return ORLOJ_OK;
}

orloj_status alloc_flag(unsigned int **dflag, cudaStream_t s) {
  if (cudaMallocAsync((void **)dflag, sizeof(unsigned), s) != cudaSuccess)
    return fail(ORLOJ_ERR_OOM, "cannot allocate validation scratch");
  if (cudaMemsetAsync(*dflag, 0, sizeof(unsigned), s) != cudaSuccess)
    return fail(ORLOJ_ERR_CUDA, "memset of validation scratch failed");
  return ORLOJ_OK;
}

// TIER 0's g polynomial (priority_kernel.cuh): P(u) ~ G(u) = e^{-b} (1 - e^{-b u/2}) / u
// (G(0) = e^{-b} b / 2) on [0, U], the lowest degree D <= 5 that fits, by
// interpolation at the D + 1 Chebyshev nodes (a Vandermonde solve in v = u / U, then c_k = q_k / U^k),
// coefficients rounded to fp32.  Accepted when, on a grid of 257 points, the
// fit holds to 2^-23.5 relative (fp64 coefficients) and to 2^-22.5 with the fp32
// coefficients (each rounded once: 2^-24 of its term), and u P(u) stays far
// from the fp32 range for every |u| <= 2^31 (j = 0 rows: g finite).
bool prio_fit_g(double b, double U, float *c, int *degree) {
  constexpr int DMAX = 5;
  auto G = [&](double u) { return u > 0.0 ? std::exp(-b) * -std::expm1(-b * u / 2.0) / u : std::exp(-b) * b / 2.0; };
  // the lowest degree that fits (higher coefficients 0: no noise terms that
  // would blow up outside [0, U])
  for (int D = 0; D <= DMAX; ++D) {
    double q[DMAX + 1] = {0.0};
    if (U > 0.0 && D > 0) {
      double A[DMAX + 1][DMAX + 2];
      for (int i = 0; i <= D; ++i) {
        const double v = 0.5 * (1.0 + std::cos(M_PI * (i + 0.5) / (D + 1)));
        double pw = 1.0;
        for (int k = 0; k <= D; ++k, pw *= v) A[i][k] = pw;
        A[i][D + 1] = G(v * U);
      }
      for (int col = 0; col <= D; ++col) {  // Gauss-Jordan, partial pivoting
        int piv = col;
        for (int r = col + 1; r <= D; ++r)
          if (std::fabs(A[r][col]) > std::fabs(A[piv][col])) piv = r;
        for (int k = 0; k <= D + 1; ++k) std::swap(A[col][k], A[piv][k]);
        for (int r = 0; r <= D; ++r) {
          if (r == col) continue;
          const double f = A[r][col] / A[col][col];
          for (int k = col; k <= D + 1; ++k) A[r][k] -= f * A[col][k];
        }
      }
      double sc = 1.0;
      for (int k = 0; k <= D; ++k, sc /= U) q[k] = A[k][D + 1] / A[k][k] * sc;
    } else {
      q[0] = G(U / 2.0);
    }
    for (int k = 0; k <= DMAX; ++k) c[k] = (float)q[k];
    auto P = [&](double u, bool f32) {
      double r = f32 ? (double)c[DMAX] : q[DMAX];
      for (int k = DMAX - 1; k >= 0; --k) r = r * u + (f32 ? (double)c[k] : q[k]);
      return r;
    };
    bool ok = true;
    for (int i = 0; i <= 256 && ok; ++i) {
      const double u = U * i / 256.0;
      ok = std::fabs(P(u, false) / G(u) - 1.0) <= std::ldexp(1.0, -23.5) &&  // the fit
           std::fabs(P(u, true) / G(u) - 1.0) <= std::ldexp(1.0, -22.5);     // + fp32 coefficients
    }
    if (!ok) continue;
    *degree = D;
    double bound = 0.0;  // bounds |u P(u)| and every Horner partial times u for |u| <= 2^31
    for (int k = 0; k <= DMAX; ++k) bound += std::fabs((double)c[k]) * std::ldexp(1.0, 31 * (k + 1));
    return bound < 1e37;
  }
  return false;
}

template <bool SMEM_TABLE, bool STEPS, int TIER>
cudaError_t prio_launch(unsigned grid, size_t smem, cudaStream_t s, const double *log_table,
                        const double *log_expected, int32_t S, int32_t B, double b, const ProfileDev &prof,
                        const StepsDev &steps, const PrioCoef &cf, const orloj_queues *q, float *out,
                        const void *gtab) {
  static std::atomic<uint64_t> configured{0};  // per instantiation and device
  cudaError_t e = ensure_max_dyn_smem(priority_scores_kernel<SMEM_TABLE, STEPS, TIER>, 96 << 10, configured);
  if (e != cudaSuccess) return e;
  // one wave of resident blocks (grid-stride over queues): the per-size tables
  // are staged once per block
  static WaveCache wc;
  int64_t cap = 148;
  if ((e = one_wave(priority_scores_kernel<SMEM_TABLE, STEPS, TIER>, 256, smem, wc, &cap)) != cudaSuccess) return e;
  grid = (unsigned)((int64_t)grid < cap ? grid : cap);
  priority_scores_kernel<SMEM_TABLE, STEPS, TIER><<<grid, 256, smem, s>>>(
      log_table, log_expected, S, B, b, prof, steps, cf, q->num_queues, q->queue_offsets, q->deadline_ticks,
      q->now_ticks, out, gtab);
  return cudaGetLastError();
}

template <bool SMEM_TABLE, bool STEPS>
cudaError_t prio_launch_tier(int tier, unsigned grid, size_t smem, cudaStream_t s, const double *log_table,
                             const double *log_expected, int32_t S, int32_t B, double b, const ProfileDev &prof,
                             const StepsDev &steps, const PrioCoef &cf, const orloj_queues *q, float *out,
                             const void *gtab) {
  return tier == 0   ? prio_launch<SMEM_TABLE, STEPS, 0>(grid, smem, s, log_table, log_expected, S, B, b, prof,
                                                          steps, cf, q, out, gtab)
         : tier == 2 ? prio_launch<SMEM_TABLE, STEPS, 2>(grid, smem, s, log_table, log_expected, S, B, b, prof,
                                                          steps, cf, q, out, gtab)
                     : prio_launch<SMEM_TABLE, STEPS, 1>(grid, smem, s, log_table, log_expected, S, B, b, prof,
                                                          steps, cf, q, out, gtab);
}

orloj_status priority_scores_impl(const orloj_store *store, const orloj_latency_profile *profile, int32_t S,
                                  double b, const double *log_table, const double *log_expected,
                                  const orloj_queues *queues, const orloj_cost_steps *cs, float *out,
                                  void *stream) {
  orloj_status st;
  if ((st = check_store(store, ORLOJ_MAX_BINS))) return st;
  if ((st = check_queues(queues))) return st;
  ProfileDev prof;
  if ((st = compile_profile(profile, store->num_bins, ORLOJ_MAX_KMAX, &prof))) return st;
  if (S < 1 || S > profile->kmax || !(b > 0.0) || !log_table || !log_expected)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "priority_scores: need 1 <= num_sizes <= kmax, b > 0, tables");
  StepsDev steps;
  std::memset(&steps, 0, sizeof(steps));
  if (cs) {
    if (cs->num_steps < 1 || cs->num_steps > PRIO_MAX_STEPS || !cs->offset_ticks || !cs->cost)
      return fail(ORLOJ_ERR_INVALID_ARGUMENT, "cost steps: need 1..%d steps and both arrays", PRIO_MAX_STEPS);
    double prev_c = 0.0;
    for (int i = 0; i < cs->num_steps; ++i) {
      const int64_t o = cs->offset_ticks[i];
      const double dc = cs->cost[i] - prev_c;
      if ((i > 0 && o <= cs->offset_ticks[i - 1]) || o < -(1ll << 40) || o > (1ll << 40) || !(dc > 0.0))
        return fail(ORLOJ_ERR_INVALID_ARGUMENT,
                    "cost steps: offsets must increase (|offset| <= 2^40) and costs strictly increase from 0");
      steps.off[steps.n] = o;
      steps.logdc[steps.n] = (float)std::log(dc);
      steps.boff[steps.n] = b * (double)o;
      ++steps.n;
      prev_c = cs->cost[i];
    }
  }
  if (queues->num_queues == 0) return ok();
  if (!out) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "priority_scores: output is NULL");
  // Grid-stride over queues: ~resident blocks, so the per-size constants are
  // staged once per block, not once per 8 queues.
  const int B = store->num_bins;
  const int64_t want = (queues->num_queues + 7) / 8;
  const unsigned grid = (unsigned)(want < (1 << 30) ? want : (1 << 30));  // capped at one wave in prio_launch
  // Tier (priority_kernel.cuh): TIER 0 (strict-count lookup, fitted g) when
  // the fit holds and every horizon a_k + w_k B + 1 fits under the tier's slack
  // cap 2^30 - 2 - max w; else TIER 1.
  int32_t wmax = 0;
  for (int k = 0; k < S; ++k) wmax = prof.w[k] > wmax ? prof.w[k] : wmax;
  const int64_t cap0 = (1ll << 30) - 2 - wmax;
  PrioCoef cf;
  int deg = 5;
  bool t0 = b <= 0.05 && prio_fit_g(b, 2.0 * (wmax - 1), cf.c, &deg);
  for (int k = 0; k < S && t0; ++k) t0 = (int64_t)prof.a[k] + (int64_t)prof.w[k] * B + 1 <= cap0;
  const int tier = !t0 ? 1 : deg <= 4 ? 2 : 0;  // 0 / 2: fitted, degree 5 / <= 4
  cf.half_b = (float)(b / 2.0);
  cf.half_b_log2e = (float)(b / 2.0 * 1.4426950408889634);
  cf.gb = (float)(-std::expm1(-b));
  cf.cap = t0 ? (int32_t)cap0 : 0x3fffffff;
  // the re-based table in shared memory when it fits the budget, else in global memory
  const bool smem_table = PrioSmem::table_bytes(S, B, tier) <= (88u << 10);
  const size_t smem = PrioSmem::bytes(S, B, smem_table, tier);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  void *gtab = nullptr;
  if (!smem_table) {
    const int64_t ne = (int64_t)S * (B + 2);
    if (cudaMallocAsync(&gtab, (size_t)ne * PrioSmem::entry_bytes(tier), s) != cudaSuccess)
      return fail(ORLOJ_ERR_OOM, "priority_scores: cannot allocate the re-based table");
    if (tier != 1)  // the fitted tiers share one table layout
      priority_rebase_kernel<0><<<(unsigned)((ne + 255) / 256), 256, 0, s>>>(log_table, log_expected, S, B, b, prof,
                                                                            gtab);
    else
      priority_rebase_kernel<1><<<(unsigned)((ne + 255) / 256), 256, 0, s>>>(log_table, log_expected, S, B, b, prof,
                                                                            gtab);
  }
  if (cs)
    e = smem_table ? prio_launch_tier<true, true>(tier, grid, smem, s, log_table, log_expected, S, B, b, prof, steps,
                                                   cf, queues, out, gtab)
                   : prio_launch_tier<false, true>(tier, grid, smem, s, log_table, log_expected, S, B, b, prof, steps,
                                                    cf, queues, out, gtab);
  else
    e = smem_table ? prio_launch_tier<true, false>(tier, grid, smem, s, log_table, log_expected, S, B, b, prof, steps,
                                                    cf, queues, out, gtab)
                   : prio_launch_tier<false, false>(tier, grid, smem, s, log_table, log_expected, S, B, b, prof,
                                                     steps, cf, queues, out, gtab);
  if (gtab) cudaFreeAsync(gtab, s);
  if (e != cudaSuccess) return cuda_fail(e, "priority_scores launch");
  return ok();
}

}  // namespace

extern "C" {

const char *orloj_last_error(void) { return g_last_error.c_str(); }

int32_t orloj_abi_version(void) { return ORLOJ_ABI_VERSION; }

orloj_status orloj_store_build(const uint32_t *counts, int32_t D, int32_t B, float *out, void *stream) {
  ORLOJ_NVTX("orloj_store_build");
  if (!counts || !out || D < 1 || B < 4 || B % 4)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store_build: need counts, out, D >= 1, B a positive multiple of 4");
  if (B > ORLOJ_MAX_BINS) return fail(ORLOJ_ERR_CAPACITY, "store_build: B=%d > %d", B, ORLOJ_MAX_BINS);
  if (!aligned16(out)) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store_build: out must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned int *dflag;
  orloj_status st = alloc_flag(&dflag, s);
  if (st) return st;
  const int64_t threads = (int64_t)D * 32;
  store_build_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(counts, D, B, out, dflag);
  unsigned int hf = 0;
  if ((st = run_flag_check(dflag, s, &hf))) return st;
  if (hf) return fail(ORLOJ_ERR_COLD_START, "store_build: a histogram has total count 0 (cold start)");
  return ok();
}

orloj_status orloj_score_batches(const orloj_store *store, const orloj_latency_profile *profile,
                                 const orloj_queues *queues, float *E, float *P, float *EL, void *stream) {
  ORLOJ_NVTX("orloj_score_batches");
  ScoreParams p;
  orloj_status st = prepare_score(store, profile, queues, &p);
  if (st) return st;
  if (p.Q == 0) return ok();
  if (!E && !P && !EL) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "score_batches: no output requested");
  p.E = E;
  p.P = P;
  p.EL = EL;
  cudaError_t e = launch_score(p, false, store_bytes(store), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "score_batches launch");
  return ok();
}

orloj_status orloj_pick_batch(const orloj_store *store, const orloj_latency_profile *profile,
                              const orloj_queues *queues, int32_t *best_k, float *best_E, void *stream) {
  ORLOJ_NVTX("orloj_pick_batch");
  ScoreParams p;
  orloj_status st = prepare_score(store, profile, queues, &p);
  if (st) return st;
  if (p.Q == 0) return ok();
  if (!best_k || !best_E) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "pick_batch: best_k / best_expected NULL");
  p.best_k = best_k;
  p.best_E = best_E;
  cudaError_t e = launch_score(p, true, store_bytes(store), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "pick_batch launch");
  return ok();
}

constexpr int64_t ZERO_COPY_BYTES = 64 << 10;  // host arrays read in place below this size

size_t orloj_pick_batch_host_workspace(int64_t Q, int64_t N) {
  if (Q < 0 || N < 0) return 0;
  return align256((Q + 1) * 8) + align256(N * 8) + align256(N * 4) + align256(Q * 8) + align256(Q * 4) +
         align256(Q * 4);
}

orloj_status orloj_pick_batch_host(const orloj_store *store, const orloj_latency_profile *profile, int64_t Q,
                                   const int64_t *off_h, const int64_t *dl_h, const int32_t *dist_h,
                                   const int64_t *now_h, int32_t *bk_h, float *bE_h, void *ws, size_t ws_bytes,
                                   void *stream) {
  ORLOJ_NVTX("orloj_pick_batch_host");
  if (Q < 0 || !off_h || (Q > 0 && (!now_h || !bk_h || !bE_h)))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "pick_batch_host: bad host arrays");
  const int64_t N = off_h[Q] - off_h[0];
  if (N < 0 || (N > 0 && (!dl_h || !dist_h)))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "pick_batch_host: bad member arrays");
  // Small calls (a scheduler's per-decision call): when every host array is
  // pinned and mapped into the device address space (UVA), the kernel reads the
  // queues and writes k* / E* over PCIe directly — one launch, no copies.
  if ((Q + 1) * 8 + N * 12 + Q * 8 <= ZERO_COPY_BYTES) {
    const void *hp[6] = {off_h, dl_h, dist_h, now_h, bk_h, bE_h};
    void *dp[6];
    bool mapped = true;
    for (int i = 0; i < 6 && mapped; ++i) {
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, hp[i]) != cudaSuccess || at.type != cudaMemoryTypeHost || !at.devicePointer) {
        mapped = false;
        cudaGetLastError();
      } else {
        dp[i] = at.devicePointer;
      }
    }
    if (mapped) {
      orloj_queues q{Q, (const int64_t *)dp[0], nullptr, (const int64_t *)dp[1], (const int32_t *)dp[2],
                     (const int64_t *)dp[3]};
      return orloj_pick_batch(store, profile, &q, (int32_t *)dp[4], (float *)dp[5], stream);
    }
  }
  if (!ws || ((uintptr_t)ws & 255u) || ws_bytes < orloj_pick_batch_host_workspace(Q, N))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "pick_batch_host: workspace too small or misaligned");
  char *w = (char *)ws;
  int64_t *off_d = (int64_t *)w;  w += align256((Q + 1) * 8);
  int64_t *dl_d = (int64_t *)w;   w += align256(N * 8);
  int32_t *dist_d = (int32_t *)w; w += align256(N * 4);
  int64_t *now_d = (int64_t *)w;  w += align256(Q * 8);
  int32_t *bk_d = (int32_t *)w;   w += align256(Q * 4);
  float *bE_d = (float *)w;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(off_d, off_h, (Q + 1) * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && N) e = cudaMemcpyAsync(dl_d, dl_h, N * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && N) e = cudaMemcpyAsync(dist_d, dist_h, N * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && Q) e = cudaMemcpyAsync(now_d, now_h, Q * 8, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "pick_batch_host H2D");
  orloj_queues q{Q, off_d, nullptr, dl_d, dist_d, now_d};
  orloj_status st = orloj_pick_batch(store, profile, &q, bk_d, bE_d, stream);
  if (st) return st;
  if (Q) {
    e = cudaMemcpyAsync(bk_h, bk_d, Q * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bE_h, bE_d, Q * 4, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "pick_batch_host D2H");
  }
  return ok();
}

orloj_status orloj_score_model_batches(const orloj_store *store, const orloj_queues *queues,
                                       const orloj_score_model *model, float *E, int32_t *best_k, float *best_E,
                                       void *stream) {
  ORLOJ_NVTX("orloj_score_model_batches");
  orloj_status st;
  if ((st = check_store(store, MODEL_MAX_BINS))) return st;
  if ((st = check_queues(queues))) return st;
  if (!model || model->kmax < 1 || model->kmax > 32 || !model->duration_ticks ||
      (model->interpolate != 0 && model->interpolate != 1))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "score model: need 1 <= kmax <= 32, a duration table, interpolate 0/1");
  ModelParams p;
  std::memset(&p, 0, sizeof(p));
  if (model->num_steps == 0) {
    p.nsteps = 1;
    p.off[0] = 0;
    p.dc[0] = 1.f;
  } else {
    if (model->num_steps < 0 || model->num_steps > MODEL_MAX_STEPS || !model->step_offset_ticks || !model->step_cost)
      return fail(ORLOJ_ERR_INVALID_ARGUMENT, "score model: 0..%d steps with both arrays", MODEL_MAX_STEPS);
    double prev = 0.0;
    for (int i = 0; i < model->num_steps; ++i) {
      const int64_t o = model->step_offset_ticks[i];
      const double dc = model->step_cost[i] - prev;
      if ((i > 0 && o <= model->step_offset_ticks[i - 1]) || o < -(1ll << 40) || o > (1ll << 40) || !(dc > 0.0))
        return fail(ORLOJ_ERR_INVALID_ARGUMENT,
                    "score model steps: offsets must increase (|offset| <= 2^40), costs strictly increase from 0");
      p.off[i] = o;
      p.dc[i] = (float)dc;
      prev = model->step_cost[i];
    }
    p.nsteps = model->num_steps;
  }
  if (queues->num_queues == 0) return ok();
  if (!E) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "score model: expected_finish is NULL");
  p.log2F = store->log2_cdf;
  p.D = store->num_dists;
  p.B = store->num_bins;
  p.kmax = model->kmax;
  p.Q = queues->num_queues;
  p.offsets = queues->queue_offsets;
  p.deadline = queues->deadline_ticks;
  p.now = queues->now_ticks;
  p.dist = queues->dist_id;
  p.dur = model->duration_ticks;
  p.E = E;
  p.best_k = best_k;
  p.best_E = best_E;
  p.smem_store = (int64_t)p.D * p.B * 4 <= (32 << 10);
  const size_t smem = model_smem_bytes(p.kmax, p.B, p.D, p.smem_store);
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)((p.Q + MODEL_WARPS - 1) / MODEL_WARPS);
  cudaError_t e;
  // row analysis (arithmetic grids -> exact division): the caller's plan, or a
  // stream-ordered scratch analysed now
  ModelRow *rows = nullptr;
  if (model->plan) {
    p.rows = static_cast<const ModelRow *>(model->plan);
  } else {
    if (cudaMallocAsync((void **)&rows, 32 * sizeof(ModelRow), s) != cudaSuccess)
      return fail(ORLOJ_ERR_OOM, "score model: cannot allocate the row scratch");
    model_prep_kernel<<<1, 256, 0, s>>>(p.dur, p.kmax, p.B, rows);
    p.rows = rows;
  }
  const bool one = p.nsteps == 1 && p.off[0] == 0 && p.dc[0] == 1.f;
  if (model->interpolate) {
    e = cudaFuncSetAttribute(model_interp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) model_interp_kernel<<<grid, MODEL_WARPS * 32, smem, s>>>(p);
  } else {
    // upper-edge model: the score_small layout (rows first, butterfly sums), B <= 32 BPL
    const int bpl = p.B <= 32 ? 1 : p.B <= 64 ? 2 : 4;
    const size_t sm = bpl == 1 ? ModelEdgeShape<1>::bytes(p.kmax, p.B, p.D, p.smem_store)
                      : bpl == 2 ? ModelEdgeShape<2>::bytes(p.kmax, p.B, p.D, p.smem_store)
                                 : ModelEdgeShape<4>::bytes(p.kmax, p.B, p.D, p.smem_store);
    auto go = [&](auto kern) {
      cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (r == cudaSuccess) kern<<<grid, MODEL_WARPS * 32, sm, s>>>(p);
      return r;
    };
    if (bpl == 1) e = one ? go(model_edge_kernel<1, true>) : go(model_edge_kernel<1, false>);
    else if (bpl == 2) e = one ? go(model_edge_kernel<2, true>) : go(model_edge_kernel<2, false>);
    else e = one ? go(model_edge_kernel<4, true>) : go(model_edge_kernel<4, false>);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (rows) cudaFreeAsync(rows, s);
  if (e != cudaSuccess) return cuda_fail(e, "score_model launch");
  return ok();
}

orloj_status orloj_score_model_prepare(const orloj_score_model *model, int32_t num_bins, void *plan, void *stream) {
  ORLOJ_NVTX("orloj_score_model_prepare");
  static_assert(32 * sizeof(ModelRow) <= ORLOJ_SCORE_MODEL_PLAN_BYTES, "plan size");
  if (!model || model->kmax < 1 || model->kmax > 32 || !model->duration_ticks || !plan || num_bins < 1 ||
      num_bins > MODEL_MAX_BINS)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "score_model_prepare: need a model (1 <= kmax <= 32), 1 <= B <= %d, plan",
                MODEL_MAX_BINS);
  model_prep_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(model->duration_ticks, model->kmax, num_bins,
                                                          static_cast<ModelRow *>(plan));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "score_model_prepare launch");
  return ok();
}

orloj_status orloj_priority_table(const orloj_store *store, const orloj_latency_profile *profile, int32_t S,
                                  const float *weights, double b, double *log_table, double *log_expected,
                                  void *stream) {
  ORLOJ_NVTX("orloj_priority_table");
  orloj_status st;
  if ((st = check_store(store, ORLOJ_MAX_BINS))) return st;
  ProfileDev prof;
  if ((st = compile_profile(profile, store->num_bins, ORLOJ_MAX_KMAX, &prof))) return st;
  if (S < 1 || S > profile->kmax || !(b > 0.0) || !log_table || !log_expected)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "priority_table: need 1 <= num_sizes <= kmax, b > 0, outputs");
  for (int k = 0; k < S; ++k)
    if (!(b * prof.w[k] < 700.0)) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "priority_table: b * w_%d >= 700", k + 1);
  cudaStream_t s = (cudaStream_t)stream;
  priority_table_kernel<<<S, 128, (size_t)store->num_bins * 8, s>>>(store->log2_cdf, store->num_dists,
                                                                     store->num_bins, weights, prof, b, log_table,
                                                                     log_expected);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "priority_table");
  return ok();
}


orloj_status orloj_priority_scores(const orloj_store *store, const orloj_latency_profile *profile, int32_t S,
                                   double b, const double *log_table, const double *log_expected,
                                   const orloj_queues *queues, float *out, void *stream) {
  ORLOJ_NVTX("orloj_priority_scores");
  return priority_scores_impl(store, profile, S, b, log_table, log_expected, queues, nullptr, out, stream);
}

orloj_status orloj_priority_scores_steps(const orloj_store *store, const orloj_latency_profile *profile, int32_t S,
                                         double b, const double *log_table, const double *log_expected,
                                         const orloj_queues *queues, const orloj_cost_steps *steps, float *out,
                                         void *stream) {
  ORLOJ_NVTX("orloj_priority_scores_steps");
  if (!steps) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "priority_scores_steps: steps is NULL");
  return priority_scores_impl(store, profile, S, b, log_table, log_expected, queues, steps, out, stream);
}

orloj_status orloj_pop_batch(const orloj_queues *queues, const float *logp, int32_t S, const int32_t *bs,
                             int32_t *sel, void *stream) {
  ORLOJ_NVTX("orloj_pop_batch");
  orloj_status st;
  if ((st = check_queues(queues))) return st;
  if (S < 1) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "pop_batch: num_sizes < 1");
  if (queues->num_queues == 0) return ok();
  if (!logp || !bs || !sel) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "pop_batch: NULL array");
  const int64_t threads = (queues->num_queues + POP_QPW - 1) / POP_QPW * 32;  // POP_QPW queues per warp
  pop_batch_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      logp, S, queues->num_queues, queues->queue_offsets, bs, sel);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pop_batch launch");
  return ok();
}

orloj_status orloj_histogram_accumulate(const int32_t *dist_id, const int64_t *solo_ticks, int64_t n,
                                        int64_t bin_ticks, uint32_t *counts, int32_t D, int32_t B, void *stream) {
  ORLOJ_NVTX("orloj_histogram_accumulate");
  if (n < 0 || D < 1 || B < 1 || bin_ticks <= 0 || !counts || (n > 0 && (!dist_id || !solo_ticks)))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "histogram_accumulate: bad sizes or pointers");
  if ((int64_t)D * B > (1ll << 30)) return fail(ORLOJ_ERR_CAPACITY, "histogram_accumulate: D*B too large");
  if (n == 0) return ok();
  const size_t hb = (size_t)D * B * 4;
  const int use_smem = hb <= (48u << 10);
  const int64_t want = (n + 255) / 256;
  const unsigned blocks = (unsigned)(want < 148 * 8 ? want : 148 * 8);
  hist_accumulate_kernel<<<blocks, 256, use_smem ? hb : 0, (cudaStream_t)stream>>>(dist_id, solo_ticks, n, bin_ticks,
                                                                                    counts, D, B, use_smem);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "histogram_accumulate launch");
  return ok();
}

orloj_status orloj_profile_outcomes(const int32_t *dist_id, const int16_t *true_bin, const uint8_t *outcome,
                                    const uint8_t *sample_mask, int64_t n, uint32_t *counts, int32_t D, int32_t B,
                                    void *stream) {
  ORLOJ_NVTX("orloj_profile_outcomes");
  if (n < 0 || D < 1 || B < 1 || !counts || (n > 0 && (!dist_id || !true_bin || !outcome)))
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "profile_outcomes: bad sizes or pointers");
  if ((int64_t)D * B > (1ll << 30)) return fail(ORLOJ_ERR_CAPACITY, "profile_outcomes: D*B too large");
  if (n == 0) return ok();
  const size_t hb = (size_t)D * B * 4;
  const int use_smem = hb <= (48u << 10);
  const int64_t want = (n + 255) / 256;
  const unsigned blocks = (unsigned)(want < 148 * 8 ? want : 148 * 8);
  profile_outcomes_kernel<<<blocks, 256, use_smem ? hb : 0, (cudaStream_t)stream>>>(
      dist_id, true_bin, outcome, sample_mask, n, counts, D, B, use_smem);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "profile_outcomes launch");
  return ok();
}

orloj_status orloj_store_refresh(const uint32_t *counts, int32_t D, int32_t B, uint32_t min_samples, float *out,
                                 void *stream) {
  ORLOJ_NVTX("orloj_store_refresh");
  if (!counts || !out || D < 1 || B < 4 || B % 4)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store_refresh: need counts, out, D >= 1, B a positive multiple of 4");
  if (B > ORLOJ_MAX_BINS) return fail(ORLOJ_ERR_CAPACITY, "store_refresh: B=%d > %d", B, ORLOJ_MAX_BINS);
  if (!aligned16(out)) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store_refresh: out must be 16-byte aligned");
  const int64_t threads = (int64_t)D * 32;
  store_build_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      counts, D, B, out, nullptr, min_samples > 1 ? (uint64_t)min_samples : 1ull);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "store_refresh launch");
  return ok();
}

orloj_status orloj_validate_store(const orloj_store *store, void *stream) {
  ORLOJ_NVTX("orloj_validate_store");
  orloj_status st;
  if ((st = check_store(store, ORLOJ_MAX_BINS))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned int *dflag;
  if ((st = alloc_flag(&dflag, s))) return st;
  validate_store_kernel<<<148 * 8, 256, 0, s>>>(store->log2_cdf, store->num_dists, store->num_bins, dflag);
  unsigned hf = 0;
  if ((st = run_flag_check(dflag, s, &hf))) return st;
  if (hf) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "store rows must be non-decreasing, <= 0, and end with 0.0f");
  return ok();
}

orloj_status orloj_validate_queues(const orloj_store *store, const orloj_queues *q, void *stream) {
  ORLOJ_NVTX("orloj_validate_queues");
  orloj_status st;
  if ((st = check_store(store, ORLOJ_MAX_BINS))) return st;
  if ((st = check_queues(q))) return st;
  if (q->num_queues == 0) return ok();
  cudaStream_t s = (cudaStream_t)stream;
  unsigned int *dflag;
  if ((st = alloc_flag(&dflag, s))) return st;
  validate_queues_kernel<<<148 * 8, 256, 0, s>>>(q->queue_offsets, q->num_queues, q->arrival_ticks,
                                                  q->deadline_ticks, q->dist_id, store->num_dists, dflag);
  unsigned hf = 0;
  if ((st = run_flag_check(dflag, s, &hf))) return st;
  if (hf & 1u) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "queues: bad offsets or dist_id out of range");
  if (hf & 2u) return fail(ORLOJ_ERR_UNSORTED, "queues: members not in (deadline, arrival, index) order");
  return ok();
}

orloj_status orloj_validate_trace(const orloj_store *store, const orloj_trace *tr, void *stream) {
  ORLOJ_NVTX("orloj_validate_trace");
  orloj_status st;
  if ((st = check_store(store, ORLOJ_REPLAY_MAX_BINS))) return st;
  if (!tr || tr->num_scenarios < 0 || tr->num_buckets < 1)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "trace: need num_scenarios >= 0 and num_buckets >= 1");
  if (tr->num_scenarios == 0) return ok();
  cudaStream_t s = (cudaStream_t)stream;
  unsigned int *dflag;
  if ((st = alloc_flag(&dflag, s))) return st;
  validate_trace_kernel<<<148 * 8, 256, 0, s>>>(tr->arrival_offsets, tr->num_scenarios, tr->arrival_ticks,
                                                 tr->dist_id, tr->true_bin, tr->slo_ticks, tr->bucket,
                                                 tr->num_buckets, store->num_dists, store->num_bins, dflag);
  unsigned hf = 0;
  if ((st = run_flag_check(dflag, s, &hf))) return st;
  if (hf & 1u) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "trace: offsets / ids / bins / buckets / slo out of range");
  if (hf & 2u) return fail(ORLOJ_ERR_UNSORTED, "trace: arrivals not non-decreasing within a scenario");
  return ok();
}

}  // extern "C"
