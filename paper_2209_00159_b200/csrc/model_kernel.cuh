// model_kernel.cuh — scoring-model variants: the
// expected finish count with
//   * a per-size duration table dur[k][m] (m = 0..B: the batch of k whose
//     slowest member sits at bin position m runs dur[k][m] ticks) — Eq. 3's
//     a_k + w_k m, or any non-decreasing grid (e.g. log-spaced bins);
//   * the bin model: mass at the upper bin edges (A1) or uniform within each
//     bin (linear CDF inside bins), the batch time then being the
//     table interpolated linearly between grid positions;
//   * a piecewise-step cost: deadlines D_r + off_s with cost
//     increments dc_s, i.e. the weighted finish count
//       E_k = sum_{r<=k} sum_s dc_s P(t + L_{B_k} <= D_r + off_s).
// With the Eq. 3 table, upper-edge bins and one unit step this is E_k of the
// main scorer.  Warp per queue (kmax <= 32: lane r = member r), the table
// and the (small) store staged in shared memory (a shared-memory binary
// search beat L1-cached global reads 25 us to 45 us at C2).  Not the C3 hot
// kernel: a variant for C2-sized workloads.
#pragma once
#include "common.cuh"

namespace orloj {

constexpr int MODEL_WARPS = 4;
constexpr int MODEL_MAX_STEPS = 8;
constexpr int MODEL_MAX_BINS = 128;

struct ModelParams {
  const float *log2F;
  int32_t D, B, kmax;
  int64_t Q;
  const int64_t *offsets, *deadline, *now;
  const int32_t *dist;
  const int64_t *dur;  // device [kmax][B+1]
  int32_t nsteps;
  int64_t off[MODEL_MAX_STEPS];
  float dc[MODEL_MAX_STEPS];
  bool smem_store;
  float *E;          // [Q][kmax]
  int32_t *best_k;   // [Q] or null
  float *best_E;     // [Q] or null
};

__host__ __device__ inline size_t model_smem_bytes(int kmax, int B, int D, bool smem_store) {
  return (size_t)kmax * (B + 1) * 8 + (smem_store ? (size_t)D * B * 4 : 0) +
         (size_t)MODEL_WARPS * ((B + 4) * 4 + 32 * 4 + 32 * 33 * 4);
}

template <bool INTERP>
__global__ void __launch_bounds__(MODEL_WARPS * 32) model_score_kernel(const __grid_constant__ ModelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int B = p.B, kmax = p.kmax;
  int64_t *s_dur = reinterpret_cast<int64_t *>(smem_raw);                     // [kmax][B+1]
  float *s_store = reinterpret_cast<float *>(s_dur + (size_t)kmax * (B + 1));  // [D][B] (smem_store)
  float *s_warp = s_store + (p.smem_store ? (size_t)p.D * B : 0);
  for (int e = threadIdx.x; e < kmax * (B + 1); e += blockDim.x) s_dur[e] = p.dur[e];
  if (p.smem_store)
    for (int e = threadIdx.x; e < p.D * B; e += blockDim.x) s_store[e] = p.log2F[e];
  __syncthreads();
  const float *store = p.smem_store ? s_store : p.log2F;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float *stg = s_warp + wid * ((B + 4) + 32 + 32 * 33) + 4;  // LG_k row, stg[-1] unused
  int32_t *s_d = reinterpret_cast<int32_t *>(stg + B);  // member distributions [32]
  float *part = reinterpret_cast<float *>(s_d + 32);      // [k-1][lane] partial sums, stride 33
  const int64_t q = (int64_t)blockIdx.x * MODEL_WARPS + wid;
  if (q >= p.Q) return;
  const int64_t base0 = p.offsets[0];
  const int64_t b0 = p.offsets[q] - base0;
  const int n = (int)(p.offsets[q + 1] - p.offsets[q]);
  const int K = n < kmax ? n : kmax;
  const int64_t t = p.now[q];
  const int64_t sig = lane < K ? p.deadline[b0 + lane] - t : 0;
  const int dr = lane < K ? p.dist[b0 + lane] : 0;
  s_d[lane] = dr;
  __syncwarp();
  float lg[MODEL_MAX_BINS / 32];
#pragma unroll
  for (int v = 0; v < MODEL_MAX_BINS / 32; ++v) lg[v] = 0.f;
  for (int k = 1; k <= K; ++k) {
    const int64_t *dk = s_dur + (size_t)(k - 1) * (B + 1);
    if (!INTERP) {
      const int d = s_d[k - 1];
#pragma unroll
      for (int v = 0; v < MODEL_MAX_BINS / 32; ++v) {
        const int e = 32 * v + lane;
        if (e < B) {
          lg[v] += store[(size_t)d * B + e];
          stg[e] = lg[v];
        }
      }
      __syncwarp();
    }
    float acc = 0.f;
    if (lane < k) {
      for (int s = 0; s < p.nsteps; ++s) {
        const int64_t x = sig + p.off[s];
        float P;
        // largest m in 0..B with dur[k][m] <= x (0 if none): branch-free
        // binary search with a fixed trip count (rows non-decreasing in m)
        int lo = 0;
#pragma unroll
        for (int st = MODEL_MAX_BINS; st > 0; st >>= 1)
          if (lo + st <= B && dk[lo + st] <= x) lo += st;
        if (!INTERP) {
          // i* = #{m in 1..B : dur[k][m] <= x}  (A1: mass at the upper edges)
          P = lo == 0 ? 0.f : ex2_approx(stg[lo - 1]);
        } else {
          // largest m in 0..B with dur[k][m] <= x; position m + u inside the grid
          if (x < dk[0]) {
            P = 0.f;
          } else {
            if (lo == B) {
              P = 1.f;
            } else {
              const float u = (float)((double)(x - dk[lo]) / (double)(dk[lo + 1] - dk[lo]));
              P = 1.f;
              for (int j = 0; j < k; ++j) {
                const float *row = store + (size_t)s_d[j] * B;
                const float f0 = lo == 0 ? 0.f : ex2_approx(row[lo - 1]);
                const float f1 = ex2_approx(row[lo]);
                P *= fmaf(u, f1 - f0, f0);
              }
            }
          }
        }
        acc = fmaf(p.dc[s], P, acc);
      }
    }
    part[(k - 1) * 33 + lane] = acc;  // reduced after the loop: no shuffle chain per k
    __syncwarp();
  }
  // E_k in lane k-1: sum of the members' partials (lanes >= k contributed 0)
  float E = 0.f;
  if (lane < K)
    for (int j = 0; j <= lane; ++j) E += part[lane * 33 + j];
  for (int k = K + 1 + lane; k <= kmax; k += 32) p.E[q * kmax + k - 1] = 0.f;
  if (lane < K) p.E[q * kmax + lane] = E;
  // argmax, ties -> smallest k (E >= 0: float bits order like values)
  const uint32_t bits = lane < K ? __float_as_uint(E) : 0u;
  const uint32_t mx = __reduce_max_sync(FULL, bits);
  const uint32_t kb = __reduce_min_sync(FULL, (lane < K && bits == mx) ? (uint32_t)(lane + 1) : 0x7fffffffu);
  if (lane == 0) {
    if (p.best_k) p.best_k[q] = K ? (int32_t)kb : 0;
    if (p.best_E) p.best_E[q] = K ? __uint_as_float(mx) : 0.f;
  }
}

}  // namespace orloj
