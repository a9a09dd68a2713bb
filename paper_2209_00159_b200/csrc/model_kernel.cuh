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
// search beat L1-cached global reads 25 us to 45 us at C2).  Each block also
// checks every row for an arithmetic grid dur[m] = dur[0] + w m (Eq. 3); such
// a row is searched by the main scorer's exact integer division (umulhi by a
// magic constant, common.cuh lookup_bin) instead of the 8-step binary search
// -- the same m, so the same results.  The upper-edge model runs in
// model_edge_kernel (the main short-queue scorer's layout), the within-bin-
// uniform (interpolated) one in model_interp_kernel.  Not the C3 hot kernel:
// a variant for C2-sized workloads.
#pragma once
#include "common.cuh"

namespace orloj {

constexpr int MODEL_WARPS = 4;
constexpr int MODEL_MAX_STEPS = 8;
constexpr int MODEL_MAX_BINS = 128;

// Arithmetic-grid description of a duration row dur[m] = a + w m (Eq. 3) in
// the main scorer's lookup form (common.cuh lookup_bin: doubled slack, division
// magic); bit 31 of shl set = the row is such a grid (else: search the table).
struct ModelRow {
  int32_t a2, wB2;  // 2 a, 2 w B  (a + w B <= 2^30 - 1)
  uint32_t mag, shl;
};
__device__ __forceinline__ bool model_lin(const ModelRow &r) { return (r.shl >> 31) != 0; }
__device__ __forceinline__ int model_lookup(const ModelRow &r, int32_t s2) {
  return lookup_bin(s2, r.a2, r.wB2, r.mag, r.shl & 31u);
}

struct ModelParams {
  const float *log2F;
  int32_t D, B, kmax;
  int64_t Q;
  const int64_t *offsets, *deadline, *now;
  const int32_t *dist;
  const int64_t *dur;  // device [kmax][B+1]
  const struct ModelRow *rows;  // device [32] (model_prep_kernel)
  int32_t nsteps;
  int64_t off[MODEL_MAX_STEPS];
  float dc[MODEL_MAX_STEPS];
  bool smem_store;
  float *E;          // [Q][kmax]
  int32_t *best_k;   // [Q] or null
  float *best_E;     // [Q] or null
};

// shared memory of model_interp_kernel
__host__ __device__ inline size_t model_smem_bytes(int kmax, int B, int D, bool smem_store) {
  return (size_t)kmax * (B + 1) * 8 + (size_t)32 * sizeof(ModelRow) + (smem_store ? (size_t)D * B * 4 : 0) +
         (size_t)MODEL_WARPS * (32 * 4 + 32 * 33 * 4);
}

// One block (orloj_score_model_prepare, or once per call without a plan): mark
// each row of the duration table that is an arithmetic grid dur[m] = dur[0] +
// w m (w >= 1, dur[0] >= 0, horizon below 2^30) and give it the division
// magic of common.cuh lookup_bin.
// All threads check entries in parallel (shared-memory OR per row).
static __global__ void model_prep_kernel(const int64_t *__restrict__ dur, int kmax, int B, ModelRow *__restrict__ rows) {
  __shared__ int bad[32];
  if (threadIdx.x < 32) bad[threadIdx.x] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < kmax * (B + 1); e += blockDim.x) {
    const int k = e / (B + 1), m = e - k * (B + 1);
    const int64_t *d = dur + (size_t)k * (B + 1);
    if (d[m] != d[0] + (d[1] - d[0]) * m) atomicOr(&bad[k], 1);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    ModelRow r{};
    const int k = threadIdx.x;
    if (k < kmax) {
      const int64_t *d = dur + (size_t)k * (B + 1);
      const int64_t a = d[0], w = d[1] - d[0];
      if (bad[k] == 0 && a >= 0 && w >= 1 && a + w * B <= 0x3fffffffll) {
        uint32_t c = 0;
        while ((1ull << c) < (uint64_t)w) ++c;
        r.a2 = (int32_t)(2 * a);
        r.wB2 = (int32_t)(2 * w * B);
        r.mag = (uint32_t)(((1ull << (31 + c)) + (uint64_t)w - 1) / (uint64_t)w);
        r.shl = c | 0x80000000u;
      }
    }
    rows[k] = r;
  }
}

// Largest m in 0..B with dk[m] <= x (0 if none): branch-free binary search with
// a fixed trip count (rows non-decreasing in m).  Out of line: the edge kernel
// unrolls its size loop, and only a row that is not an arithmetic grid calls it.
__device__ __forceinline__ int model_search_inl(const int64_t *dk, int B, int64_t x) {
  int lo = 0;
#pragma unroll
  for (int s2 = MODEL_MAX_BINS; s2 > 0; s2 >>= 1)
    if (lo + s2 <= B && dk[lo + s2] <= x) lo += s2;
  return lo;
}
__device__ __noinline__ int model_search(const int64_t *dk, int B, int64_t x) {
  int lo = 0;
#pragma unroll
  for (int s2 = MODEL_MAX_BINS; s2 > 0; s2 >>= 1)
    if (lo + s2 <= B && dk[lo + s2] <= x) lo += s2;
  return lo;
}

// Within-bin-uniform (interpolated) model: P_r(k) = prod_{j<=k} F_j^lin(m + u)
// is not a prefix sum of logs, so no LG rows: warp per queue, for k = 1..K
// lanes r < k evaluate their own product over the members j <= k (O(K^3) per
// queue, the model's own cost); per-k partial sums reduced once after the loop.
__global__ void __launch_bounds__(MODEL_WARPS * 32) model_interp_kernel(const __grid_constant__ ModelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int B = p.B, kmax = p.kmax;
  int64_t *s_dur = reinterpret_cast<int64_t *>(smem_raw);                          // [kmax][B+1]
  ModelRow *s_row = reinterpret_cast<ModelRow *>(s_dur + (size_t)kmax * (B + 1));  // [32]
  float *s_store = reinterpret_cast<float *>(s_row + 32);                           // [D][B] (smem_store)
  float *s_warp = s_store + (p.smem_store ? (size_t)p.D * B : 0);
  for (int e = threadIdx.x; e < kmax * (B + 1); e += blockDim.x) s_dur[e] = p.dur[e];
  // the model reads F itself: stage 2^{log2 F} (the same ex2_approx per entry as
  // an in-loop conversion, once per block instead of per use)
  if (p.smem_store)
    for (int e = threadIdx.x; e < p.D * B; e += blockDim.x) s_store[e] = ex2_approx(p.log2F[e]);
  if (threadIdx.x < 32) s_row[threadIdx.x] = p.rows[threadIdx.x];
  __syncthreads();
  const float *store = p.smem_store ? s_store : p.log2F;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t *s_d = reinterpret_cast<int32_t *>(s_warp + wid * (32 + 32 * 33));  // member distributions [32]
  float *part = reinterpret_cast<float *>(s_d + 32);                           // [k-1][lane] partials, stride 33
  const int64_t q = (int64_t)blockIdx.x * MODEL_WARPS + wid;
  if (q >= p.Q) return;
  const int64_t base0 = p.offsets[0];
  const int64_t b0 = p.offsets[q] - base0;
  const int n = (int)(p.offsets[q + 1] - p.offsets[q]);
  const int K = n < kmax ? n : kmax;
  const int64_t t = p.now[q];
  const int64_t sig = lane < K ? p.deadline[b0 + lane] - t : 0;
  s_d[lane] = lane < K ? p.dist[b0 + lane] : 0;
  __syncwarp();
  for (int k = 1; k <= K; ++k) {
    const int64_t *dk = s_dur + (size_t)(k - 1) * (B + 1);
    const ModelRow rk = s_row[k - 1];
    float acc = 0.f;
    if (lane < k) {
      for (int st = 0; st < p.nsteps; ++st) {
        const int64_t x = sig + p.off[st];
        // largest m in 0..B with dur[k][m] <= x (0 if none): exact division on a
        // grid row (warp-uniform), else the fixed-trip binary search
        const int lo = model_lin(rk) ? model_lookup(rk, sigma2(x)) : model_search_inl(dk, B, x);
        float P;
        if (x < dk[0]) {
          P = 0.f;
        } else if (lo == B) {
          P = 1.f;
        } else {  // position m + u inside the grid
          const float u = (float)((double)(x - dk[lo]) / (double)(dk[lo + 1] - dk[lo]));
          P = 1.f;
          for (int j = 0; j < k; ++j) {
            const float *row = store + (size_t)s_d[j] * B;
            const float f0 = lo == 0 ? 0.f : (p.smem_store ? row[lo - 1] : ex2_approx(row[lo - 1]));
            const float f1 = p.smem_store ? row[lo] : ex2_approx(row[lo]);
            P *= fmaf(u, f1 - f0, f0);
          }
        }
        acc = fmaf(p.dc[st], P, acc);
      }
    }
    part[(k - 1) * 33 + lane] = acc;  // reduced after the loop: no shuffle chain per k
  }
  __syncwarp();
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


// Upper-edge bin model (interpolate = 0), the score_small_kernel layout
// (score_small_kernel.cuh): the warp builds LG_1..LG_K of its queue first
// (lanes over bins, rows with a -inf head), then lane r-1 owns member r and for
// k = 1..32 (unrolled) finds its position m in row k of the duration table
// (exact division on an arithmetic grid, else the fixed-trip binary search),
// P_r(k) = 2^{LG_k[m]} (head: m = 0, P = 0), summed over the cost steps, and
// pushes it into the transposing butterfly that leaves E_k in lane k-1.  No
// per-k barrier or partial-sum matrix: the rows are built before any lookup.
template <int BPL>
struct ModelEdgeShape {
  static constexpr int ROW = 32 * BPL + 1;
  __host__ __device__ static size_t bytes(int kmax, int B, int D, bool smem_store) {
    return (size_t)kmax * (B + 1) * 8 + (size_t)32 * sizeof(ModelRow) + (smem_store ? (size_t)D * B * 4 : 0) +
           (size_t)MODEL_WARPS * 32 * ROW * 4;
  }
};

template <int BPL, bool ONE>
__global__ void __launch_bounds__(MODEL_WARPS * 32) model_edge_kernel(const __grid_constant__ ModelParams p) {
  constexpr int ROW = ModelEdgeShape<BPL>::ROW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int B = p.B, kmax = p.kmax;
  int64_t *s_dur = reinterpret_cast<int64_t *>(smem_raw);                          // [kmax][B+1]
  ModelRow *s_row = reinterpret_cast<ModelRow *>(s_dur + (size_t)kmax * (B + 1));  // [32]
  float *s_store = reinterpret_cast<float *>(s_row + 32);                           // [D][B] (smem_store)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float *lgs = s_store + (p.smem_store ? (size_t)p.D * B : 0) + (size_t)wid * 32 * ROW;  // row k-1 = LG_k
  // the queue's offsets / now are requested before the block stages its tables,
  // so their latency overlaps the staging and the barriers
  const int64_t q = (int64_t)blockIdx.x * MODEL_WARPS + wid;
  const bool live = q < p.Q;
  int64_t o0 = 0, o1 = 0, t = 0;
  if (live) {
    o0 = p.offsets[q];
    o1 = p.offsets[q + 1];
    t = p.now[q];
  }
  const int64_t base0 = p.offsets[0];
  if (p.smem_store)
    for (int e = threadIdx.x; e < p.D * B; e += blockDim.x) s_store[e] = p.log2F[e];
  lgs[lane * ROW] = -INFINITY;
  bool lin = true;
  if (threadIdx.x < 32) {
    const ModelRow r = p.rows[threadIdx.x];
    s_row[threadIdx.x] = r;
    lin = (int)threadIdx.x >= kmax || model_lin(r);
  }
  const bool all_lin = __syncthreads_and(lin);  // block-uniform
  if (!all_lin)  // some row is not an arithmetic grid: stage the table for its search
    for (int e = threadIdx.x; e < kmax * (B + 1); e += blockDim.x) s_dur[e] = p.dur[e];
  __syncthreads();
  const float *store = p.smem_store ? s_store : p.log2F;
  if (!live) return;
  const int64_t b0 = o0 - base0;
  const int n = (int)(o1 - o0);
  const int K = n < kmax ? n : kmax;
  const int64_t sig = lane < K ? p.deadline[b0 + lane] - t : 0;
  const int32_t s2 = sigma2(sig);  // ONE: the one unit step at offset 0
  const int dr = lane < K ? p.dist[b0 + lane] : 0;

  float E = 0.f;
  if (ONE && all_lin && p.smem_store) {
    // one unit step, every row an arithmetic grid (Eq. 3), store in shared memory: the short-queue
    // scorer's register-row form (score_small_kernel.cuh) — LG_k held across the
    // lanes, member lane+1 looked up in it by one shuffle right after row k is
    // added, no staged rows; the same adds, ex2 and butterfly as the staged form
    // below, so the values are identical
    float acc[BPL];
#pragma unroll
    for (int e = 0; e < BPL; ++e) acc[e] = 0.f;
    int col[BPL];
#pragma unroll
    for (int e = 0; e < BPL; ++e) col[e] = min(32 * e + lane, B - 1);  // lanes past the last bin: never looked up
    float pend[5];
    const int nlane = -lane;
    uint32_t ca[BPL];  // 32-bit shared-space address of the lane's column in row 0
#pragma unroll
    for (int e = 0; e < BPL; ++e) ca[e] = smem_base(s_store) + 4u * (uint32_t)col[e];
    const uint32_t rb = smem_base(s_row);
    const int dB4 = dr * B * 4;  // byte offset of member lane+1's row
#pragma unroll
    for (int k = 1; k <= 32; ++k) {
      const uint32_t ro = (uint32_t)__shfl_sync(FULL, dB4, k - 1);  // rows past K: row 0, reach only E_k > K
#pragma unroll
      for (int e = 0; e < BPL; ++e) acc[e] += lds_f32_nv(ca[e] + ro);
      const int4 rk = lds_v4s32(rb + 16u * (uint32_t)(k - 1));  // ModelRow {a2, wB2, mag, shl}
      const int m = lookup_bin(s2, rk.x, rk.y, (uint32_t)rk.z, (uint32_t)rk.w & 31u);  // 1-based bin, 0: none
      const int from = m - 1;                         // shfl takes the lane mod 32
      float lg = __shfl_sync(FULL, acc[0], from);
#pragma unroll
      for (int e = 1; e < BPL; ++e) {
        const float o = __shfl_sync(FULL, acc[e], from);
        lg = (from >> 5) == e ? o : lg;
      }
      const float x = ex2_approx(lg);
      E = bfly_push(pend, min(nlane + (k - 1), from) >= 0 ? x : 0.f, k - 1, lane);  // r <= k and m > 0
    }
  } else {
  // LG_k for k = 1..K (the same fp32 adds in the same order as the main scorer)
  float acc[BPL];
#pragma unroll
  for (int e = 0; e < BPL; ++e) acc[e] = 0.f;
  for (int k = 0; k < K; ++k) {
    const float *row = store + (size_t)__shfl_sync(FULL, dr, k) * B;
#pragma unroll
    for (int e = 0; e < BPL; ++e) {
      const int i = 32 * e + lane;
      if (i < B) {
        acc[e] += row[i];
        lgs[k * ROW + 1 + i] = acc[e];
      }
    }
  }
  __syncwarp();

  const uint32_t row0 = opaque_u32(smem_addr(lgs));
  if (all_lin) {
    // every row an arithmetic grid: per cost step the main scorer's loop, no
    // branch per size (rows k > K are stale; they reach only E_k, k > K,
    // unused); the butterfly is linear, so the steps' sums add up (one unit
    // step: E = 1 * sum exactly)
#pragma unroll 1
    for (int st = 0; st < (ONE ? 1 : p.nsteps); ++st) {
      const int32_t s2s = ONE ? s2 : sigma2(sig + p.off[st]);
      float pend[5], Es = 0.f;
#pragma unroll
      for (int k = 1; k <= 32; ++k) {
        const float x =
            ex2_approx(lds_f32_nv(row0 + 4u * (uint32_t)((k - 1) * ROW + model_lookup(s_row[k - 1], s2s))));
        Es = bfly_push(pend, lane < k ? x : 0.f, k - 1, lane);
      }
      E = fmaf(ONE ? 1.f : p.dc[st], Es, E);
    }
  } else {
  float pend[5];
#pragma unroll
  for (int k = 1; k <= 32; ++k) {
    float v = 0.f;
    if (k <= K) {  // warp-uniform
      const ModelRow rk = s_row[k - 1];
      const int64_t *dk = s_dur + (size_t)(k - 1) * (B + 1);
      const uint32_t lk = row0 + 4u * (uint32_t)((k - 1) * ROW);
      if (ONE) {
        // i* = #{m >= 1 : dur[k][m] <= sigma} (A1: mass at the upper edges); lk[0] = -inf gives P = 0
        const int lo = model_lin(rk) ? model_lookup(rk, s2) : model_search(dk, B, sig);
        v = ex2_approx(lds_f32_nv(lk + 4u * (uint32_t)lo));
      } else {
#pragma unroll 1
        for (int st = 0; st < p.nsteps; ++st) {
          const int64_t x = sig + p.off[st];
          const int lo = model_lin(rk) ? model_lookup(rk, sigma2(x)) : model_search(dk, B, x);
          v = fmaf(p.dc[st], ex2_approx(lds_f32_nv(lk + 4u * (uint32_t)lo)), v);
        }
      }
      v = lane < k ? v : 0.f;  // members r <= k
    }
    E = bfly_push(pend, v, k - 1, lane);
  }
  }
  }  // staged rows
  const int k = lane + 1;
  const bool valid = k <= K;
  for (int kk = K + 1 + lane; kk <= kmax; kk += 32) p.E[q * kmax + kk - 1] = 0.f;
  if (valid) p.E[q * kmax + lane] = E;
  const uint32_t bits = valid ? __float_as_uint(E) : 0u;
  const uint32_t mx = __reduce_max_sync(FULL, bits);
  const uint32_t kb = __reduce_min_sync(FULL, (valid && bits == mx) ? (uint32_t)k : 0x7fffffffu);
  if (lane == 0) {
    if (p.best_k) p.best_k[q] = K ? (int32_t)kb : 0;
    if (p.best_E) p.best_E[q] = K ? __uint_as_float(mx) : 0.f;
  }
}

}  // namespace orloj
