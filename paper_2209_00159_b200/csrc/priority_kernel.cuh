// priority_kernel.cuh — Eq. 1-2 priority scores and PopBatch (SURVEY §8(f)
// item 2; PAPER.md:423-455 Eq. 1-2, :585-593 batch formation, :306-373 Alg. 1).
//
// Batch latency of size bs (Eq. 3-4, 6, 9 with the A1 grid): a batch of bs
// requests drawn from the mixture of all application distributions
// has its latency in bin i = (l1, l2] = (a + w(i-1), a + w i] with probability
// pm_i = F_mix(tau_i)^bs - F_mix(tau_{i-1})^bs, spread uniformly over the bin
// (the histogram of Eq. 2, density h_i = pm_i / w).  Priority (Eq. 1, c = 1,
// tau ~ Exp(b)) with slack sigma = D - t, summed per bin as Eq. 2:
//   full bins (l2 <= sigma):  (h/b) (e^{b l2} - e^{b l1}) e^{-b sigma}
//   partial bin (l1 < sigma < l2): (h/b) (1 - e^{-b (sigma - l1)})
// divided by E[L] = sum_i pm_i (l1 + l2) / 2.  In the log domain (no overflow
// at any b or t): with the prefix
//   C[i] = log sum_{j<=i} (h_j/b) e^{b l1_j} (e^{b w} - 1)          (C[0] = -inf)
// and i* = #bins with l2 <= sigma (the scorer's exact integer lookup),
//   log p = logaddexp(C[i*] - b sigma, log(h_{i*+1}/b) + log(-expm1(-b (sigma - l1_{i*+1}))))
//           - log E[L].
// C changes only at the milestones sigma = l_i: p(t) = alpha e^{bt} + beta.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace orloj {

// Order-preserving key of a float (larger float -> larger unsigned key).
__device__ __forceinline__ uint32_t fkey(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}


// One block per batch size: mixture CDF, pmf of the max of bs draws, E[L],
// the full-bin prefix C[0..B] and the per-bin log(h_i / b) H[0..B] (H[0] =
// -inf), all fp64.  table layout [S][2][B+1]: [s][0][i] = C[i], [s][1][i] = H[i].
static __global__ void priority_table_kernel(const float *__restrict__ log2F, int32_t D, int32_t B,
                                      const float *__restrict__ weights, const __grid_constant__ ProfileDev prof,
                                      double b, double *__restrict__ table, double *__restrict__ logEL) {
  extern __shared__ double s_mix[];  // [B]
  const int bs = blockIdx.x + 1;
  double wsum = 0.0;
  for (int d = 0; d < D; ++d) wsum += weights ? (double)weights[d] : 1.0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    double f = 0.0;
    for (int d = 0; d < D; ++d) f += (weights ? (double)weights[d] : 1.0) * exp2((double)log2F[(int64_t)d * B + i]);
    s_mix[i] = i == B - 1 ? 1.0 : f / wsum;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double a = prof.a[bs - 1], w = prof.w[bs - 1];
  double *C = table + (int64_t)(bs - 1) * 2 * (B + 1);
  double *H = C + (B + 1);
  C[0] = -INFINITY;
  H[0] = -INFINITY;
  const double lgw = log(expm1(b * w));  // log(e^{bw} - 1)
  const double lwb = log(w * b);
  // log G_i = bs log F_mix(tau_i) and log pm_i = log G_i + log(1 - G_{i-1}/G_i):
  // no underflow (F^bs leaves the fp64 range for small F and large bs)
  double prevlG = -INFINITY, acc = -INFINITY, mean_bin = 0.0;
  for (int i = 1; i <= B; ++i) {
    const double lG = s_mix[i - 1] > 0.0 ? (double)bs * log(s_mix[i - 1]) : -INFINITY;
    const double lpm = lG > prevlG ? lG + log(-expm1(prevlG - lG)) : -INFINITY;
    prevlG = lG;
    mean_bin += exp(lpm) * (i - 0.5);
    double h = -INFINITY;
    if (lpm > -INFINITY) {
      h = lpm - lwb;
      const double x = h + b * (a + w * (i - 1)) + lgw;
      const double m = acc > x ? acc : x;
      acc = m + log(exp(acc - m) + exp(x - m));
    }
    C[i] = acc;
    H[i] = h;
  }
  logEL[bs - 1] = log(a + w * mean_bin);
}

// Score kernel (orloj_priority_scores).  Warp per queue (grid-stride over
// queues: a block stages the per-size constants once and reuses them for many
// queues), lanes over members, chunks of PRIO_CHUNK members per lane with the
// size loop outside the member loop.  No fp64 and no branch per element: the
// fp64 tables are re-based once per block into an fp32 table in shared memory
// so that the full-bin term is one FFMA.
//
// TIER 1 (any b, any profile): entry (k, i), i = 0..B, is {C'_i, H'_{i+1}} with
//   C'_i = C[i] - b l2_i - log E[L]   (l2_i = a_k + w_k i; -inf where C = -inf)
//   H'_{i+1} = H[i+1] - log E[L]      (-inf at i = B: no bin beyond the last).
// The scorer's lookup gives i = i*(sigma) and the exact integer x = sigma - l2_i:
//   log p(full bins) = C[i] - b sigma - log E[L] = C'_i - b x,
// and with x > 0, i < B (x is then sigma - l1_{i+1} in (0, w)) the partial bin
//   log p = log(e^{lp} + e^{H'} g),  g = 1 - e^{-b x}   (prio_combine, general g).
//
// TIERS 0 / 2 (when the host's polynomial fit below holds and every
// horizon a_k + w_k B + 1 is under the tier's slack cap; the P1 case): a
// strict-count lookup
//   j = #bins with l2 < sigma, + 1   (= floor((sigma - 1 - a + w) / w) clamped to [0, B+1])
// puts sigma in bin j with x = sigma - l1_j in (0, w] for 1 <= j <= B (a full
// last bin is the same value as a partial one at x = w), j = B+1 beyond the
// last bin, and j = 0 exactly when sigma <= a (p = 0).  Entry (k, j), j = 0..B+1:
//   {C[j-1] - b l1_j - b - log E[L],  H[j] - log E[L]},   entry 0 = {-inf, -inf},
//   H'_{B+1} = -inf.
// With u = 2 (x - 1) (an exact integer from the lookup, no select):
//   lp = T.x - (b/2) u,   g = g_b + e_b g(b u / 2) = g_b + u P(u)
// (g_b = 1 - e^{-b}, e_b = e^{-b}; both terms positive, no cancellation).  P is
// a degree-5 polynomial fitted by the host (Chebyshev interpolation of
// e_b (1 - e^{-b u/2}) / u on [0, 2 (max w - 1)], fp64, coefficients rounded
// to fp32, then checked on a grid: 2^-23.5 relative for the fit, 2^-22.5 with the fp32 coefficients;
// degree 5 is TIER 0, degree <= 4 TIER 2, no fit TIER 1; a relative error e in g
// moves log p by at most e, 2^-22.5 = 1.7e-7 against the 1e-6 + 2^-22 |log p| budget).  j = 0
// gives lp = Hn = -inf: prio_combine returns -inf (the host also checks that P
// is finite for every u the cap allows).
//
// C' <= -log E[L] (each full-bin term is at most pm_j), so |C'| + b x = |log p|
// whenever E[L] >= 1 tick: the fp32 re-based form keeps the 2^-23 relative
// bound of an fp64 full-bin term.  Slack above the tier's cap (the
// last entry there: the cap is above every profile's horizon) adds
// b (sigma - cap) in a warp-uniform slow path.
// Output [S][N] (size-major: each store of a warp is one contiguous 128-B line,
// and PopBatch reads one size row coalesced).
// Table entries: TIER 0 float4 {C', H', D2 = (C' - H') log2 e, 0} (the log-add-exp's
// exponent in one FFMA), TIER 1 float2 {C', H'}.
// Tiers: 1 = general; 0 and 2 = the fitted-polynomial form (degree 5 and <= 4).
__host__ __device__ constexpr bool prio_fitted(int tier) { return tier != 1; }
template <int TIER> using PrioEntry = typename std::conditional<prio_fitted(TIER), float4, float2>::type;
struct PrioSmem {
  static __host__ __device__ size_t entry_bytes(int tier) { return prio_fitted(tier) ? 16 : 8; }
  static __host__ __device__ size_t table_bytes(int S, int B, int tier) { return (size_t)S * (B + 2) * entry_bytes(tier); }
  static __host__ __device__ size_t bytes(int S, int B, bool smem_table, int tier) {
    return (size_t)S * (16 + 8) + (smem_table ? table_bytes(S, B, tier) : 0);
  }
};

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// g = 1 - e^{-t}, t = b x >= 0: the Taylor series to t^8 below t = 1/2
// (truncation < 2^-26 relative, no cancellation), else 1 - 2^{-t log2 e}
// (g > 0.39 there).  Both sides evaluated, one select (no divergence).
__device__ __forceinline__ float prio_g_general(float t) {
  float c = -1.f / 40320.f;
  c = fmaf(c, t, 1.f / 5040.f);
  c = fmaf(c, t, -1.f / 720.f);
  c = fmaf(c, t, 1.f / 120.f);
  c = fmaf(c, t, -1.f / 24.f);
  c = fmaf(c, t, 1.f / 6.f);
  c = fmaf(c, t, -0.5f);
  c = fmaf(c, t, 1.f);
  const float big = 1.f - ex2_approx(-t * 1.4426950408889634f);
  return t < 0.5f ? c * t : big;
}

// The partial bin of Eq. 2 in the log domain: log(e^lp + e^Hn g).  With
// d = -|lp - Hn| one term of the sum is exactly 1:
//   lp >= Hn:  lp + log(1 + e^d g),   else  Hn + log(e^d + g),
// two MUFU (ex2, lg2).  Hn = -inf (no partial bin) gives e = 0, y = 1 and lp
// exactly; lp = Hn = -inf gives d = NaN, clamped to -150 (e = 0 after ftz),
// and -inf.  g must be finite.
__device__ __forceinline__ float prio_combine(float lp, float Hn, float g) {
  const float e = ex2_approx(fmaxf(-fabsf(lp - Hn) * 1.4426950408889634f, -150.f));
  const bool hi = lp >= Hn;
  const float y = hi ? fmaf(e, g, 1.f) : e + g;
  return fmaf(0.6931471805599453f, lg2_approx(y), hi ? lp : Hn);
}

// Pre-rebasing form kept for the replay's Alg. 1 PopBatch (replay_kernel.cuh),
// which scores one window at a time from the fp64 global tables.
__device__ __forceinline__ float prio_partial(float lp, float Hn, float t) {
  return prio_combine(lp, Hn, prio_g_general(t));
}

// One element of the score kernel with the table read from global memory
// (tab_k = table + (k-1) 2 (B+1)), fp64 full-bin term: the replay's Alg. 1 path.
__device__ __forceinline__ float prio_elem_global(const double *__restrict__ tab_k, double lEL, int B, int4 lk,
                                                  int32_t w, int32_t s2, double bsig, float bf) {
  const int i = lookup_bin(s2, lk.x, lk.y, (uint32_t)lk.z, (uint32_t)lk.w);
  const int32_t x = ((s2 - lk.x) >> 1) - w * i;
  const double Ci = tab_k[i] - lEL;
  const float Hn = (i < B && x > 0) ? (float)(tab_k[B + 1 + i + 1] - lEL) : -INFINITY;
  const float lp = (float)(Ci + bsig);
  return prio_combine(lp, Hn, prio_g_general(bf * (float)(x > 0 ? x : 0)));
}

constexpr int PRIO_CHUNK = 8;  // members per lane per pass
#ifdef PRIO_MIN_BLOCKS  // experiments: -DPRIO_MIN_BLOCKS=5 caps registers for 5 resident blocks per SM
#define PRIO_BOUNDS __launch_bounds__(256, PRIO_MIN_BLOCKS)
#else
#define PRIO_BOUNDS __launch_bounds__(256)
#endif
constexpr int PRIO_MAX_STEPS = 8;

// Piecewise-step cost: deadlines D_r + off[s] with cost
// increments dc[s] = c_s - c_{s-1} > 0; p = sum_s dc[s] p_single(sigma + off[s]).
struct StepsDev {
  int32_t n;
  int64_t off[PRIO_MAX_STEPS];
  float logdc[PRIO_MAX_STEPS];   // log dc[s]
  double boff[PRIO_MAX_STEPS];   // b off[s]
};

// Per-call constants of the g tiers (host-computed in fp64, rounded once).
struct PrioCoef {
  float half_b;  // b / 2
  float half_b_log2e;  // b / 2 log2 e
  float gb;      // 1 - e^{-b}
  float c[6];    // P(u) = c0 + c1 u + ... + c5 u^5 (TIER 0, host-fitted)
  int32_t cap;   // slack cap (ticks) of the tier's lookup
};

__device__ __forceinline__ float logaddexpf_(float a, float b) {
  const float M = fmaxf(a, b);
  return M == -INFINITY ? M : M + log1pf(__expf(fminf(a, b) - M));
}

// Slack of a member, clamped to [0, cap] and doubled.
__device__ __forceinline__ int32_t prio_s2(int64_t sigma, int32_t cap) {
  return 2 * (int32_t)(sigma < 0 ? 0 : sigma > cap ? cap : sigma);
}

// Per-size constants in shared memory: lk = {lookup offset, 2 w (bins+1), mag,
// sh}, nw2 = -2 w (TIER 0) or -w (TIER 1).
template <int TIER>
__device__ __forceinline__ int4 prio_lk(const ProfileDev &prof, int k, int B) {
  return prio_fitted(TIER) ? make_int4(2 * (prof.a[k] + 1 - prof.w[k]), 2 * prof.w[k] * (B + 1), (int)prof.mag[k],
                               (int)prof.sh[k])
                   : make_int4(prof.a2[k], prof.wB2[k], (int)prof.mag[k], (int)prof.sh[k]);
}

// Re-based table entry (k, e) of the tier (layout above; stride B+2).
template <int TIER>
__device__ __forceinline__ PrioEntry<TIER> prio_entry(const double *__restrict__ table,
                                                      const double *__restrict__ logEL, const ProfileDev &prof, int B,
                                                      double b, int k, int e) {
  const double lEL = logEL[k];
  const double *tab = table + (size_t)k * 2 * (B + 1);
  const double a = prof.a[k], w = prof.w[k];
  if constexpr (prio_fitted(TIER)) {
    // D2 = (C' - H') log2 e from the fp64 values, rounded once; +inf when H' = -inf
    // (also when C' = -inf too: the y = 1 branch then returns lp = -inf, p = 0),
    // so the exponent is never NaN and needs no clamp
    if (e == 0) return make_float4(-INFINITY, -INFINITY, INFINITY, 0.f);
    const double C = tab[e - 1];
    const double Cr = C == -INFINITY ? -INFINITY : C - b * (a + w * (e - 1)) - b - lEL;
    const double Hr = e <= B ? tab[B + 1 + e] - lEL : -INFINITY;
    const double D2 = Hr == -INFINITY ? INFINITY : (Cr - Hr) * 1.4426950408889634;
    return make_float4((float)Cr, (float)Hr, (float)D2, 0.f);
  } else {
    if (e > B) return make_float2(-INFINITY, -INFINITY);  // unused pad
    const double C = tab[e];
    return make_float2(C == -INFINITY ? -INFINITY : (float)(C - b * (a + w * e) - lEL),
                       e < B ? (float)(tab[B + 1 + e + 1] - lEL) : -INFINITY);
  }
}

// Table row of one size: shared (a 32-bit shared-space address taken after the
// staging barrier, so the non-volatile loads depend on it and stay below the
// barrier) or global (tables above the shared-memory budget).
struct PrioTabS {
  uint32_t base;
  template <class E>
  __device__ __forceinline__ E ld(int j) const {
    E v;
    if constexpr (sizeof(E) == 16)
      asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
          : "r"(base + 16u * (uint32_t)j));
    else
      asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(base + 8u * (uint32_t)j));
    return v;
  }
};
struct PrioTabG {
  const unsigned char *p;  // row base (entries of the tier's type)
  template <class E>
  __device__ __forceinline__ E ld(int j) const { return __ldg(reinterpret_cast<const E *>(p) + j); }
};

// The log-add-exp of TIER 0 with its exponent d2 = (lp - Hn) log2 e given:
// log(e^lp + e^Hn g) = (d2 >= 0 ? lp : Hn) + log(1 + 2^-|d2| g  or  2^-|d2| + g)
// (prio_combine with d2 from one FFMA of the table's D2, which is +inf
// wherever Hn = -inf, so no clamp: 2^-inf = 0 after ftz).
__device__ __forceinline__ float prio_combine_d2(float lp, float Hn, float d2, float g) {
  const float e = ex2_approx(-fabsf(d2));  // d2 is never NaN (the table's D2, prio_entry)
  const bool hi = d2 >= 0.f;
  const float y = hi ? fmaf(e, g, 1.f) : e + g;
  return fmaf(0.6931471805599453f, lg2_approx(y), hi ? lp : Hn);
}

// log p of one (member, size): s2 = prio_s2(sigma), tk the size's re-based
// table row, bxe = b (sigma - cap) above the cap, else 0.
template <int TIER, class Tab>
__device__ __forceinline__ float prio_elem(const Tab &tk, const int4 &lk, int32_t nw, int32_t s2, float bf,
                                           const PrioCoef &cf, float bxe) {
  const int32_t x2 = s2 - lk.x;
  int32_t xc = x2 < lk.y ? x2 : lk.y;
  xc = xc > 0 ? xc : 0;
  const int j = (int)(__umulhi((uint32_t)xc, (uint32_t)lk.z) >> (uint32_t)lk.w);
  const PrioEntry<TIER> T = tk.template ld<PrioEntry<TIER>>(j);
  if constexpr (prio_fitted(TIER)) {
    const float u = (float)(x2 + nw * j);  // 2 (x - 1), x = sigma - l1_j
    const float lp = fmaf(-cf.half_b, u, T.x) - bxe;
    const float d2 = fmaf(-cf.half_b_log2e, u, T.z) - bxe * 1.4426950408889634f;  // (lp - Hn) log2 e
    float c;
    if constexpr (TIER == 0) {  // degree 5
      c = fmaf(cf.c[5], u, cf.c[4]);
      c = fmaf(c, u, cf.c[3]);
    } else {  // degree <= 4 (TIER 2)
      c = fmaf(cf.c[4], u, cf.c[3]);
    }
    c = fmaf(c, u, cf.c[2]);
    c = fmaf(c, u, cf.c[1]);
    c = fmaf(c, u, cf.c[0]);
    return prio_combine_d2(lp, T.y, d2, fmaf(u, c, cf.gb));
  } else {
    const int32_t x = (x2 >> 1) + nw * j;  // sigma - l2_i
    const float Hn = x > 0 ? T.y : -INFINITY;
    const float xf = (float)x;
    const float lp = fmaf(-bf, xf, T.x) - bxe;
    return prio_combine(lp, Hn, prio_g_general(bf * fmaxf(xf, 0.f)));
  }
}

// The size loop of one chunk (Tab: shared or global rows).
template <int TIER, bool STEPS, class Tab>
__device__ __forceinline__ void prio_chunk(const Tab &t0, int32_t rowb, const int4 *s_lk, const int2 *s_wk, int S,
                                           float *out0, int64_t N, int nv, unsigned mode, const int64_t (&sg)[PRIO_CHUNK],
                                           const int32_t (&s2)[PRIO_CHUNK], const float (&bxe)[PRIO_CHUNK],
                                           double b, float bf, const PrioCoef &cf, const StepsDev &steps);

template <bool SMEM_TABLE, bool STEPS, int TIER>
__global__ void PRIO_BOUNDS priority_scores_kernel(
    const double *__restrict__ table, const double *__restrict__ logEL, int32_t S, int32_t B, double b,
    const __grid_constant__ ProfileDev prof, const __grid_constant__ StepsDev steps, const PrioCoef cf, int64_t Q,
    const int64_t *__restrict__ offsets, const int64_t *__restrict__ deadline, const int64_t *__restrict__ now,
    float *__restrict__ out, const void *__restrict__ gtab) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int4 *s_lk = reinterpret_cast<int4 *>(smem_raw);       // [S]
  int2 *s_wk = reinterpret_cast<int2 *>(s_lk + S);      // [S] {nw, unused}
  PrioEntry<TIER> *s_T = reinterpret_cast<PrioEntry<TIER> *>(s_wk + S);  // [S][B+2] (SMEM_TABLE)
  for (int k = threadIdx.x; k < S; k += blockDim.x) {
    s_lk[k] = prio_lk<TIER>(prof, k, B);
    s_wk[k] = make_int2(prio_fitted(TIER) ? -2 * prof.w[k] : -prof.w[k], 0);
  }
  if (SMEM_TABLE)
    for (int e = threadIdx.x; e < S * (B + 2); e += blockDim.x) {
      const int k = e / (B + 2);
      s_T[e] = prio_entry<TIER>(table, logEL, prof, B, b, k, e - k * (B + 2));
    }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float bf = (float)b;
  const int64_t base0 = offsets[0], N = offsets[Q] - base0;
  const int64_t wpb = blockDim.x >> 5;
  const int32_t cap = cf.cap;
  const bool vec_ok = (N & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(deadline) & 15) == 0;

  for (int64_t q = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); q < Q; q += (int64_t)gridDim.x * wpb) {
    const int64_t b0 = offsets[q] - base0, e0 = offsets[q + 1] - base0;
    const int64_t t = now[q];
    for (int64_t c0 = b0; c0 < e0; c0 += 32 * PRIO_CHUNK) {
      // Member of (lane, m): the strided map c0 + lane + 32 m, or (a full chunk
      // at a 4-aligned start, aligned arrays) the vector map c0 + 128 (m / 4) +
      // 4 lane + m % 4: each lane loads 4 consecutive deadlines (2 x 16 B) and
      // stores 4 consecutive scores (16 B) per size.
      const bool vec = vec_ok && e0 - c0 >= 32 * PRIO_CHUNK && (c0 & 3) == 0;  // warp-uniform
      const int64_t rem = e0 - c0 - lane;
      const int nv = vec ? PRIO_CHUNK : rem <= 0 ? 0 : rem >= 32 * PRIO_CHUNK ? PRIO_CHUNK : (int)((rem + 31) >> 5);
      int64_t sg[PRIO_CHUNK];   // sigma
      int32_t s2[PRIO_CHUNK];
      float bxe[PRIO_CHUNK];    // b (sigma - cap) above the cap, else 0
      bool over = false;
      // all loads first, unconditional (a lane past the queue end re-reads the
      // last member: in bounds, never stored), so they are in flight together
      int64_t dl[PRIO_CHUNK];
      if (vec) {
#pragma unroll
        for (int h = 0; h < PRIO_CHUNK / 4; ++h) {
          const longlong2 *p2 = reinterpret_cast<const longlong2 *>(deadline + c0 + 128 * h + 4 * lane);
          const longlong2 x0 = __ldg(p2), x1 = __ldg(p2 + 1);
          dl[4 * h] = x0.x;
          dl[4 * h + 1] = x0.y;
          dl[4 * h + 2] = x1.x;
          dl[4 * h + 3] = x1.y;
        }
      } else {
#pragma unroll
        for (int m = 0; m < PRIO_CHUNK; ++m) {
          const int64_t j = c0 + lane + 32 * m;
          dl[m] = __ldg(deadline + (j < e0 ? j : e0 - 1));
        }
      }
#pragma unroll
      for (int m = 0; m < PRIO_CHUNK; ++m) {
        const int64_t sigma = m < nv ? dl[m] - t : 0;
        sg[m] = sigma;
        s2[m] = prio_s2(sigma, cap);
        over |= sigma > cap;
      }
      over = __any_sync(0xffffffffu, over);
#pragma unroll
      for (int m = 0; m < PRIO_CHUNK; ++m) bxe[m] = over && sg[m] > cap ? (float)(b * (double)(sg[m] - cap)) : 0.f;
      // warp-uniform specialisations: a full chunk stores unpredicated, the
      // vector map stores 16 B, and only a chunk with a slack above the cap
      // pays the extra subtraction
      const unsigned mode = (over ? 1u : 0u) | (__all_sync(0xffffffffu, nv == PRIO_CHUNK) ? 2u : 0u) | (vec ? 4u : 0u);
      float *out0 = out + c0 + (vec ? 4 * lane : lane);
      if (SMEM_TABLE)
        prio_chunk<TIER, STEPS>(PrioTabS{smem_base(s_T)}, (int32_t)sizeof(PrioEntry<TIER>) * (B + 2), s_lk, s_wk, S,
                                out0, N, nv, mode, sg, s2, bxe, b, bf, cf, steps);
      else
        prio_chunk<TIER, STEPS>(PrioTabG{static_cast<const unsigned char *>(gtab)},
                                (int32_t)sizeof(PrioEntry<TIER>) * (B + 2), s_lk, s_wk, S, out0, N, nv, mode, sg, s2,
                                bxe, b, bf, cf, steps);
    }
  }
}

// One size's scores of a chunk: PRED stores only members m < nv; VEC stores
// groups of 4 consecutive members as one 16-B store (out at ok + 128 (m / 4)).
template <int TIER, bool PRED, bool OVER, bool VEC, class Tab>
__device__ __forceinline__ void prio_size(const Tab &tk, const int4 &lk, int32_t nw, float *ok, int nv,
                                          const int32_t (&s2)[PRIO_CHUNK], const float (&bxe)[PRIO_CHUNK], float bf,
                                          const PrioCoef &cf) {
  float r[PRIO_CHUNK];
#pragma unroll
  for (int m = 0; m < PRIO_CHUNK; ++m) r[m] = prio_elem<TIER>(tk, lk, nw, s2[m], bf, cf, OVER ? bxe[m] : 0.f);
  if (VEC) {
#pragma unroll
    for (int h = 0; h < PRIO_CHUNK / 4; ++h)
      *reinterpret_cast<float4 *>(ok + 128 * h) = make_float4(r[4 * h], r[4 * h + 1], r[4 * h + 2], r[4 * h + 3]);
  } else {
#pragma unroll
    for (int m = 0; m < PRIO_CHUNK; ++m)
      if (!PRED || m < nv) ok[32 * m] = r[m];
  }
}

template <int TIER, bool STEPS, class Tab>
__device__ __forceinline__ void prio_chunk(const Tab &t0, int32_t rowb, const int4 *s_lk, const int2 *s_wk, int S,
                                           float *out0, int64_t N, int nv, unsigned mode, const int64_t (&sg)[PRIO_CHUNK],
                                           const int32_t (&s2)[PRIO_CHUNK], const float (&bxe)[PRIO_CHUNK],
                                           double b, float bf, const PrioCoef &cf, const StepsDev &steps) {
  const int32_t cap = cf.cap;
  Tab tk = t0;
  auto step = [&]() {
    if constexpr (sizeof(Tab) == sizeof(uint32_t)) tk.base += (uint32_t)rowb;
    else tk.p += rowb;  // bytes
  };
  if (STEPS) {
    for (int k = 0; k < S; ++k, step()) {
      const int4 lk = s_lk[k];
      const int32_t nw = s_wk[k].x;
      float *ok = out0 + (int64_t)k * N;
#pragma unroll 1
      for (int m = 0; m < PRIO_CHUNK; ++m) {
        float lp = -INFINITY;
        for (int st = 0; st < steps.n; ++st) {
          const int64_t sgs = sg[m] + steps.off[st];
          const float bx = sgs > cap ? (float)(b * (double)(sgs - cap)) : 0.f;
          lp = logaddexpf_(lp, steps.logdc[st] + prio_elem<TIER>(tk, lk, nw, prio_s2(sgs, cap), bf, cf, bx));
        }
        if (m < nv) ok[(mode & 4u) ? 128 * (m >> 2) + (m & 3) : 32 * m] = lp;
      }
    }
    return;
  }
  if (mode == 6u) {  // the common case: full, vector, no slack above the cap; two sizes per iteration
    int k = 0;
    for (; k + 1 < S; k += 2) {
      const int4 lk0 = s_lk[k], lk1 = s_lk[k + 1];
      const int32_t nw0 = s_wk[k].x, nw1 = s_wk[k + 1].x;
      float *ok = out0 + (int64_t)k * N;
      prio_size<TIER, false, false, true>(tk, lk0, nw0, ok, nv, s2, bxe, bf, cf);
      step();
      prio_size<TIER, false, false, true>(tk, lk1, nw1, ok + N, nv, s2, bxe, bf, cf);
      step();
    }
    if (k < S) prio_size<TIER, false, false, true>(tk, s_lk[k], s_wk[k].x, out0 + (int64_t)k * N, nv, s2, bxe, bf, cf);
    return;
  }
  for (int k = 0; k < S; ++k, step()) {
    const int4 lk = s_lk[k];
    const int32_t nw = s_wk[k].x;
    float *ok = out0 + (int64_t)k * N;
    switch (mode) {
      case 7u: prio_size<TIER, false, true, true>(tk, lk, nw, ok, nv, s2, bxe, bf, cf); break;
      case 2u: prio_size<TIER, false, false, false>(tk, lk, nw, ok, nv, s2, bxe, bf, cf); break;
      case 3u: prio_size<TIER, false, true, false>(tk, lk, nw, ok, nv, s2, bxe, bf, cf); break;
      case 0u: prio_size<TIER, true, false, false>(tk, lk, nw, ok, nv, s2, bxe, bf, cf); break;
      default: prio_size<TIER, true, true, false>(tk, lk, nw, ok, nv, s2, bxe, bf, cf); break;
    }
  }
}

// Re-based table in global memory (sizes whose table exceeds the shared-memory
// budget): one thread per entry, the same values as the shared-memory staging.
template <int TIER>
__global__ void priority_rebase_kernel(const double *__restrict__ table, const double *__restrict__ logEL, int32_t S,
                                       int32_t B, double b, const __grid_constant__ ProfileDev prof,
                                       void *__restrict__ gtab) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)S * (B + 2)) return;
  const int k = (int)(e / (B + 2));
  static_cast<PrioEntry<TIER> *>(gtab)[e] = prio_entry<TIER>(table, logEL, prof, B, b, k, (int)(e - (int64_t)k * (B + 2)));
}

// Compare-exchange for a descending sort of (key, -index) pairs: after it,
// (ka, ia) is the better of the two (higher key; equal key -> lower index).
__device__ __forceinline__ void cx(uint32_t &ka, int &ia, uint32_t &kb, int &ib) {
  const bool sw = kb > ka || (kb == ka && ib < ia);
  const uint32_t tk = sw ? kb : ka;
  const int ti = sw ? ib : ia;
  kb = sw ? ka : kb;
  ib = sw ? ia : ib;
  ka = tk;
  ia = ti;
}

// PopBatch: per queue, the (up to) bs members with the highest
// log-priority for batch size bs, ties -> earlier member; -inf (no bin of L_bs
// fits before the deadline) and NaN are never selected.  Writes member indices
// (relative to the queue, highest priority first) to sel[q][0..bs), -1 after
// the last.  Warp per queue, member r = 32 s + lane in lane `lane`, slot s
// (n <= 256), keys order-preserving (0 = not selectable).
//
// Fast path (exact, warp-uniform test): let each lane's head be its best member
// (first of its maximal keys) and k2 its best other key.  If every k2 is below
// every selectable head, the selectable members in order are the selectable
// heads, then (if any) selectable non-heads; so when either no non-head is
// selectable or at least bs heads are, the answer is the best bs heads: one
// bitonic sort of (key desc, index asc) across the lanes, rank r ends in lane
// r, and lane r writes its member when r < bs and it is selectable.  A queue
// whose selectable top forms a contiguous run of at most 32 members (e.g. a
// unimodal priority over the deadline-sorted queue, or the few members with
// enough slack for a large batch) always takes it.
// General path: each lane sorts its 8 (19-comparator network), keeps its head in
// registers and the rest in shared memory; every round the lane holding the
// best head (REDUX max over keys, then min over member indices among equal
// keys) pops it and loads its next; round r's winner is kept by lane r.
// Bitonic sort of one packed (key << 32 | ~member) per lane across each group
// of W lanes (W = 32: the warp), descending: rank r ends in lane r.  Packed keys are distinct (distinct
// members), so one 64-bit compare orders (key desc, member asc).
template <int W = 32>
__device__ __forceinline__ uint64_t pop_bitonic32(uint64_t me, int lane) {
#pragma unroll
  for (int kk = 2; kk <= W; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      const uint64_t p = __shfl_xor_sync(FULL, me, j);
      // in a descending block the lower lane of a pair keeps the better one:
      // take the partner's iff (p > me) == (bit j of lane == bit kk of lane)
      const bool take = (p > me) ^ ((lane & j) != 0) ^ ((lane & kk) != 0);
      me = take ? p : me;
    }
  }
  return me;
}

// fkey of -inf: every selectable (finite or +inf) key is above it; lanes past
// the queue end hold 0.
constexpr uint32_t POP_KNEG = 0x007fffffu;

// order-preserving key of a log-priority: NaN -> fkey(-inf) (never selected),
// -0 + 0 = +0 (-0 ties +0)
__device__ __forceinline__ uint32_t pop_fkey(float x) {
  const uint32_t u = __float_as_uint(fmaxf(x + 0.0f, -INFINITY));
  return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}

// One queue of PopBatch: v[s] = log-priority of member 32 s + lane (any value
// past the queue end, masked by n), bs in 1..S; lst: this warp's shared lists.
__device__ __forceinline__ void pop_one(const float (&v)[8], int n, int bs, int lane, uint2 (*lst)[32],
                                        int32_t *__restrict__ out) {
  // lane head (first maximal slot) and the best other value, on the raw
  // floats: a NaN never wins a strict compare and fmaxf drops it; slot 0 is
  // sanitised (NaN -> -inf), -0 == +0 compares equal (the first one is the
  // head), slots past the queue end are -inf.  Only the head and the best other
  // value are turned into keys (the general path below builds all 8).
  const bool full = n >= 256;  // warp-uniform
  float vh, v2 = -INFINITY;
  int sh = 0;
  auto scan = [&](const float(&w)[8]) {
    vh = fmaxf(w[0], -INFINITY);
#pragma unroll
    for (int s = 1; s < 8; ++s) {
      const bool gt = w[s] > vh;
      v2 = gt ? vh : fmaxf(v2, w[s]);
      sh = gt ? s : sh;
      vh = gt ? w[s] : vh;
    }
  };
  if (full) {
    scan(v);
  } else {
    float w[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) w[s] = 32 * s + lane < n ? v[s] : -INFINITY;
    scan(w);
  }
  const uint32_t kh = pop_fkey(vh), k2 = pop_fkey(v2);
  // worst selectable head (all-ones if none) and best non-head
  const uint32_t hsel = __reduce_min_sync(FULL, kh > POP_KNEG ? kh : 0xffffffffu);
  const uint32_t mx2 = __reduce_max_sync(FULL, k2);
  if (mx2 < hsel && (mx2 <= POP_KNEG || __popc(__ballot_sync(FULL, kh > POP_KNEG)) >= bs)) {
    uint64_t me = ((uint64_t)kh << 32) | (uint32_t)~(32 * sh + lane);
    // only the m selectable heads need ordering: with m <= 16 (m <= 8) they are
    // compacted into lanes 0..m-1 through shared memory (the rest hold key 0)
    // and a 16- (8-) lane network sorts them
    const unsigned selb = __ballot_sync(FULL, kh > POP_KNEG);
    const int m = __popc(selb);
    if (m <= 16) {
      uint2 *cmp = lst[0];
      cmp[lane] = make_uint2(0u, 0u);
      __syncwarp();
      if (kh > POP_KNEG) cmp[__popc(selb & ((1u << lane) - 1u))] = make_uint2((uint32_t)me, (uint32_t)(me >> 32));
      __syncwarp();
      const uint2 c = cmp[lane];
      me = ((uint64_t)c.y << 32) | c.x;
      me = m <= 8 ? pop_bitonic32<8>(me, lane) : pop_bitonic32<16>(me, lane);
    } else {
      me = pop_bitonic32<32>(me, lane);
    }
    out[lane] = (lane < bs && (uint32_t)(me >> 32) > POP_KNEG) ? (int)~(uint32_t)me : -1;
    return;
  }
  uint32_t k[8];
  int id[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    k[s] = (full || 32 * s + lane < n) ? pop_fkey(v[s]) : 0u;
    id[s] = 32 * s + lane;
  }
  // Batcher odd-even merge sort network for 8 (19 comparators), descending.
  cx(k[0], id[0], k[1], id[1]); cx(k[2], id[2], k[3], id[3]); cx(k[4], id[4], k[5], id[5]); cx(k[6], id[6], k[7], id[7]);
  cx(k[0], id[0], k[2], id[2]); cx(k[1], id[1], k[3], id[3]); cx(k[4], id[4], k[6], id[6]); cx(k[5], id[5], k[7], id[7]);
  cx(k[1], id[1], k[2], id[2]); cx(k[5], id[5], k[6], id[6]);
  cx(k[0], id[0], k[4], id[4]); cx(k[1], id[1], k[5], id[5]); cx(k[2], id[2], k[6], id[6]); cx(k[3], id[3], k[7], id[7]);
  cx(k[2], id[2], k[4], id[4]); cx(k[3], id[3], k[5], id[5]);
  cx(k[1], id[1], k[2], id[2]); cx(k[3], id[3], k[4], id[4]); cx(k[5], id[5], k[6], id[6]);
  #pragma unroll
  for (int s = 1; s < 8; ++s) lst[s][lane] = make_uint2(k[s], (uint32_t)id[s]);
  lst[8][lane] = make_uint2(0u, 0x7fffffffu);
  __syncwarp();
  uint32_t hk = k[0];
  int hid = id[0], pos = 0, mine = -1;
  for (int round = 0; round < bs; ++round) {
    const uint32_t mx = __reduce_max_sync(FULL, hk);
    if (mx <= POP_KNEG) break;  // no selectable member left (warp-uniform)
    const int win = (int)__reduce_min_sync(FULL, hk == mx ? (uint32_t)hid : 0x7fffffffu);
    if (lane == round) mine = win;
    if (hid == win) {  // pop the head (member indices are distinct)
      pos = pos < 8 ? pos + 1 : 8;
      const uint2 nx = lst[pos][lane];
      hk = nx.x;
      hid = (int)nx.y;
    }
  }
  out[lane] = mine;
}

// QPW queues per warp: every queue's offsets and all QPW x 8 member loads are
// issued before the first queue is processed, so the loads of the later queues
// are in flight while the earlier ones sort (ORLOJ_POP_QPW; 1 = one queue per warp).
#ifndef ORLOJ_POP_QPW
#define ORLOJ_POP_QPW 2
#endif
constexpr int POP_QPW = ORLOJ_POP_QPW;
static __global__ void __launch_bounds__(256) pop_batch_kernel(const float *__restrict__ logp, int32_t S, int64_t Q,
                                                               const int64_t *__restrict__ offsets,
                                                               const int32_t *__restrict__ bs_q,
                                                               int32_t *__restrict__ sel) {
  __shared__ uint2 s_list[8][9][32];  // per warp: sorted (key, id) positions 1..7 of each lane, 8 = sentinel
  const int lane = threadIdx.x & 31;
  const int64_t q0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * POP_QPW;
  if (q0 >= Q) return;
  const int64_t base0 = offsets[0], N = offsets[Q] - base0;
  int64_t b0[POP_QPW];
  int n[POP_QPW], bs[POP_QPW];
#pragma unroll
  for (int j = 0; j < POP_QPW; ++j) {
    const int64_t q = q0 + j;
    b0[j] = 0;
    n[j] = 0;
    bs[j] = 0;
    if (q < Q) {
      b0[j] = offsets[q] - base0;
      n[j] = (int)(offsets[q + 1] - offsets[q]);
      const int b = bs_q[q];
      bs[j] = (b >= 1 && b <= S) ? b : 0;
    }
  }
  // all loads first and unconditional within a queue, so they are in flight
  // together (a short queue's lanes past the end re-read its last member,
  // masked later)
  float v[POP_QPW][8];
#pragma unroll
  for (int j = 0; j < POP_QPW; ++j) {
    if (n[j] <= 0 || !bs[j]) continue;  // nothing selectable (warp-uniform)
    const float *row = logp + (int64_t)(bs[j] - 1) * N + b0[j];
    if (n[j] >= 256) {
#pragma unroll
      for (int s = 0; s < 8; ++s) v[j][s] = __ldg(row + 32 * s + lane);
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) v[j][s] = __ldg(row + min(32 * s + lane, n[j] - 1));
    }
  }
  uint2(*lst)[32] = s_list[threadIdx.x >> 5];
#pragma unroll
  for (int j = 0; j < POP_QPW; ++j) {
    if (q0 + j >= Q) break;
    int32_t *out = sel + (q0 + j) * 32;
    if (n[j] <= 0 || !bs[j]) {
      out[lane] = -1;
      continue;
    }
    if (j > 0) __syncwarp();  // the previous queue's list reads are done
    pop_one(v[j], n[j], bs[j], lane, lst, out);
  }
}

}  // namespace orloj
