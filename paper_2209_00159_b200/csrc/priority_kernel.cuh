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

// Warp per queue (grid-stride over queues: a block stages the per-size
// constants once and reuses them for many queues), lanes over members, chunks
// of 8 members per lane with the size loop outside the member loop (the
// per-size constants are loaded once per 8 members).  Per block, shared memory
// holds for every size k: the lookup constants {2a, 2wB, mag, sh} (one 16-B
// load), w, and -- when SMEM_TABLE -- the table re-based on log E[L]:
//   sC[k][i] = C[i] - log E[L]   (fp64: it meets b sigma, both can be large)
//   sH[k][i] = H[i] - log E[L]   (fp32)
// Per element (member r, size k), with A = sC[i*] - b sigma (fp64 -> fp32):
//   no partial bin:  log p = A
//   partial bin, x = sigma - l1 in (0, w):  g = 1 - e^{-b x},
//      log p = log(e^A + e^{sH[i*+1]} g)  (prio_partial)
// Output [S][N] (size-major: each store of a warp is one contiguous 128-B
// line, and PopBatch reads one size row coalesced).
struct PrioSmem {
  static __host__ __device__ size_t table_bytes(int S, int B) { return (size_t)S * (B + 1) * (8 + 4); }
  static __host__ __device__ size_t bytes(int S, int B, bool smem_table) {
    return (size_t)S * (16 + 4) + (smem_table ? table_bytes(S, B) : 0);
  }
};

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The partial bin of Eq. 2 in the log domain: log(e^lp + e^Hn g), g = 1 - e^{-t},
// t = b x > 0.  g: the Taylor series to t^8 below t = 1/2 (truncation < 2^-26
// relative, no cancellation), else 1 - 2^{-t log2 e} (g > 0.39 there).  With
// d = -|lp - Hn| one term of the sum is exactly 1:
//   lp >= Hn:  lp + log(1 + e^d g),   else  Hn + log(e^d + g),
// two MUFU (ex2, lg2) per element.
__device__ __forceinline__ float prio_partial(float lp, float Hn, float t) {
  float c = -1.f / 40320.f;
  c = fmaf(c, t, 1.f / 5040.f);
  c = fmaf(c, t, -1.f / 720.f);
  c = fmaf(c, t, 1.f / 120.f);
  c = fmaf(c, t, -1.f / 24.f);
  c = fmaf(c, t, 1.f / 6.f);
  c = fmaf(c, t, -0.5f);
  c = fmaf(c, t, 1.f);
  const float g = t < 0.5f ? c * t : 1.f - ex2_approx(-t * 1.4426950408889634f);
  const bool hi = lp >= Hn;
  const float e = ex2_approx(-fabsf(lp - Hn) * 1.4426950408889634f);
  const float y = hi ? fmaf(e, g, 1.f) : e + g;
  return fmaf(0.6931471805599453f, lg2_approx(y), hi ? lp : Hn);
}

// One element of the score kernel with the table read from global memory
// (tab_k = table + (k-1) 2 (B+1)); the same arithmetic, value for value, as the
// shared-memory path (which stages tab - lEL in fp64 and (float)(tab - lEL)).
__device__ __forceinline__ float prio_elem_global(const double *__restrict__ tab_k, double lEL, int B, int4 lk,
                                                  int32_t w, int32_t s2, double bsig, float bf) {
  const int i = lookup_bin(s2, lk.x, lk.y, (uint32_t)lk.z, (uint32_t)lk.w);
  const int32_t x = ((s2 - lk.x) >> 1) - w * i;
  const double Ci = tab_k[i] - lEL;
  const float Hn = (i < B && x > 0) ? (float)(tab_k[B + 1 + i + 1] - lEL) : -INFINITY;
  float lp = (float)(Ci + bsig);
  if (Hn > -INFINITY) lp = prio_partial(lp, Hn, bf * (float)x);
  return lp;
}

constexpr int PRIO_CHUNK = 8;  // members per lane per pass
constexpr int PRIO_MAX_STEPS = 8;

// Piecewise-step cost: deadlines D_r + off[s] with cost
// increments dc[s] = c_s - c_{s-1} > 0; p = sum_s dc[s] p_single(sigma + off[s]).
struct StepsDev {
  int32_t n;
  int64_t off[PRIO_MAX_STEPS];
  float logdc[PRIO_MAX_STEPS];   // log dc[s]
  double boff[PRIO_MAX_STEPS];   // b off[s]
};

__device__ __forceinline__ float logaddexpf_(float a, float b) {
  const float M = fmaxf(a, b);
  return M == -INFINITY ? M : M + log1pf(__expf(fminf(a, b) - M));
}

template <bool SMEM_TABLE, bool STEPS>
__global__ void __launch_bounds__(256) priority_scores_kernel(
    const double *__restrict__ table, const double *__restrict__ logEL, int32_t S, int32_t B, double b,
    const __grid_constant__ ProfileDev prof, const __grid_constant__ StepsDev steps, int64_t Q,
    const int64_t *__restrict__ offsets, const int64_t *__restrict__ deadline, const int64_t *__restrict__ now,
    float *__restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int4 *s_lk = reinterpret_cast<int4 *>(smem_raw);                                          // [S]
  double *s_C = reinterpret_cast<double *>(s_lk + S);                                       // [S][B+1]
  float *s_H = reinterpret_cast<float *>(s_C + (SMEM_TABLE ? (size_t)S * (B + 1) : 0));    // [S][B+1]
  int32_t *s_w = reinterpret_cast<int32_t *>(s_H + (SMEM_TABLE ? (size_t)S * (B + 1) : 0));  // [S]
  for (int k = threadIdx.x; k < S; k += blockDim.x) {
    s_lk[k] = make_int4(prof.a2[k], prof.wB2[k], (int)prof.mag[k], (int)prof.sh[k]);
    s_w[k] = prof.w[k];
  }
  if (SMEM_TABLE)
    for (int e = threadIdx.x; e < S * (B + 1); e += blockDim.x) {
      const int k = e / (B + 1), i = e - k * (B + 1);
      const double lEL = logEL[k];
      s_C[e] = table[(size_t)k * 2 * (B + 1) + i] - lEL;
      s_H[e] = (float)(table[(size_t)k * 2 * (B + 1) + B + 1 + i] - lEL);
    }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float bf = (float)b;
  const int64_t base0 = offsets[0], N = offsets[Q] - base0;
  const int64_t wpb = blockDim.x >> 5;

  // log p_single for size k at slack sigma (s2 = sigma2(sigma), bsig = -b sigma)
  auto single = [&](int k, const int4 &lk, int32_t w, double lEL, int32_t s2, double bsig) -> float {
    const int i = lookup_bin(s2, lk.x, lk.y, (uint32_t)lk.z, (uint32_t)lk.w);
    // x = sigma - l1 of bin i+1 (exact: below the horizon 2 sigma - 2a fits int32;
    // sigma < 0 gives x = -a <= 0)
    const int32_t x = ((s2 - lk.x) >> 1) - w * i;
    const bool part = i < B && x > 0;
    double Ci;
    float Hn = -INFINITY;
    if (SMEM_TABLE) {
      Ci = s_C[k * (B + 1) + i];
      if (part) Hn = s_H[k * (B + 1) + i + 1];
    } else {
      Ci = table[(size_t)k * 2 * (B + 1) + i] - lEL;
      if (part) Hn = (float)(table[(size_t)k * 2 * (B + 1) + B + 1 + i + 1] - lEL);
    }
    float lp = (float)(Ci + bsig);
    if (Hn > -INFINITY) lp = prio_partial(lp, Hn, bf * (float)x);  // 0 < b x < b w
    return lp;
  };

  for (int64_t q = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); q < Q; q += (int64_t)gridDim.x * wpb) {
    const int64_t b0 = offsets[q] - base0, e0 = offsets[q + 1] - base0;
    const int64_t t = now[q];
    for (int64_t c0 = b0; c0 < e0; c0 += 32 * PRIO_CHUNK) {
      // members of this lane in the chunk: c0 + lane + 32 m < e0  <=>  m < nv (32-bit compares below)
      const int64_t rem = e0 - c0 - lane;
      const int nv = rem <= 0 ? 0 : rem >= 32 * PRIO_CHUNK ? PRIO_CHUNK : (int)((rem + 31) >> 5);
      double bsig[PRIO_CHUNK];  // -b sigma
      int64_t sg[PRIO_CHUNK];   // sigma (STEPS)
      int32_t s2[PRIO_CHUNK];
#pragma unroll
      for (int m = 0; m < PRIO_CHUNK; ++m) {
        const int64_t j = c0 + lane + 32 * m;
        const int64_t sigma = j < e0 ? deadline[j] - t : 0;
        sg[m] = sigma;
        bsig[m] = -b * (double)sigma;
        s2[m] = sigma2(sigma);
      }
      for (int k = 0; k < S; ++k) {
        const int4 lk = s_lk[k];
        const int32_t w = s_w[k];
        float *ok = out + (int64_t)k * N + c0 + lane;  // member m at ok[32 m]
        const double lEL = SMEM_TABLE ? 0.0 : logEL[k];
#pragma unroll
        for (int m = 0; m < PRIO_CHUNK; ++m) {
          if (m >= nv) break;
          float lp;
          if (STEPS) {
            lp = -INFINITY;
            for (int st = 0; st < steps.n; ++st)
              lp = logaddexpf_(lp, steps.logdc[st] + single(k, lk, w, lEL, sigma2(sg[m] + steps.off[st]),
                                                           bsig[m] - steps.boff[st]));
          } else {
            lp = single(k, lk, w, lEL, s2[m], bsig[m]);
          }
          ok[32 * m] = lp;
        }
      }
    }
  }
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
// the last.  Warp per queue, members strided over lanes, 8 per lane (n <= 256):
// each lane sorts its 8 once (19-comparator network), then every round the
// lane holding the best head (REDUX max over keys, then min over member
// indices among equal keys) pops it.  Round r's winner is kept by lane r and
// the 32 results leave in one coalesced store.
static __global__ void __launch_bounds__(256) pop_batch_kernel(const float *__restrict__ logp, int32_t S, int64_t Q,
                                                        const int64_t *__restrict__ offsets,
                                                        const int32_t *__restrict__ bs_q, int32_t *__restrict__ sel) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= Q) return;
  const int64_t base0 = offsets[0];
  const int64_t b0 = offsets[q] - base0, N = offsets[Q] - base0;
  const int n = (int)(offsets[q + 1] - offsets[q]);
  int bs = bs_q[q];
  bs = (bs >= 1 && bs <= S) ? bs : 0;
  uint32_t k[8];
  int id[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int r = 32 * s + lane;
    id[s] = r;
    k[s] = 0u;
    if (r < n && bs) {
      const float v = logp[(int64_t)(bs - 1) * N + b0 + r];
      k[s] = (v == -INFINITY || v != v) ? 0u : fkey(v == 0.0f ? 0.0f : v);  // -0 ties +0
    }
  }
  // Batcher odd-even merge sort network for 8 (19 comparators), descending.
  cx(k[0], id[0], k[1], id[1]); cx(k[2], id[2], k[3], id[3]); cx(k[4], id[4], k[5], id[5]); cx(k[6], id[6], k[7], id[7]);
  cx(k[0], id[0], k[2], id[2]); cx(k[1], id[1], k[3], id[3]); cx(k[4], id[4], k[6], id[6]); cx(k[5], id[5], k[7], id[7]);
  cx(k[1], id[1], k[2], id[2]); cx(k[5], id[5], k[6], id[6]);
  cx(k[0], id[0], k[4], id[4]); cx(k[1], id[1], k[5], id[5]); cx(k[2], id[2], k[6], id[6]); cx(k[3], id[3], k[7], id[7]);
  cx(k[2], id[2], k[4], id[4]); cx(k[3], id[3], k[5], id[5]);
  cx(k[1], id[1], k[2], id[2]); cx(k[3], id[3], k[4], id[4]); cx(k[5], id[5], k[6], id[6]);
  int mine = -1;
  for (int round = 0; round < bs; ++round) {
    const uint32_t mx = __reduce_max_sync(FULL, k[0]);
    if (mx == 0u) break;  // no selectable member left (warp-uniform)
    const int win = (int)__reduce_min_sync(FULL, k[0] == mx ? (uint32_t)id[0] : 0x7fffffffu);
    if (lane == round) mine = win;
    if (id[0] == win && k[0] == mx) {  // pop the head
#pragma unroll
      for (int s = 0; s < 7; ++s) {
        k[s] = k[s + 1];
        id[s] = id[s + 1];
      }
      k[7] = 0u;
    }
  }
  sel[q * 32 + lane] = mine;
}

}  // namespace orloj
