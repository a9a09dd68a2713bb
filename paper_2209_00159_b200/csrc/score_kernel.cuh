// score_kernel.cuh — K1/K2: distribution-aware scoring of every deadline-prefix
// candidate batch, one warp per queue.
//
// Per queue q at time t (member r = 0..K-1 in deadline order, K = min(n_q, kmax)):
//   LG_k[i]  = LG_{k-1}[i] + log2 F_{d_k}(tau_i)          (Eq. 6/8 product, log2 domain)
//   i*(r,k)  = clamp(floor((D_r - t - a_k) / w_k), 0, B)  (Eq. 3-4, Eq. 9 CDF form)
//   P_r(k)   = 2^{LG_k[i*]}  (0 when i* = 0)               (step SLO cost)
//   E_k      = sum_{r<k} P_r(k);  k* = smallest argmax
//
// Layout: lane `l` owns bins [l*BPL, l*BPL + BPL) of the running LG in
// registers (one 32-byte load per row at B = 256); member r lives in lane r % 32,
// slot r / 32.  Per k the lane adds row d_k (prefetched PF rows ahead into a
// register ring — up to PF*BPL*4 bytes in flight per lane), stages LG_k in a
// double-buffered shared-memory row (index -1 holds -inf for i* = 0), then
// every member r < k gathers LG_k[i*-1] and applies ex2.  The 32 per-lane
// partial sums of a chunk of 32 consecutive k are reduced with the
// transposing butterfly (31 shuffles per 32 k), leaving E_k in lane (k-1) % 32.
#pragma once
#include "common.cuh"

namespace orloj {

struct ScoreParams {
  const float *log2F;
  int32_t B;
  int32_t kmax;
  int64_t Q;
  const int64_t *offsets;
  const int64_t *deadline;
  const int32_t *dist;
  const int64_t *now;
  float *E;          // [Q][kmax] or null
  float *P;          // packed [Q][kmax(kmax+1)/2] or null
  float *EL;         // [Q][kmax] or null
  int32_t *best_k;   // [Q] or null (pick)
  float *best_E;     // [Q] or null
  ProfileDev prof;
};

constexpr int SCORE_WARPS = 8;

template <int BPL, int SLOTS, bool PICK, bool STREAM>
__global__ void __launch_bounds__(SCORE_WARPS * 32)
score_kernel(const __grid_constant__ ScoreParams p) {
  constexpr int BPAD = 32 * BPL;
  constexpr int STG = BPAD + 4;             // 4-float head keeps rows 16-B aligned; [3] = -inf
  constexpr int PF = BPL == 8 ? 4 : 8;      // rows in flight per warp

  __shared__ __align__(16) float s_stage[SCORE_WARPS][2][STG];

  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * SCORE_WARPS + wid;
  if (q >= p.Q) return;

  float *stg[2] = {&s_stage[wid][0][4], &s_stage[wid][1][4]};
  if (lane == 0) {
    stg[0][-1] = -INFINITY;
    stg[1][-1] = -INFINITY;
  }

  const int B = p.B;
  const int kmax = p.kmax;
  const int64_t off = p.offsets[q];
  const int64_t n = p.offsets[q + 1] - off;
  const int K = (int)(n < kmax ? n : kmax);
  const int64_t now = p.now[q];
  const int64_t *dl = p.deadline + off;
  const int32_t *ids = p.dist + off;

  // sigma of the members this lane owns
  int32_t sig[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int r = 32 * s + lane;
    sig[s] = r < K ? clamp_sigma(dl[r] - now) : -1;
  }

  // bins this lane owns: [lane*BPL, lane*BPL + BPL) (B % 8 == 4: the last lane's half)
  const bool vok = lane * BPL < B;
  const bool vhalf = lane * BPL + BPL > B;
  const float *myrow = p.log2F + lane * BPL;

  float lg[BPL];
#pragma unroll
  for (int b = 0; b < BPL; ++b) lg[b] = 0.f;

  Vec<BPL> ring[PF];
  int id_cur = lane < K ? ids[lane] : 0;
  int id_nxt = 32 + lane < K ? ids[32 + lane] : 0;
#pragma unroll
  for (int j = 0; j < PF; ++j) {
    const int d = __shfl_sync(FULL, id_cur, j);
    ring[j] = (j < K && vok) ? ldrow<BPL, STREAM>(myrow + (int64_t)d * B, vhalf) : vzero<BPL>();
  }

  const int nchunks = (K + 31) >> 5;
  const int nchunks_out = (kmax + 31) >> 5;
  const int64_t tri = (int64_t)kmax * (kmax + 1) / 2;
  float bestE = -1.f;
  int bestk = 0;

  for (int c = 0; c < nchunks; ++c) {
    float pend[5];
    float pendL[5];
    float Ek = 0.f, Sk = 0.f;
#pragma unroll
    for (int kk = 0; kk < 32; ++kk) {
      const int k = 32 * c + kk + 1;
      float part = 0.f, partL = 0.f;
      if (k <= K) {
        // LG_k = LG_{k-1} + row d_k
        const Vec<BPL> cur = ring[kk % PF];
#pragma unroll
        for (int e = 0; e < BPL; ++e) lg[e] += cur.x[e];
        // refill the ring slot with row k + PF
        {
          const int jn = kk + PF;  // index within chunk c (may spill into c+1)
          const int d = jn < 32 ? __shfl_sync(FULL, id_cur, jn & 31) : __shfl_sync(FULL, id_nxt, jn & 31);
          const bool ok = k + PF <= K;
          if (ok && vok) ring[kk % PF] = ldrow<BPL, STREAM>(myrow + (int64_t)d * B, vhalf);
        }
        // stage LG_k
        float *sg = stg[kk & 1];
        st_stage<BPL>(sg + lane * BPL, lg);
        __syncwarp();
        const int32_t a = p.prof.a[k - 1], wB = p.prof.wB[k - 1];
        const uint32_t mg = p.prof.mag[k - 1], sh = p.prof.sh[k - 1];
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
          if (s < c || (s == c && lane <= kk)) {
            const int i = lookup_bin(sig[s], a, wB, mg, sh);
            const float pr = ex2_approx(sg[i - 1]);
            part += pr;
            if (!PICK && p.P) p.P[q * tri + (int64_t)k * (k - 1) / 2 + 32 * s + lane] = pr;
          }
        }
        if (!PICK && p.EL) {
          // E[max bin] = B - sum_{i<B} G_k(tau_i)  (summation by parts of Eq. 5)
#pragma unroll
          for (int e = 0; e < BPL; ++e) {
            const int bin = lane * BPL + e;  // 0-based: tau_{bin+1}
            if (bin < B - 1) partL += ex2_approx(lg[e]);
          }
        }
      }
      Ek = bfly_push(pend, part, kk, lane);
      if (!PICK && p.EL) Sk = bfly_push(pendL, partL, kk, lane);
    }
    // lane l now holds E_k for k = 32c + l + 1
    const int k = 32 * c + lane + 1;
    const bool valid = k <= K;
    const float E = valid ? Ek : 0.f;
    if (!PICK) {
      if (k <= kmax) {
        if (p.E) p.E[q * kmax + k - 1] = E;
        if (p.EL) {
          const double el = valid ? (double)p.prof.a[k - 1] + (double)p.prof.w[k - 1] * ((double)B - (double)Sk) : 0.0;
          p.EL[q * kmax + k - 1] = (float)el;
        }
      }
    } else if (valid && E > bestE) {
      bestE = E;
      bestk = k;
    }
    // next chunk's ids
    id_cur = id_nxt;
    id_nxt = 32 * (c + 2) + lane < K ? ids[32 * (c + 2) + lane] : 0;
  }

  if (!PICK) {
    for (int c = nchunks; c < nchunks_out; ++c) {
      const int k = 32 * c + lane + 1;
      if (k <= kmax) {
        if (p.E) p.E[q * kmax + k - 1] = 0.f;
        if (p.EL) p.EL[q * kmax + k - 1] = 0.f;
      }
    }
  } else {
    // warp argmax, ties -> smallest k.  E >= 0, so float bits order like values.
    const uint32_t bits = bestk ? __float_as_uint(bestE) : 0u;
    const uint32_t mx = __reduce_max_sync(FULL, bits);
    const uint32_t kb = __reduce_min_sync(FULL, (bestk && bits == mx) ? (uint32_t)bestk : 0x7fffffffu);
    if (lane == 0) {
      const bool empty = K == 0;
      p.best_k[q] = empty ? 0 : (int32_t)kb;
      p.best_E[q] = empty ? 0.f : __uint_as_float(mx);
    }
  }
}

}  // namespace orloj
