// score_kernel.cuh — K1/K2: distribution-aware scoring of every deadline-prefix
// candidate batch, one warp per queue.
//
// Per queue q at time t (member r = 0..K-1 in deadline order, K = min(n_q, kmax)):
//   LG_k[i]  = LG_{k-1}[i] + log2 F_{d_k}(tau_i)          (Eq. 6/8 product, log2 domain)
//   i*(r,k)  = clamp(floor((D_r - t - a_k) / w_k), 0, B)  (Eq. 3-4, Eq. 9 CDF form)
//   P_r(k)   = 2^{LG_k[i*]}  (0 when i* = 0)               (step SLO cost)
//   E_k      = sum_{r<k} P_r(k);  k* = smallest argmax
//
// Row pipeline: every warp owns a ring of R shared-memory slots; one elected
// lane streams the queue's rows log2F[d_k] into it with bulk async copies (the
// TMA engine, cp.async.bulk + mbarrier complete_tx), R rows ahead — R KB in
// flight per warp without holding registers.  Each slot is also the staging
// row: lane l adds its bins of row k into its running LG (registers) and writes
// LG_k back over the same slot, so after one __syncwarp every member can gather
// LG_k[i*] from it.  The slot is refilled one iteration later.  A 16-byte head
// before every slot holds -inf for i* = 0.
//
// Layout: lane l owns BPL bins as NV vectors of V = min(BPL, 4) floats, vector v
// covering bins [(32 v + l) V, +V): conflict-free vector shared-memory accesses.
// Member r lives in lane r % 32, slot r / 32.  The 32 per-lane partial sums of a
// chunk of 32 consecutive k are reduced with the transposing butterfly (31
// shuffles per 32 k), leaving E_k in lane (k-1) % 32.  K is made warp-uniform
// (REDUX) so the member-slot switch compiles to uniform branches.
#pragma once
#include "common.cuh"

// Unroll of the k-group loop inside a 32-k chunk (8 groups of G = 4).  Fully
// unrolled (8) keeps every ring-slot index and butterfly level compile-time,
// but the C3 pick kernel is then 6,136 SASS instructions with a 3,275-
// instruction hot loop, and ncu showed no_instruction (instruction-fetch)
// stalls; unrolled by 2 it is ~2,000 instructions and the C3 pick went from
// 2.94 to 2.51 ms on one box (1 / 2 / 4 / 8: 2.71 / 2.51 / 2.61 / 2.94 ms).
#ifndef ORLOJ_SCORE_KG_UNROLL
#define ORLOJ_SCORE_KG_UNROLL 2
#endif
namespace orloj {
constexpr int SCORE_KG_UNROLL = ORLOJ_SCORE_KG_UNROLL;
}

namespace orloj {

struct ScoreParams {
  const float *log2F;
  int32_t D;
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

#ifndef ORLOJ_RING
#define ORLOJ_RING 8
#endif

template <int BPL>
struct ScoreShape {
  static constexpr int R = ORLOJ_RING;         // ring slots per warp (two groups of G rows)
  static constexpr int G = R / 2;              // rows per barrier group; divides 32
  static constexpr int SLOT = 32 * BPL + 4;    // floats per slot incl. the 16-B head
  __host__ __device__ static constexpr size_t smem_bytes() { return (size_t)SCORE_WARPS * (R * SLOT * 4 + 2 * 8); }
};

// SMEMS: the whole store (a few application histograms, D*B*4 <= 48 KiB) is
// staged in shared memory once per CTA and rows are read from there; the TMA
// ring is then unused and its slots only stage LG_k.
template <int BPL, int SLOTS, bool PICK, bool STREAM, bool SMEMS>
__global__ void __launch_bounds__(SCORE_WARPS * 32)
score_kernel(const __grid_constant__ ScoreParams p) {
  constexpr int V = BPL < 4 ? BPL : 4;      // floats per vector
  constexpr int NV = BPL / V;               // vectors per lane per row
  constexpr int R = ScoreShape<BPL>::R;
  constexpr int G = ScoreShape<BPL>::G;
  constexpr int SLOT = ScoreShape<BPL>::SLOT;

  extern __shared__ __align__(16) float s_dyn[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  float *ring = s_dyn + wid * (R * SLOT);                       // slot j: ring + j*SLOT, row at +4
  uint64_t *bars = reinterpret_cast<uint64_t *>(s_dyn + SCORE_WARPS * R * SLOT) + wid * 2;
  float *s_store = reinterpret_cast<float *>(s_dyn + SCORE_WARPS * R * SLOT + 2 * 2 * SCORE_WARPS);
  if constexpr (SMEMS) {
    const int DB = p.D * p.B;
    for (int e = threadIdx.x * 4; e < DB; e += blockDim.x * 4)
      *reinterpret_cast<float4 *>(s_store + e) = __ldg(reinterpret_cast<const float4 *>(p.log2F + e));
    __syncthreads();
  }

  const int64_t q = (int64_t)blockIdx.x * SCORE_WARPS + wid;
  if (q >= p.Q) return;

  const int B = p.B;
  const int kmax = p.kmax;
  const int64_t off = p.offsets[q] - p.offsets[0];   // offsets may start at any base (chunked calls)
  const int64_t n = p.offsets[q + 1] - p.offsets[q];
  const int K = warp_uniform((int)(n < kmax ? n : kmax));
  const int64_t now = p.now[q];
  const int64_t *dl = p.deadline + off;
  const int32_t *ids = p.dist + off;
  const uint32_t row_bytes = (uint32_t)B * 4u;
  const uint32_t ring_s = smem_addr(ring);
  const uint32_t bar_s = smem_addr(bars);
  const uint64_t pol = STREAM ? l2_evict_first_policy() : 0;

  int id_cur = lane < K ? ids[lane] : 0;
  int id_nxt = 32 + lane < K ? ids[32 + lane] : 0;
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < R; ++j) ring[j * SLOT + 3] = -INFINITY;
    if constexpr (!SMEMS) {
      mbar_init(bar_s, 1);
      mbar_init(bar_s + 8, 1);
      mbar_init_fence();
    }
  }
  __syncwarp();
  // prologue: rows 0 .. R-1 in two barrier groups
#pragma unroll
  for (int g = 0; g < (SMEMS ? 0 : 2); ++g) {
    const int nrows = min(max(K - g * G, 0), G);
    arm_barrier(lane == 0 && nrows > 0, bar_s + 8 * g, (uint32_t)nrows * row_bytes);
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int j = g * G + i;
      const int d = __shfl_sync(FULL, id_cur, j);
      bulk_row<STREAM>(lane == 0 && j < K, ring_s + (j * SLOT + 4) * 4, p.log2F + (int64_t)d * B, row_bytes,
                       bar_s + 8 * g, pol);
    }
  }

  // doubled slack of the members this lane owns; 0 (-> bin 0 -> P = 0) beyond K
  int32_t sig[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int r = 32 * s + lane;
    sig[s] = r < K ? sigma2(dl[r] - now) : 0;
  }

  bool vok[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) vok[v] = (32 * v + lane) * V < B;

  float lg[BPL];
#pragma unroll
  for (int b = 0; b < BPL; ++b) lg[b] = 0.f;

  const int nchunks = (K + 31) >> 5;
  const int nchunks_out = (kmax + 31) >> 5;
  const int64_t tri = (int64_t)kmax * (kmax + 1) / 2;
  float bestE = -1.f;
  int bestk = 0;

  for (int c = 0; c < nchunks; ++c) {
    int32_t sigp = 0;   // slack of this lane's member in slot c
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) sigp = s == c ? sig[s] : sigp;
    float pend[5];
    float pendL[5];
    float Ek = 0.f, Sk = 0.f;
#pragma unroll SCORE_KG_UNROLL
    for (int kg = 0; kg < 32; kg += G) {
      // one group of G consecutive k = k0 .. k0+G-1 (rows j0 .. j0+G-1, one barrier)
      const int k0 = 32 * c + kg + 1;
      const int j0 = k0 - 1;
      float part[G], partL[G];
#pragma unroll
      for (int i = 0; i < G; ++i) part[i] = partL[i] = 0.f;
      if (k0 <= K) {
        if constexpr (!SMEMS) mbar_wait(bar_s + 8 * ((kg / G) % 2), (uint32_t)(j0 / R) & 1u);
        // LG_k = LG_{k-1} + row d_k, written over row k's slot, for the G rows
#pragma unroll
        for (int i = 0; i < G; ++i) {
          const int dsm = SMEMS ? __shfl_sync(FULL, id_cur, kg + i) : 0;   // row id (SMEMS)
          if (k0 + i <= K) {
            float *sl = ring + ((kg + i) % R) * SLOT + 4;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              if (vok[v]) {
                float *pv = sl + (32 * v + lane) * V;
                const Vec<V> x = *reinterpret_cast<const Vec<V> *>(
                    SMEMS ? s_store + dsm * B + (32 * v + lane) * V : pv);
#pragma unroll
                for (int e = 0; e < V; ++e) lg[v * V + e] += x.x[e];
                st_vec<V>(pv, &lg[v * V]);
              }
            }
            if (!PICK && p.EL) {
              // E[max bin] = B - sum_{i<B} G_k(tau_i)  (summation by parts of Eq. 5)
#pragma unroll
              for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int e = 0; e < V; ++e) {
                  const int bin = (32 * v + lane) * V + e;  // 0-based: tau_{bin+1}
                  if (bin < B - 1) partL[i] += ex2_approx(lg[v * V + e]);
                }
            }
          }
        }
        __syncwarp();
        // the previous group (rows j0-G .. j0-1) is fully consumed: refill it
        // with rows j0+G .. j0+2G-1
        if (!SMEMS && j0 >= G) {
          const int pg = ((kg / G) + 1) % 2;
          const int nrows = min(max(K - (j0 + G), 0), G);
          arm_barrier(lane == 0 && nrows > 0, bar_s + 8 * pg, (uint32_t)nrows * row_bytes);
#pragma unroll
          for (int i = 0; i < G; ++i) {
            const int jn = kg + G + i;  // index of row j0+G+i within chunk c (may spill into c+1)
            const int d = jn < 32 ? __shfl_sync(FULL, id_cur, jn & 31) : __shfl_sync(FULL, id_nxt, jn & 31);
            const int ps = (kg + G + i) % R;
            bulk_row<STREAM>(lane == 0 && j0 + G + i < K, ring_s + (ps * SLOT + 4) * 4, p.log2F + (int64_t)d * B,
                             row_bytes, bar_s + 8 * pg, pol);
          }
        }
        int32_t a2[G], wB2[G];
        uint32_t mg[G], sh[G];
        uint32_t sgl[G];   // shared address of LG_{k0+i}(tau_0) = -inf; bin b at + 4b
#pragma unroll
        for (int i = 0; i < G; ++i) {
          a2[i] = p.prof.a2[k0 - 1 + i];
          wB2[i] = p.prof.wB2[k0 - 1 + i];
          mg[i] = p.prof.mag[k0 - 1 + i];
          sh[i] = p.prof.sh[k0 - 1 + i];
          sgl[i] = ring_s + (((kg + i) % R) * SLOT + 3) * 4;
        }
        // members of the full slots s < c (Duff's device on the warp-uniform c);
        // each case scores one member against the G k's of the group (G-way ILP)
        switch (c) {
#define ORLOJ_FULL_SLOT(S)                                                                     \
  case (S) + 1:                                                                                \
    if constexpr ((S) < SLOTS) {                                                               \
      _Pragma("unroll") for (int i = 0; i < G; ++i) {                                          \
        const float pr = ex2_approx(lds_f32(sgl[i] + 4 * lookup_bin(sig[(S)], a2[i], wB2[i], mg[i], sh[i]))); \
        part[i] += pr;                                                                         \
        if (!PICK && p.P && k0 + i <= K)                                                       \
          p.P[q * tri + (int64_t)(k0 + i) * (k0 + i - 1) / 2 + 32 * (S) + lane] = pr;          \
      }                                                                                        \
    }                                                                                          \
    [[fallthrough]];
          ORLOJ_FULL_SLOT(6)
          ORLOJ_FULL_SLOT(5)
          ORLOJ_FULL_SLOT(4)
          ORLOJ_FULL_SLOT(3)
          ORLOJ_FULL_SLOT(2)
          ORLOJ_FULL_SLOT(1)
          ORLOJ_FULL_SLOT(0)
#undef ORLOJ_FULL_SLOT
          default:
            break;
        }
        // the partial slot c: member 32c + lane joins at k = 32c + lane + 1
#pragma unroll
        for (int i = 0; i < G; ++i) {
          float pr = ex2_approx(lds_f32(sgl[i] + 4 * lookup_bin(sigp, a2[i], wB2[i], mg[i], sh[i])));
          pr = lane <= kg + i ? pr : 0.f;
          part[i] += pr;
          if (!PICK && p.P && lane <= kg + i && k0 + i <= K)
            p.P[q * tri + (int64_t)(k0 + i) * (k0 + i - 1) / 2 + 32 * c + lane] = pr;
        }
#pragma unroll
        for (int i = 0; i < G; ++i)
          if (k0 + i > K) part[i] = partL[i] = 0.f;   // tail of the last group
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        Ek = bfly_push(pend, part[i], kg + i, lane);
        if (!PICK && p.EL) Sk = bfly_push(pendL, partL[i], kg + i, lane);
      }
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
