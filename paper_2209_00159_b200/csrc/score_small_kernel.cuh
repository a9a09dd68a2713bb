// score_small_kernel.cuh — K1/K2 for short queues over a small store (kmax <= 32,
// B <= 64, the store staged in shared memory: C1, C2, C4 of SURVEY §8(d)).
//
// Same quantities as score_kernel.cuh, laid out for
// queues that fit one warp:
//   LG_k[i] = LG_{k-1}[i] + log2 F_{d_k}(tau_i)   lanes over bins; rows LG_1..LG_K
//                                                   staged in shared memory, each
//                                                   with a -inf head for i* = 0
//   lane r-1 then owns member r: for k = 1..32 (unrolled, so a_k, w_k and the
//   division magic are immediate constant-bank operands) it looks up
//   P_r(k) = 2^{LG_k[i*(r,k)]} in row k — every lane reads the same row, so the
//   data-dependent bins are distinct banks or broadcasts (no bank conflicts) —
//   and pushes it into the transposing butterfly (common.cuh), which leaves
//   E_k = sum_{r<=k} P_r(k) in lane k-1 after 31 shuffles.
// The adds that build LG_k are the same fp32 adds in the same order as
// score_kernel's, so LG and every P_r(k) are identical; E_k is the same
// butterfly tree as score_kernel's, within the 1e-5 k tolerance.  Argmax: two
// REDUX (max of float bits, then min k).  Used by pick and by score when
// neither P nor E[L_B] is requested.
#pragma once
#include "common.cuh"
#include "score_kernel.cuh"

namespace orloj {

constexpr int SMALL_WARPS = 8;

// shared memory: store [D][B] | lookup constants int4 [32] | per warp LG rows [32][32 BPL + 1]
template <int BPL>
struct SmallShape {
  static constexpr int ROW = 32 * BPL + 1;  // row k-1: [0] = -inf (i* = 0), [i] = LG_k(tau_i)
  __host__ __device__ static size_t bytes(int D, int B) {
    return (((size_t)D * B * 4 + 15) & ~(size_t)15) + 32 * 16 + (size_t)SMALL_WARPS * 32 * ROW * 4;
  }
};

template <int BPL, bool PICK>
__global__ void __launch_bounds__(SMALL_WARPS * 32) score_small_kernel(const __grid_constant__ ScoreParams p) {
  constexpr int ROW = SmallShape<BPL>::ROW;
  extern __shared__ __align__(16) float s_dyn[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int D = p.D, B = p.B, kmax = p.kmax;
  float *s_store = s_dyn;
  int4 *s_prof = reinterpret_cast<int4 *>(s_dyn + (((size_t)D * B + 3) & ~(size_t)3));
  float *lgs = reinterpret_cast<float *>(s_prof + 32) + wid * 32 * ROW;  // row k-1 = LG_k

  // the queue's offsets / now are requested before the block stages the store,
  // so their latency overlaps the staging and the barrier
  const int64_t q = (int64_t)blockIdx.x * SMALL_WARPS + wid;
  const bool live = q < p.Q;
  int64_t o0 = 0, o1 = 0, now = 0;
  if (live) {
    o0 = p.offsets[q];
    o1 = p.offsets[q + 1];
    now = p.now[q];
  }
  const int64_t base0 = p.offsets[0];  // offsets may start at any base (chunked calls)

  for (int e = threadIdx.x * 4; e < D * B; e += blockDim.x * 4)
    *reinterpret_cast<float4 *>(s_store + e) = __ldg(reinterpret_cast<const float4 *>(p.log2F + e));
  if (threadIdx.x < 32) {  // sizes beyond kmax: constants that look up bin 0 (never counted)
    const int k = threadIdx.x;
    s_prof[k] = k < kmax ? make_int4(p.prof.a2[k], p.prof.wB2[k], (int)p.prof.mag[k], (int)p.prof.sh[k])
                         : make_int4(0, 0, 0, 0);
  }
  lgs[lane * ROW] = -INFINITY;
  __syncthreads();

  if (!live) return;
  const int64_t off = o0 - base0;
  const int64_t n = o1 - o0;
  const int K = (int)(n < kmax ? n : kmax);
  // both member loads unconditional (a lane past the end re-reads the last member, masked below)
  int64_t dl = 0;
  int32_t dd = 0;
  if (n > 0) {
    const int64_t j = off + (lane < n ? lane : n - 1);
    dl = p.deadline[j];
    dd = p.dist[j];
  }
  const int32_t sig = lane < K ? sigma2(dl - now) : 0;
  const int idB = lane < K ? dd * B * 4 : 0;  // byte offset of member lane's row

  // a2: LG_k for k = 1..K, lanes over bins (bin lane + 32 e + 1); 32-bit
  // shared-space addresses (common.cuh SArr), kept in registers
  float acc[BPL];
#pragma unroll
  for (int e = 0; e < BPL; ++e) acc[e] = 0.f;
  bool bok[BPL];
#pragma unroll
  for (int e = 0; e < BPL; ++e) bok[e] = lane + 32 * e < B;
  const uint32_t a_lane = smem_base(s_store) + 4u * lane;
  const SArr<float> dst{opaque_u32(smem_addr(lgs) + 4u * (1 + lane))};
  if (K == 32 && B == 32 * BPL) {  // full queue, full bins (C2, C4): unrolled, unpredicated
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const uint32_t src = a_lane + (uint32_t)__shfl_sync(FULL, idB, k);
#pragma unroll
      for (int e = 0; e < BPL; ++e) {
        acc[e] += lds_f32_nv(src + 128u * e);
        dst.st(k * ROW + 32 * e, acc[e]);
      }
    }
  } else {
#pragma unroll 8
  for (int k = 0; k < K; ++k) {
    const uint32_t src = a_lane + (uint32_t)__shfl_sync(FULL, idB, k);
#pragma unroll
    for (int e = 0; e < BPL; ++e) {
      if (bok[e]) {
        acc[e] += lds_f32_nv(src + 128u * e);  // read-only store: free to issue ahead
        dst.st(k * ROW + 32 * e, acc[e]);
      }
    }
  }
  }
  __syncwarp();

  // a3-a5: lane r-1 looks up its member in every row k (constants of size k:
  // one broadcast 128-bit load); the butterfly sums over r.  Lanes >= K hold
  // sigma = 0, i.e. bin 0 and P = 0; rows k > K were not built, but they only
  // reach E_k for k > K, which is never used.
  const uint32_t row0 = opaque_u32(smem_addr(lgs));
  float pend[5];
  float E = 0.f;
#pragma unroll
  for (int k = 1; k <= 32; ++k) {
    const int4 c = s_prof[k - 1];
    const int bi = lookup_bin(sig, c.x, c.y, (uint32_t)c.z, (uint32_t)c.w);
    const float x = ex2_approx(lds_f32_nv(row0 + 4u * (uint32_t)((k - 1) * ROW + bi)));
    const float v = lane < k ? x : 0.f;  // members r <= k
    E = bfly_push(pend, v, k - 1, lane);
  }

  // a6: argmax, ties -> smallest k (E >= 0: float bits order like values)
  const int k = lane + 1;
  const bool valid = k <= K;
  if constexpr (PICK) {
    const uint32_t bits = valid ? __float_as_uint(E) : 0u;
    const uint32_t mx = __reduce_max_sync(FULL, bits);
    const uint32_t kb = __reduce_min_sync(FULL, (valid && bits == mx) ? (uint32_t)k : 0x7fffffffu);
    if (lane == 0) {
      p.best_k[q] = K == 0 ? 0 : (int32_t)kb;
      p.best_E[q] = K == 0 ? 0.f : __uint_as_float(mx);
    }
  } else {
    if (k <= kmax && p.E) p.E[q * kmax + k - 1] = valid ? E : 0.f;
  }
}

}  // namespace orloj
