// score_small_kernel.cuh — K1/K2 for short queues over a small store (kmax <= 32,
// B <= 64, the store staged in shared memory: C1, C2, C4 of SURVEY §8(d)).
//
// Same quantities as score_kernel.cuh, laid out for
// queues that fit one warp, with no per-warp shared memory:
//   LG_k[i] = LG_{k-1}[i] + log2 F_{d_k}(tau_i)   lanes over bins (bin lane + 32 e + 1),
//                                                   held in registers across the warp
//   lane r-1 owns member r: right after LG_k is formed (k = 1..32, unrolled, so
//   a_k, w_k and the division magic are constant-bank operands of the kernel
//   parameters) it looks up P_r(k) = 2^{LG_k[i*(r,k)]} with one shuffle from
//   lane i* - 1 (i* = 0: P = 0) and pushes it into the transposing butterfly
//   (common.cuh), which leaves E_k = sum_{r<=k} P_r(k) in lane k-1 after 31
//   shuffles.
// Shared memory holds only the store: the rows LG_k are never written back, so
// the kernel's shared-memory traffic is the 32 store-row reads per queue (the
// earlier layout staged every row and gathered from it: ~235 wavefronts per C4
// queue, which bounded it).  The adds that build LG_k are the same fp32 adds in
// the same order as score_kernel's, so LG and every P_r(k) are identical; E_k is
// the same butterfly tree as score_kernel's, within the 1e-5 k tolerance.
// Argmax: two REDUX (max of float bits, then min k).  Used by pick and by score
// when neither P nor E[L_B] is requested.
#pragma once
#include "common.cuh"
#include "score_kernel.cuh"

namespace orloj {

#ifndef ORLOJ_SMALL_WARPS
#define ORLOJ_SMALL_WARPS 4
#endif
constexpr int SMALL_WARPS = ORLOJ_SMALL_WARPS;  // queues (warps) per block

// shared memory: the store [D][B]
template <int BPL>
struct SmallShape {
  __host__ __device__ static size_t bytes(int D, int B) { return ((size_t)D * B * 4 + 15) & ~(size_t)15; }
};

// GSTORE: the store stays in global memory (too large to stage: e.g. one row
// per request), each lane reading its bins of member k's row (read-only path)
template <int BPL, bool PICK, bool GSTORE = false>
__global__ void __launch_bounds__(SMALL_WARPS * 32) score_small_kernel(const __grid_constant__ ScoreParams p) {
  extern __shared__ __align__(16) float s_dyn[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int D = p.D, B = p.B, kmax = p.kmax;
  float *s_store = s_dyn;

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

  if constexpr (!GSTORE) {
    for (int e = threadIdx.x * 4; e < D * B; e += blockDim.x * 4)
      *reinterpret_cast<float4 *>(s_store + e) = __ldg(reinterpret_cast<const float4 *>(p.log2F + e));
    __syncthreads();
  }

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
  const int32_t sig = lane < K ? sigma2(dl - now) : 0;  // lanes >= K: bin 0, P = 0
  const int idB = lane < K ? dd * B * 4 : 0;            // byte offset of member lane's row (shared store)
  const int idR = lane < K ? dd : 0;                    // member lane's row (global store)
  // a lane's store column per vector (lanes past the last bin re-read bin B - 1:
  // in bounds, never looked up since i* <= B)
  uint32_t col[BPL];
#pragma unroll
  for (int e = 0; e < BPL; ++e) col[e] = smem_base(s_store) + 4u * (uint32_t)min(lane + 32 * e, B - 1);

  float acc[BPL];
#pragma unroll
  for (int e = 0; e < BPL; ++e) acc[e] = 0.f;
  float pend[5];
  float E = 0.f;
  const int nlane = -lane;
#pragma unroll
  for (int k = 1; k <= 32; ++k) {
    // a2: LG_k over the lanes (rows past K add row 0: they only reach E_k for k > K)
    if constexpr (GSTORE) {
      const float *row = p.log2F + (int64_t)__shfl_sync(FULL, idR, k - 1) * B;
#pragma unroll
      for (int e = 0; e < BPL; ++e) acc[e] += __ldg(row + min(lane + 32 * e, B - 1));
    } else {
      const uint32_t rk = (uint32_t)__shfl_sync(FULL, idB, k - 1);
#pragma unroll
      for (int e = 0; e < BPL; ++e) acc[e] += lds_f32_nv(col[e] + rk);  // read-only store: free to issue ahead
    }
    // a3-a4: member lane+1 at size k (constants beyond kmax are 0: bin 0)
    const int bi = lookup_bin(sig, p.prof.a2[k - 1], p.prof.wB2[k - 1], p.prof.mag[k - 1], p.prof.sh[k - 1]);
    const int from = bi - 1;  // shfl takes the source lane mod 32 (bi = 0: masked below)
    float lg = __shfl_sync(FULL, acc[0], from);
    if constexpr (BPL == 2) {
      const float lg1 = __shfl_sync(FULL, acc[1], from);
      lg = bi > 32 ? lg1 : lg;
    }
    const float x = ex2_approx(lg);
    // members r <= k (k - 1 - lane >= 0) with i* > 0 (bi - 1 >= 0): one min, one compare
    const float v = min(nlane + (k - 1), from) >= 0 ? x : 0.f;
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
