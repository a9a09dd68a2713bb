// common.cuh — device building blocks shared by the score / pick / replay kernels.
//
// Part of the product CUDA path (liborloj.so).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace orloj {

constexpr int KCAP = 256;          // ORLOJ_MAX_KMAX
constexpr unsigned FULL = 0xffffffffu;

// Latency profile as kernel parameters (constant bank; stream-safe, no global
// state).  For every k: a_k, w_k, w_k*B and the exact 32-bit division magic for
// floor(x / w_k), 0 <= x < 2^31 (see lookup_bin).  Index k-1.
struct ProfileDev {
  int32_t kmax;
  int32_t B;
  int32_t a[KCAP];
  int32_t w[KCAP];
  int32_t wB[KCAP];
  uint32_t mag[KCAP];
  uint32_t sh[KCAP];
};

// sigma = D_r - t clamped into int32: below 0 every lookup gives bin 0, above
// the horizon (a_kmax + w_kmax*B <= 2^31-1, checked on the host) every lookup
// saturates at B, so the clamp never changes a result.
__device__ __forceinline__ int32_t clamp_sigma(int64_t sigma) {
  sigma = sigma < -1 ? -1 : sigma;
  sigma = sigma > 0x7fffffffLL ? 0x7fffffffLL : sigma;
  return (int32_t)sigma;
}

// Eq. 3-4 + Eq. 9 (CDF form): i*(r,k) = clamp(floor((sigma - a_k) / w_k), 0, B).
// x = min(sigma - a_k, w_k*B) < 2^31; floor(x / w) = umulhi(2x, m) >> c with
// c = ceil(log2 w), m = ceil(2^(31+c) / w) < 2^32 — exact for every such x
// (x * (m*w - 2^(31+c)) < 2^31 * w <= 2^(31+c)).  Integer, bit-exact.
__device__ __forceinline__ int32_t lookup_bin(int32_t sig, int32_t a, int32_t wB, uint32_t mag,
                                              uint32_t sh) {
  int32_t x = sig - a;
  x = x < wB ? x : wB;
  uint32_t q = __umulhi((uint32_t)x << 1, mag) >> sh;
  return x < 0 ? 0 : (int32_t)q;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One level of the transposing butterfly: lanes whose bit L is 0 keep index
// `even` and send `odd`, the others the reverse.  After the five levels over 32
// values v_j (one per k), lane l holds sum over all lanes of v_l — 31 shuffles
// for 32 reductions instead of 160.
__device__ __forceinline__ float bfly_combine(float even, float odd, int L, int lane) {
  const bool hi = (lane >> L) & 1;
  const float keep = hi ? odd : even;
  const float send = hi ? even : odd;
  return keep + __shfl_xor_sync(FULL, send, 1 << L);
}

// Incremental form: push v_j for j = 0..31 in order (j a compile-time constant
// after unrolling); returns the fully reduced value after j = 31.
__device__ __forceinline__ float bfly_push(float (&pend)[5], float v, int j, int lane) {
#pragma unroll
  for (int L = 0; L < 5; ++L) {
    if (((j >> L) & 1) == 0) {
      pend[L] = v;
      return v;
    }
    v = bfly_combine(pend[L], v, L, lane);
  }
  return v;
}

// A lane's bins as one vector register group: V = 1, 2, 4 or 8 floats
// (V = 8 is one 256-bit load, new on sm_100).
template <int V> struct alignas(4 * V) Vec {
  float x[V];
};

// Row loads of V floats at p (aligned to 4V bytes).  STREAM: rows read exactly
// once (the per-request store of C3) bypass L1 and are marked evict-first in
// L2.  `half` (V = 8 only): only the first 4 floats exist (B % 8 == 4 tail).
template <int V, bool STREAM>
__device__ __forceinline__ Vec<V> ldrow(const float *p, bool half = false) {
  Vec<V> r;
  if constexpr (V == 8) {
    if (!half) {
      if constexpr (STREAM)
        asm volatile(
            "ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]),
              "=f"(r.x[6]), "=f"(r.x[7])
            : "l"(p));
      else
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                       "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7])
                     : "l"(p));
    } else {
      const float4 lo = __ldg(reinterpret_cast<const float4 *>(p));
      r.x[0] = lo.x; r.x[1] = lo.y; r.x[2] = lo.z; r.x[3] = lo.w;
      r.x[4] = r.x[5] = r.x[6] = r.x[7] = 0.f;
    }
  } else if constexpr (V == 4) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    r.x[0] = v.x; r.x[1] = v.y; r.x[2] = v.z; r.x[3] = v.w;
  } else if constexpr (V == 2) {
    const float2 v = __ldg(reinterpret_cast<const float2 *>(p));
    r.x[0] = v.x; r.x[1] = v.y;
  } else {
    r.x[0] = __ldg(p);
  }
  return r;
}

template <int V>
__device__ __forceinline__ Vec<V> vzero() {
  Vec<V> z;
#pragma unroll
  for (int i = 0; i < V; ++i) z.x[i] = 0.f;
  return z;
}

// Store V floats to shared memory as 128-bit (or narrower) stores.
template <int V>
__device__ __forceinline__ void st_stage(float *dst, const float (&v)[V]) {
  if constexpr (V >= 4) {
#pragma unroll
    for (int h = 0; h < V; h += 4)
      *reinterpret_cast<float4 *>(dst + h) = make_float4(v[h], v[h + 1], v[h + 2], v[h + 3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2 *>(dst) = make_float2(v[0], v[1]);
  } else {
    dst[0] = v[0];
  }
}

}  // namespace orloj
