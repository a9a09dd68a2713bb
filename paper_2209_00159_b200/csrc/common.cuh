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
// state).  For every k (index k-1): a_k, w_k, and for the bin lookup the
// doubled offsets 2 a_k, 2 w_k B and the exact division magic (mag, sh) for
// floor(x / w_k), 0 <= x < 2^30 (see lookup_bin).
struct ProfileDev {
  int32_t kmax;
  int32_t B;
  int32_t a[KCAP];
  int32_t w[KCAP];
  int32_t a2[KCAP];
  int32_t wB2[KCAP];
  uint32_t mag[KCAP];
  uint32_t sh[KCAP];
};

// Slack sigma = D_r - t, clamped to [0, 2^30 - 1] and doubled.  Clamping below
// at 0 changes nothing (floor(x / w) = 0 for every x < w, and x = sigma - a_k
// <= 0 there); above, the horizon a_kmax + w_kmax B <= 2^30 - 1 (checked on the
// host) makes every lookup saturate at B already.
__device__ __forceinline__ int32_t sigma2(int64_t sigma) {
  // on the two 32-bit halves: negative -> 0, >= 2^32 -> the cap, else min(lo, cap)
  const int32_t hi = (int32_t)(sigma >> 32);
  const uint32_t lo = (uint32_t)sigma;
  const uint32_t c = hi < 0 ? 0u : hi > 0 ? 0x3fffffffu : min(lo, 0x3fffffffu);
  return (int32_t)(2u * c);
}

// Eq. 3-4 + Eq. 9 (CDF form): i*(r,k) = clamp(floor((sigma - a_k) / w_k), 0, B)
// from s2 = 2 sigma:  x2 = clamp(s2 - 2 a_k, 0, 2 w_k B) = 2x,  and
// floor(x / w) = umulhi(2x, m) >> c with c = ceil(log2 w), m = ceil(2^(31+c) / w)
// < 2^32 — exact for every 0 <= x < 2^31 since x (m w - 2^(31+c)) < 2^31 w <=
// 2^(31+c).  Four integer instructions, bit-exact.
__device__ __forceinline__ int32_t lookup_bin(int32_t s2, int32_t a2, int32_t wB2, uint32_t mag,
                                              uint32_t sh) {
  int32_t x2 = s2 - a2;
  x2 = x2 < wB2 ? x2 : wB2;
  x2 = x2 > 0 ? x2 : 0;
  return (int32_t)(__umulhi((uint32_t)x2, mag) >> sh);
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

// A lane's bins: NV vectors of V floats (V = min(BPL, 4)).  Vector v of lane l
// covers floats [(32 v + l) V, +V) of a row, so each vector load / store of a
// warp is one contiguous, conflict-free 32 V-byte-per-lane sweep.
template <int V> struct alignas(4 * V) Vec {
  float x[V];
};

// Row loads of V floats (aligned to 4V bytes).  STREAM: rows read exactly once
// (the per-request store of C3) bypass L1.
template <int V, bool STREAM>
__device__ __forceinline__ Vec<V> ldrow(const float *p) {
  Vec<V> r;
  if constexpr (V == 4) {
    if constexpr (STREAM) {
      asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]) : "l"(p));
    } else {
      const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
      r.x[0] = v.x; r.x[1] = v.y; r.x[2] = v.z; r.x[3] = v.w;
    }
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

// Store V floats (V <= 4) to shared memory as one vector store.
template <int V>
__device__ __forceinline__ void st_vec(float *dst, const float *v) {
  if constexpr (V == 4) {
    *reinterpret_cast<float4 *>(dst) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2 *>(dst) = make_float2(v[0], v[1]);
  } else {
    dst[0] = v[0];
  }
}

// Warp-uniform copy of a value that is equal across the warp: REDUX writes a
// uniform register, so branches on it compile to uniform branches (no
// BSSY / BSYNC reconvergence bookkeeping).
__device__ __forceinline__ int warp_uniform(int x) {
  return (int)__reduce_max_sync(FULL, (unsigned)x);
}

// ---- bulk async copies (TMA engine, cp.async.bulk) + mbarriers -------------

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// 32-bit shared-space load (the address already includes the buffer base).
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

// Non-volatile form for read-only phases: free to be scheduled among other
// loads; the caller makes the address depend on a value produced after the
// barrier that ends the writes (e.g. an opaque_u32 base taken after it).
__device__ __forceinline__ float lds_f32_nv(uint32_t addr) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// ---- 32-bit shared-space arrays -------------------------------------------
// A generic pointer into dynamic shared memory makes the compiler rebuild the
// CTA's shared window base (S2UR CgaCtaId, ULEA, ...) at every access of a hot
// loop rather than spend a register on it; a 32-bit shared-space address kept
// in one register and explicit ld/st.shared avoid that.  smem_base() returns
// the address through an opaque move so it is computed once.
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  asm volatile("mov.u32 %0, %1;" : "=r"(x) : "r"(x));
  return x;
}
__device__ __forceinline__ uint32_t smem_base(const void *p) { return opaque_u32(smem_addr(p)); }
// a pointer the compiler must keep (or spill) rather than rebuild from thread / block ids in a loop
template <class T>
__device__ __forceinline__ T *opaque_ptr(T *p) {
  uint64_t x = reinterpret_cast<uint64_t>(p);
  asm volatile("mov.b64 %0, %1;" : "=l"(x) : "l"(x));
  return reinterpret_cast<T *>(x);
}

template <class T> struct SArr;
template <> struct SArr<int64_t> {
  uint32_t a;
  __device__ __forceinline__ int64_t ld(int i) const {
    int64_t v;
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(a + 8u * (uint32_t)i) : "memory");
    return v;
  }
  __device__ __forceinline__ void st(int i, int64_t v) const {
    asm volatile("st.shared.s64 [%0], %1;" ::"r"(a + 8u * (uint32_t)i), "l"(v) : "memory");
  }
};
template <> struct SArr<int32_t> {
  uint32_t a;
  __device__ __forceinline__ int32_t ld(int i) const {
    int32_t v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a + 4u * (uint32_t)i) : "memory");
    return v;
  }
  __device__ __forceinline__ void st(int i, int32_t v) const {
    asm volatile("st.shared.s32 [%0], %1;" ::"r"(a + 4u * (uint32_t)i), "r"(v) : "memory");
  }
};
template <> struct SArr<float> {
  uint32_t a;
  __device__ __forceinline__ float ld(int i) const {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a + 4u * (uint32_t)i) : "memory");
    return v;
  }
  __device__ __forceinline__ void st(int i, float v) const {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a + 4u * (uint32_t)i), "f"(v) : "memory");
  }
  // V consecutive floats starting at element i (4V-byte aligned)
  template <int V>
  __device__ __forceinline__ void ldv(int i, float (&x)[V]) const {
    const uint32_t ad = a + 4u * (uint32_t)i;
    if constexpr (V == 4)
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]) : "r"(ad)
                   : "memory");
    else if constexpr (V == 2)
      asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x[0]), "=f"(x[1]) : "r"(ad) : "memory");
    else
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[0]) : "r"(ad) : "memory");
  }
  template <int V>
  __device__ __forceinline__ void stv(int i, const float *x) const {
    const uint32_t ad = a + 4u * (uint32_t)i;
    if constexpr (V == 4)
      asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(ad), "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3])
                   : "memory");
    else if constexpr (V == 2)
      asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(ad), "f"(x[0]), "f"(x[1]) : "memory");
    else
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(ad), "f"(x[0]) : "memory");
  }
};
__device__ __forceinline__ int4 lds_v4s32(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
               : "memory");
  return v;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

// Make mbarrier initialisation visible to the async proxy.  CTA-local barriers
// only need the proxy fence; the cluster-scope fence.mbarrier_init also flushes
// L1 (CCTL.IVALL), which every warp of this kernel would pay.
__device__ __forceinline__ void mbar_init_fence() {
#ifdef ORLOJ_CLUSTER_INIT_FENCE
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#else
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
}

// Wait until the phase with parity `phase` of the barrier has completed.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(phase)
      : "memory");
}

// Order this thread's earlier generic-proxy shared-memory accesses before
// subsequent async-proxy (bulk copy) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Bulk copy of `bytes` (multiple of 16, 16-B aligned both sides) from global to
// shared memory completing on `bar`, issued only where `pred` is set (one lane
// per warp) — predicated, so the warp does not diverge.
template <bool STREAM>
__device__ __forceinline__ void bulk_row(bool pred, uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                                         uint64_t pol) {
  if constexpr (STREAM)
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %5, 0;\n"
        " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4; }" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol), "r"((int)pred)
        : "memory");
  else
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
        " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3]; }" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "r"((int)pred)
        : "memory");
}

// Arm `bar` for `bytes` of incoming bulk copies (predicated like bulk_row),
// after ordering earlier generic shared-memory reads of the refilled buffer
// before the async-proxy writes.
__device__ __forceinline__ void arm_barrier(bool pred, uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %2, 0;\n"
      " @p fence.proxy.async.shared::cta;\n"
      " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1; }" ::"r"(bar),
      "r"(bytes), "r"((int)pred)
      : "memory");
}

}  // namespace orloj
