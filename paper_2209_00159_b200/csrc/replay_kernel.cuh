// replay_kernel.cuh — K3: deterministic trace replay, one warp per scenario
// (readings A9, A11, A15-A17 in DESIGN.md §3).
//
// Scenario state is (t, cursor, carry): with a constant SLO per scenario the
// deadline order equals arrival order (A9), so the live queue is exactly the
// window remainder ("carry", <= kmax entries, kept in shared memory) followed by
// arrivals [cursor, ...) with arrival <= t.  Per decision:
//   1. scan: carry, then admitted arrivals, 32 at a time; ballots split
//      hopeless (P_r(1) = 0 exactly <=> i*(r,1) < first non-empty bin of d_r,
//      integer test) from kept members; kept ones are compacted into the window
//      with popc ranks (shared-memory scatter), stopping at kmax (A16);
//   2. score the window exactly like score_kernel (lane = member, lanes also
//      own the bins; store rows from shared memory), keeping the 32 per-lane
//      P_lane(k) in registers and reducing them with the transposing butterfly
//      (pairs beyond the window skipped);
//   3. argmax (REDUX max on float bits, then min k), dispatch: dur = a_k* +
//      w_k* * max true_bin (REDUX max), finished / late by ballot (A11, A17);
//   4. t += dur; carry = window[k*:].
// Counters are kept warp-uniform and added to per-bucket int64 totals at the end.
#pragma once
#include "common.cuh"

namespace orloj {

struct ReplayParams {
  const float *log2F;
  int32_t D;
  int32_t B;
  int64_t S;
  const int64_t *arr_off;
  const int64_t *arrival;
  const int32_t *dist;
  const int16_t *true_bin;
  const int64_t *slo;
  const int32_t *bucket;
  unsigned long long *counters;  // [num_buckets][7]
  int32_t *log;                  // [N + S] or null
  ProfileDev prof;
};

constexpr int REPLAY_WARPS = 4;

template <int BPL>
__global__ void __launch_bounds__(REPLAY_WARPS * 32)
replay_kernel(const __grid_constant__ ReplayParams p) {
  constexpr int BPAD = 32 * BPL;
  constexpr int STG = BPAD + 4;

  extern __shared__ __align__(16) float s_dyn[];
  const int D = p.D, B = p.B;
  float *s_store = s_dyn;                                       // [D][B]
  int32_t *s_mmin = reinterpret_cast<int32_t *>(s_store + (size_t)D * B);  // [D]
  float *s_warp = reinterpret_cast<float *>(s_mmin + ((D + 3) & ~3));
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  float *stg0 = s_warp + wid * (2 * STG + 32) + 4;
  float *stg1 = stg0 + STG;
  int32_t *s_win = reinterpret_cast<int32_t *>(stg1 + BPAD);    // [32] window (scenario-relative indices)

  // stage the (small) store and the first non-empty bin of every distribution
  for (int e = threadIdx.x; e < D * B; e += blockDim.x) s_store[e] = p.log2F[e];
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    int m = B;
    for (int i = B - 1; i >= 0; --i)
      if (s_store[d * B + i] != -INFINITY) m = i + 1;
    s_mmin[d] = m;
  }
  if (lane == 0) {
    stg0[-1] = -INFINITY;
    stg1[-1] = -INFINITY;
  }
  __syncthreads();

  const int64_t s = (int64_t)blockIdx.x * REPLAY_WARPS + wid;
  if (s >= p.S) return;

  const int kmax = p.prof.kmax;
  const int64_t base = p.arr_off[s];
  const int64_t n = p.arr_off[s + 1] - base;
  const int64_t slo = p.slo[s];
  const int64_t *arr = p.arrival + base;
  const int32_t *dis = p.dist + base;
  const int16_t *tbs = p.true_bin + base;
  const int32_t a21 = p.prof.a2[0], wB21 = p.prof.wB2[0];
  const uint32_t mg1 = p.prof.mag[0], sh1 = p.prof.sh[0];

  int64_t t = INT64_MIN;
  int64_t cursor = 0;
  int ncarry = 0, carry_off = 0;
  long long c_fin = 0, c_drop = 0, c_late = 0, c_bat = 0, c_busy = 0;
  int64_t ndec = 0;

  while (cursor < n || ncarry > 0) {
    if (ncarry == 0) {
      const int64_t ac = arr[cursor];
      if (ac > t) t = ac;
    }
    // ---- 1. scan -------------------------------------------------------
    int wc = 0;
    if (ncarry > 0) {
      const bool valid = lane < ncarry;
      const int r = valid ? s_win[carry_off + lane] : 0;
      bool keep = false;
      if (valid) {
        const int32_t i1 = lookup_bin(sigma2(arr[r] + slo - t), a21, wB21, mg1, sh1);
        keep = i1 >= s_mmin[dis[r]];
      }
      const unsigned vm = __ballot_sync(FULL, valid);
      const unsigned km = __ballot_sync(FULL, keep);
      c_drop += __popc(vm & ~km);
      __syncwarp();
      if (keep) s_win[__popc(km & ((1u << lane) - 1u))] = r;
      wc = __popc(km);
    }
    while (wc < kmax && cursor < n) {
      const int64_t idx = cursor + lane;
      const bool valid = idx < n && arr[idx] <= t;
      const unsigned vm = __ballot_sync(FULL, valid);
      if (vm == 0) break;
      bool keep = false;
      if (valid) {
        const int32_t i1 = lookup_bin(sigma2(arr[idx] + slo - t), a21, wB21, mg1, sh1);
        keep = i1 >= s_mmin[dis[idx]];
      }
      const unsigned km = __ballot_sync(FULL, keep);
      const int need = kmax - wc;
      unsigned consumed = vm;  // arrivals are sorted: vm is a prefix
      if (__popc(km) >= need) {
        // lane of the need-th kept member: its inclusive kept-rank equals need
        const unsigned le = (lane == 31) ? FULL : ((1u << (lane + 1)) - 1u);
        const unsigned at = __ballot_sync(FULL, keep && __popc(km & le) == need);
        const int pos = __ffs(at) - 1;
        consumed = pos == 31 ? FULL : ((1u << (pos + 1)) - 1u);
      }
      const unsigned kc = km & consumed;
      c_drop += __popc(vm & consumed & ~km);
      if ((kc >> lane) & 1u) s_win[wc + __popc(kc & ((1u << lane) - 1u))] = (int)idx;
      wc += __popc(kc);
      const int nc = __popc(consumed);
      cursor += nc;
      if (nc < 32) break;
    }
    ncarry = 0;
    carry_off = 0;
    wc = warp_uniform(wc);
    __syncwarp();
    if (wc == 0) continue;

    // ---- 2. score the window ---------------------------------------------
    const bool mem = lane < wc;
    const int r = mem ? s_win[lane] : 0;
    const int64_t Dr = mem ? arr[r] + slo : 0;
    const int32_t sig = mem ? sigma2(Dr - t) : 0;
    const int dr = mem ? dis[r] : 0;
    const int tb = mem ? (int)tbs[r] : 0;

    float lg[BPL];
#pragma unroll
    for (int b = 0; b < BPL; ++b) lg[b] = 0.f;
    const bool vok = lane * BPL < B;
    float v[32];
#pragma unroll
    for (int kk = 0; kk < 32; ++kk) {
      v[kk] = 0.f;
      if (kk < wc) {
        const int d = __shfl_sync(FULL, dr, kk);
        if (vok) {
          const Vec<BPL> x = *reinterpret_cast<const Vec<BPL> *>(s_store + d * B + lane * BPL);
#pragma unroll
          for (int e = 0; e < BPL; ++e) lg[e] += x.x[e];
        }
        float *sg = (kk & 1) ? stg1 : stg0;
        st_vec<BPL>(sg + lane * BPL, lg);
        __syncwarp();
        if (lane <= kk) {
          const int i = lookup_bin(sig, p.prof.a2[kk], p.prof.wB2[kk], p.prof.mag[kk], p.prof.sh[kk]);
          v[kk] = ex2_approx(sg[i - 1]);
        }
      }
    }
    // transposing butterfly; pairs entirely beyond the window are zero
#pragma unroll
    for (int L = 0; L < 5; ++L) {
#pragma unroll
      for (int m = 0; m < (16 >> L); ++m) {
        if ((m << (L + 1)) < wc) v[m] = bfly_combine(v[2 * m], v[2 * m + 1], L, lane);
        else v[m] = 0.f;
      }
    }
    // ---- 3. argmax + dispatch ----------------------------------------------
    const float E = mem ? v[0] : 0.f;
    const uint32_t mx = __reduce_max_sync(FULL, mem ? __float_as_uint(E) : 0u);
    const int kstar = (int)__reduce_min_sync(FULL, (mem && __float_as_uint(E) == mx) ? (uint32_t)lane : 32u) + 1;
    const int mbin = (int)__reduce_max_sync(FULL, lane < kstar ? (uint32_t)tb : 0u);
    const int64_t dur = (int64_t)p.prof.a[kstar - 1] + (int64_t)p.prof.w[kstar - 1] * mbin;
    const unsigned fm = __ballot_sync(FULL, lane < kstar && t + dur <= Dr);
    c_fin += __popc(fm);
    c_late += kstar - __popc(fm);
    c_bat += 1;
    c_busy += dur;
    t += dur;
    if (p.log && lane == 0) p.log[base + s + ndec] = kstar;
    ++ndec;
    ncarry = wc - kstar;
    carry_off = kstar;
    __syncwarp();
  }
  if (lane == 0) {
    if (p.log) p.log[base + s + ndec] = 0;
    unsigned long long *cs = p.counters + (int64_t)p.bucket[s] * 7;
    atomicAdd(cs + 0, (unsigned long long)n);
    atomicAdd(cs + 1, (unsigned long long)c_fin);
    atomicAdd(cs + 2, (unsigned long long)c_drop);
    atomicAdd(cs + 3, (unsigned long long)c_late);
    atomicAdd(cs + 4, (unsigned long long)c_bat);
    atomicAdd(cs + 5, (unsigned long long)c_busy);
    atomicAdd(cs + 6, (unsigned long long)(n > 0 ? t - arr[0] : 0));
  }
}

}  // namespace orloj
