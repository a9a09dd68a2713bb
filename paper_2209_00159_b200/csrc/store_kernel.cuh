// store_kernel.cuh — a0: integer counts -> log2 CDF rows, and validation kernels.
//
// F_d(tau_i) = cum_i / total_d in fp64 (reading A1), log2 in
// fp64, rounded once to fp32 (RN).  cum == total gives F = 1 and log2 = 0.0f
// exactly; cum == 0 gives -inf.  One warp per row: a warp-wide inclusive scan
// of the integer counts (exact), 32 bins at a time.
#pragma once
#include "common.cuh"

namespace orloj {

// min_total: rows with fewer samples are left as they are (the feedback loop's
// refresh keeps a row until its window holds enough samples); a row with total
// 0 sets *cold when `cold` is given (orloj_store_build: COLD_START).
__global__ void store_build_kernel(const uint32_t *__restrict__ counts, int32_t D, int32_t B,
                                   float *__restrict__ out, unsigned int *__restrict__ cold,
                                   uint64_t min_total = 1) {
  const int lane = threadIdx.x & 31;
  const int64_t d = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (d >= D) return;
  const uint32_t *row = counts + d * B;
  uint64_t total = 0;
  for (int i = lane; i < B; i += 32) total += row[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(FULL, total, o);
  if (total == 0 || total < min_total) {
    if (total == 0 && cold && lane == 0) atomicOr(cold, 1u);
    return;
  }
  uint64_t carry = 0;
  for (int i0 = 0; i0 < B; i0 += 32) {
    const int i = i0 + lane;
    uint64_t c = i < B ? row[i] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t u = __shfl_up_sync(FULL, c, o);
      if (lane >= o) c += u;
    }
    const uint64_t cum = carry + c;
    if (i < B) {
      float v;
      if (cum == 0) v = -INFINITY;
      else if (cum == total) v = 0.0f;
      else v = __double2float_rn(log2((double)cum / (double)total));
      out[d * B + i] = v;
    }
    carry += __shfl_sync(FULL, c, 31);
  }
}

// Online profiler: sample j adds 1 to counts[d][i-1],
// i = clamp(ceil(solo / bin_ticks), 1, B) (upper-edge bins, A1).  A CTA-private
// histogram in shared memory when it fits, flushed with one atomic per
// non-zero counter; otherwise global atomics.
__global__ void hist_accumulate_kernel(const int32_t *__restrict__ dist, const int64_t *__restrict__ solo,
                                       int64_t n, int64_t bin_ticks, uint32_t *__restrict__ counts, int32_t D,
                                       int32_t B, int use_smem) {
  extern __shared__ uint32_t s_h[];
  const int DB = D * B;
  if (use_smem) {
    for (int e = threadIdx.x; e < DB; e += blockDim.x) s_h[e] = 0;
    __syncthreads();
  }
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int d = dist[j];
    if (d < 0 || d >= D) continue;
    const int64_t x = solo[j];
    int64_t i = x <= 0 ? 1 : (x + bin_ticks - 1) / bin_ticks;
    i = i < 1 ? 1 : (i > B ? B : i);
    const int e = d * B + (int)i - 1;
    if (use_smem) atomicAdd(&s_h[e], 1u);
    else atomicAdd(&counts[e], 1u);
  }
  if (use_smem) {
    __syncthreads();
    for (int e = threadIdx.x; e < DB; e += blockDim.x)
      if (s_h[e]) atomicAdd(&counts[e], s_h[e]);
  }
}

// Long-term feedback loop ("finished requests are sampled
// and sent to the profiler to evaluate individually"): a replayed arrival whose
// outcome is completed (1 finished, 2 late; 3 = dropped never ran) and whose
// sample mask is non-zero adds its solo execution time — in the replay the
// hidden true bin — to counts[d][bin-1].  Same CTA-private histogram scheme.
__global__ void profile_outcomes_kernel(const int32_t *__restrict__ dist, const int16_t *__restrict__ true_bin,
                                        const uint8_t *__restrict__ outcome, const uint8_t *__restrict__ mask,
                                        int64_t n, uint32_t *__restrict__ counts, int32_t D, int32_t B,
                                        int use_smem) {
  extern __shared__ uint32_t s_h[];
  const int DB = D * B;
  if (use_smem) {
    for (int e = threadIdx.x; e < DB; e += blockDim.x) s_h[e] = 0;
    __syncthreads();
  }
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned oc = outcome[j];
    if ((oc != 1u && oc != 2u) || (mask && !mask[j])) continue;
    const int d = dist[j], i = true_bin[j];
    if (d < 0 || d >= D || i < 1 || i > B) continue;
    const int e = d * B + i - 1;
    if (use_smem) atomicAdd(&s_h[e], 1u);
    else atomicAdd(&counts[e], 1u);
  }
  if (use_smem) {
    __syncthreads();
    for (int e = threadIdx.x; e < DB; e += blockDim.x)
      if (s_h[e]) atomicAdd(&counts[e], s_h[e]);
  }
}

__global__ void fill_i64_kernel(int64_t *__restrict__ x, int64_t n, int64_t v) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    x[j] = v;
}

// flags: bit0 = value / shape violation, bit1 = order violation
__global__ void validate_store_kernel(const float *__restrict__ F, int32_t D, int32_t B,
                                      unsigned int *flags) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)D * B;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % B);
    const float v = F[e];
    bool bad = !(v <= 0.f);                        // NaN or positive
    if (i == B - 1) bad |= v != 0.f;
    if (i > 0) bad |= F[e - 1] > v;
    if (bad) atomicOr(flags, 1u);
  }
}

__global__ void validate_queues_kernel(const int64_t *__restrict__ off, int64_t Q,
                                       const int64_t *__restrict__ arrival,
                                       const int64_t *__restrict__ deadline,
                                       const int32_t *__restrict__ dist, int32_t D,
                                       unsigned int *flags) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t base = off[0];
  for (int64_t q = tid + 1; q <= Q; q += stride)
    if (off[q] < off[q - 1]) atomicOr(flags, 1u);
  for (int64_t q = tid; q < Q; q += stride) {
    const int64_t b = off[q] - base, e = off[q + 1] - base;
    for (int64_t j = b; j < e; ++j) {
      if (dist[j] < 0 || dist[j] >= D) atomicOr(flags, 1u);
      if (j > b) {
        const bool lt = deadline[j - 1] < deadline[j];
        const bool eq = deadline[j - 1] == deadline[j];
        const bool ok = lt || (eq && (arrival == nullptr || arrival[j - 1] <= arrival[j]));
        if (!ok) atomicOr(flags, 2u);
      }
    }
  }
}

__global__ void validate_trace_kernel(const int64_t *__restrict__ off, int64_t S,
                                      const int64_t *__restrict__ arrival,
                                      const int32_t *__restrict__ dist,
                                      const int16_t *__restrict__ tb,
                                      const int64_t *__restrict__ slo,
                                      const int32_t *__restrict__ bucket, int32_t nb, int32_t D,
                                      int32_t B, unsigned int *flags) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = tid; s <= S; s += stride) {
    if (s == 0 && off[0] != 0) atomicOr(flags, 1u);
    if (s > 0 && (off[s] < off[s - 1] || off[s] - off[s - 1] > 0x7fffffbfll)) atomicOr(flags, 1u);
  }
  for (int64_t s = tid; s < S; s += stride) {
    if (slo[s] < 0 || bucket[s] < 0 || bucket[s] >= nb) atomicOr(flags, 1u);
    const int64_t b = off[s], e = off[s + 1];
    for (int64_t j = b; j < e; ++j) {
      if (dist[j] < 0 || dist[j] >= D || tb[j] < 1 || tb[j] > B) atomicOr(flags, 1u);
      if (j > b && arrival[j - 1] > arrival[j]) atomicOr(flags, 2u);
    }
  }
}

}  // namespace orloj
