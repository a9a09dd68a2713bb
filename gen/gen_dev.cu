/*
 * gen_dev.cu — device build of the integer generators in gen_common.h, used to
 * materialise the full-size C3 rows (16.8 M x 256 counts) and C5 traces
 * (819 M arrivals) directly in HBM.  Input generation only: no method
 * arithmetic.  Bit-identical to gen_host.c by construction (integer-only).
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include "gen_common.h"

__global__ void gen_rows_kernel(uint64_t seed, uint64_t rho0, int64_t n_rows,
                                const uint32_t *__restrict__ templates, int32_t T, int32_t B,
                                uint32_t *__restrict__ out) {
  int64_t total = n_rows * (int64_t)B;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / B;
    int32_t i = (int32_t)(e - r * B);
    out[e] = gen_row_count(seed, rho0 + (uint64_t)r, templates, T, B, i);
  }
}

/* one warp per scenario; 32 arrivals per step with a warp inclusive scan */
__global__ void gen_trace_kernel(uint64_t seed, const uint64_t *__restrict__ scen_ids, int64_t S,
                                 int64_t n_arr, const uint32_t *__restrict__ exp_q16,
                                 uint64_t base_gap, int32_t n_apps,
                                 const uint32_t *__restrict__ cum, int32_t B, int64_t t0,
                                 int64_t *__restrict__ arrival, int32_t *__restrict__ dist,
                                 int16_t *__restrict__ true_bin) {
  int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (k >= S) return;
  uint64_t s = scen_ids[k];
  int64_t t = t0;
  for (int64_t j0 = 0; j0 < n_arr; j0 += 32) {
    int64_t j = j0 + lane;
    bool ok = j < n_arr;
    int64_t g = ok ? (int64_t)gen_gap(seed, s, (uint64_t)j, exp_q16, base_gap) : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t v = __shfl_up_sync(0xffffffffu, g, o);
      if (lane >= o) g += v;
    }
    if (ok) {
      int32_t app = gen_app(seed, s, (uint64_t)j, n_apps);
      arrival[k * n_arr + j] = t + g;
      dist[k * n_arr + j] = app;
      true_bin[k * n_arr + j] = gen_true_bin(seed, s, (uint64_t)j, cum + (int64_t)app * B, B);
    }
    t += __shfl_sync(0xffffffffu, g, 31);
  }
}

extern "C" int gen_rows_dev(uint64_t seed, uint64_t rho0, int64_t n_rows, const uint32_t *templates,
                            int32_t T, int32_t B, uint32_t *out, void *stream) {
  if (n_rows <= 0) return 0;
  gen_rows_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(seed, rho0, n_rows, templates, T, B, out);
  return (int)cudaGetLastError();
}

extern "C" int gen_trace_dev(uint64_t seed, const uint64_t *scen_ids, int64_t S, int64_t n_arr,
                             const uint32_t *exp_q16, uint64_t base_gap, int32_t n_apps,
                             const uint32_t *cum, int32_t B, int64_t t0, int64_t *arrival,
                             int32_t *dist, int16_t *true_bin, void *stream) {
  if (S <= 0) return 0;
  int64_t threads = S * 32;
  int blocks = (int)((threads + 255) / 256);
  gen_trace_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(seed, scen_ids, S, n_arr, exp_q16, base_gap,
                                                            n_apps, cum, B, t0, arrival, dist, true_bin);
  return (int)cudaGetLastError();
}
