/*
 * gen_host.c — host build of the integer generators in gen_common.h.  Used to
 * regenerate, on the CPU, exactly the inputs the device build produces for the
 * queues / scenarios the oracle checks.  No method arithmetic here.
 */
#include <stdint.h>
#include "gen_common.h"

/* counts of rows rho_list[0..n) -> out[n][B] */
void gen_rows_host(uint64_t seed, const uint64_t *rho_list, int64_t n, const uint32_t *templates,
                   int32_t T, int32_t B, uint32_t *out) {
  for (int64_t r = 0; r < n; ++r)
    for (int32_t i = 0; i < B; ++i)
      out[r * B + i] = gen_row_count(seed, rho_list[r], templates, T, B, i);
}

/* Trace of scenarios scen_ids[0..S), n_arr arrivals each, laid out contiguously
 * (scenario k occupies [k*n_arr, (k+1)*n_arr)).  arrival = t0 + inclusive prefix
 * sum of gaps. */
void gen_trace_host(uint64_t seed, const uint64_t *scen_ids, int64_t S, int64_t n_arr,
                    const uint32_t *exp_q16, uint64_t base_gap, int32_t n_apps,
                    const uint32_t *cum /* [n_apps][B] */, int32_t B, int64_t t0,
                    int64_t *arrival, int32_t *dist, int16_t *true_bin) {
  for (int64_t k = 0; k < S; ++k) {
    uint64_t s = scen_ids[k];
    int64_t t = t0;
    for (int64_t j = 0; j < n_arr; ++j) {
      t += (int64_t)gen_gap(seed, s, (uint64_t)j, exp_q16, base_gap);
      int32_t app = gen_app(seed, s, (uint64_t)j, n_apps);
      arrival[k * n_arr + j] = t;
      dist[k * n_arr + j] = app;
      true_bin[k * n_arr + j] = gen_true_bin(seed, s, (uint64_t)j, cum + (int64_t)app * B, B);
    }
  }
}
