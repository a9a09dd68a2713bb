/*
 * gen_common.h — seeded, integer-only input generators shared (as DATA
 * producers) by the CUDA path and the oracle.  This header holds NONE of the
 * method's arithmetic (no CDFs, products, lookups, probabilities): only
 * counter-based hashing, a mass-preserving integer perturbation of histogram
 * counts, and a piecewise-Poisson arrival process.  Every formula here is
 * integer, so the host build (gen_host.c, used to regenerate oracle subsets)
 * and the device build (gen_dev.cu, used for the full-size bench inputs)
 * produce bit-identical values; tests/test_gen.py and the GPU tests check it.
 *
 * Recipes are described in DESIGN.md §"Input recipe".
 */
#ifndef ORLOJ_GEN_COMMON_H
#define ORLOJ_GEN_COMMON_H
#include <stdint.h>

#ifdef __CUDACC__
#define GEN_FN __host__ __device__ static inline
#else
#define GEN_FN static inline
#endif

/* SplitMix64 finaliser. */
GEN_FN uint64_t gen_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Counter-based hash of (seed, stream, a, b). */
GEN_FN uint64_t gen_hash(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  uint64_t h = gen_mix64(seed ^ (stream * 0xA0761D6478BD642Full));
  h = gen_mix64(h ^ (a * 0xD1B54A32D192ED03ull));
  return gen_mix64(h ^ (b * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull));
}

/* ---- C3: per-request rows from templates ---------------------------------
 * Row rho copies template (h mod T) and moves 1/8 of the mass of one bin to a
 * neighbour (integer; the row total is unchanged).  Returns count of bin i. */
GEN_FN uint32_t gen_row_count(uint64_t seed, uint64_t rho, const uint32_t *templates,
                              int32_t T, int32_t B, int32_t i) {
  uint64_t h = gen_hash(seed, 11, rho, 0);
  const uint32_t *src = templates + (uint64_t)(h % (uint64_t)T) * (uint64_t)B;
  int32_t pi = (int32_t)((h >> 32) % (uint64_t)B);
  int32_t pj = (pi + 1 < B) ? pi + 1 : pi - 1;
  uint32_t delta = src[pi] >> 3;
  uint32_t c = src[i];
  if (i == pi) c -= delta;
  if (i == pj) c += delta;
  return c;
}

/* ---- C5: piecewise-constant-rate Poisson arrivals -------------------------
 * Inter-arrival gap j of scenario s: inverse-CDF exponential from a Q16 table
 * (exp_q16[u] = round(2^16 * -ln((u + 0.5) / 65536)), computed once on the
 * host in fp64 and handed to both builds), scaled by the block mean gap.  The
 * rate is multiplied by U[0.5, 1.5) every 1000 arrivals (stand-in for the
 * scaled Azure trace). */
GEN_FN uint64_t gen_gap(uint64_t seed, uint64_t s, uint64_t j, const uint32_t *exp_q16,
                        uint64_t base_gap) {
  uint64_t blk = j / 1000u;
  uint64_t f_q16 = 32768u + (gen_hash(seed, 21, s, blk) & 0xFFFFu); /* [0.5, 1.5) in Q16 */
  uint64_t mean_gap = (base_gap << 16) / f_q16;                      /* rate x f => gap / f */
  uint64_t u = gen_hash(seed, 22, s, j) & 0xFFFFu;
  return ((uint64_t)exp_q16[u] * mean_gap) >> 16;
}

/* Application (distribution id) of arrival j: uniform over n_apps. */
GEN_FN int32_t gen_app(uint64_t seed, uint64_t s, uint64_t j, int32_t n_apps) {
  return (int32_t)(gen_hash(seed, 23, s, j) % (uint64_t)n_apps);
}

/* Hidden true bin (1..B) of arrival j drawn from the app's integer counts:
 * smallest i with cum_i > u, u uniform on [0, total) with total = 2^30. */
GEN_FN int16_t gen_true_bin(uint64_t seed, uint64_t s, uint64_t j, const uint32_t *cum_row,
                            int32_t B) {
  uint32_t u = (uint32_t)(gen_hash(seed, 24, s, j) & ((1u << 30) - 1u));
  int32_t i = 0;
  while (i < B - 1 && cum_row[i] <= u) ++i;
  return (int16_t)(i + 1);
}

#endif /* ORLOJ_GEN_COMMON_H */
