/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (parity oracle; never on the product path).
 *
 * A plain, slow, obviously correct fp64 CPU implementation of what the Orloj
 * batch-scoring hot path computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares no code, header, table or constant with
 * paper_2209_00159_b200/ (the CUDA path) and includes nothing from it.
 *
 * Model (PAPER.md problem statement :241-255; Eq. 3-9 :477-543), with the
 * readings of DESIGN.md §3:
 *   - member execution times X_j are independent, each discrete
 *     on the grid {tau_1..tau_B} with pmf counts[d_j][i] / total[d_j]   (A1);
 *   - a batch of the first k queue members runs L = a_k + w_k * max_j X_j
 *     ticks (Eq. 3 :479-484 + Eq. 4 :486-491 + Eq. 9 in CDF form :537-541),
 *     X in bin units;
 *   - P_r(k) = Pr(t + L <= D_r)  (step cost, miss <=> penalty :411-419; A11
 *     inclusive deadline);  E_k = sum_{r<=k} P_r(k);  k* = smallest argmax (A10).
 * The CDF of the max is the product of the member CDFs (Eq. 6 :503-507 for the
 * i.i.d. case; Eq. 8 :512-535 integrates to the same product, see
 * tests/test_oracle_eq8.py), evaluated here in the LINEAR domain, in fp64,
 * with no logarithms.
 *
 * Every function is pinned by tests in tests/test_oracle_*.py (closed forms,
 * brute-force enumeration, Eq. 8 literal evaluator, exact worked examples,
 * invariants).  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ECOLD 2

static void set_threads(int32_t nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

int32_t oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Step 1: the empirical CDF at the upper
 * bin edges, F_d(tau_i) = (sum_{j<=i} count[d][j]) / total_d, in fp64.
 * F[d*B + i-1] holds F_d(tau_i); F_d(tau_B) = 1 exactly.  total == 0 is the
 * cold-start error. */
int32_t oracle_cdf(const uint32_t *counts, int32_t D, int32_t B, double *F) {
  if (D < 0 || B < 1) return OR_EINVAL;
  for (int64_t d = 0; d < D; ++d) {
    uint64_t total = 0;
    for (int32_t i = 0; i < B; ++i) total += counts[d * B + i];
    if (total == 0) return OR_ECOLD;
    uint64_t cum = 0;
    for (int32_t i = 0; i < B; ++i) {
      cum += counts[d * B + i];
      F[d * B + i] = (double)cum / (double)total;
    }
  }
  return OR_OK;
}

/* Step 4 (Eq. 3-4, Eq. 9 CDF form): the largest bin m with a_k + w_k*m <= sigma,
 * clamped to [0, B]; int64 floor division (sigma - a_k >= 0 here).  P_r(k) is
 * then Pr(max bin <= i*) = G_k[i*] (0 when i* = 0, A12). */
static int64_t lookup(int64_t sigma, int64_t a, int64_t w, int32_t B) {
  int64_t x = sigma - a;
  if (x < 0) return 0;
  int64_t i = x / w;
  return i < B ? i : B;
}

/* Neumaier compensated sum. */
typedef struct { double s, c; } nsum;
static void nsum_add(nsum *acc, double x) {
  double t = acc->s + x;
  if (fabs(acc->s) >= fabs(x)) acc->c += (acc->s - t) + x;
  else acc->c += (x - t) + acc->s;
  acc->s = t;
}
static double nsum_get(const nsum *acc) { return acc->s + acc->c; }

/* Score one window (the first K members of a deadline-ordered queue) at time
 * `now`.  member_deadline[r], member_dist[r] for r < K.  Writes E[k-1] (k=1..K),
 * optionally P (packed, k(k-1)/2 + r) and EL (E[L_{B_k}], Eq. 5 with A5).
 * G has B+1 doubles of scratch.  Returns k* (smallest argmax; 0 iff K == 0). */
static int32_t score_window(const double *F, int32_t B, const int64_t *a, const int64_t *w,
                            int32_t K, const int64_t *member_deadline, const int32_t *member_dist,
                            int64_t now, double *E, double *P, double *EL, double *G) {
  /* G_0 = 1 for every bin; G[0] stands for "bin 0" (nothing fits) and stays 0. */
  G[0] = 0.0;
  for (int32_t i = 1; i <= B; ++i) G[i] = 1.0;
  int32_t best = 0;
  double bestE = 0.0;
  for (int32_t k = 1; k <= K; ++k) {
    /* Step 3: G_k[i] = prod_{j<=k} F_{d_j}(tau_i) (Eq. 6/8 product form). */
    const double *Fd = F + (int64_t)member_dist[k - 1] * B;
    for (int32_t i = 1; i <= B; ++i) G[i] *= Fd[i - 1];
    /* Steps 2, 4, 5, 6: sigma_r, lookup, P_r(k), E_k. */
    nsum acc = {0.0, 0.0};
    for (int32_t r = 0; r < k; ++r) {
      int64_t sigma = member_deadline[r] - now;
      int64_t istar = lookup(sigma, a[k - 1], w[k - 1], B);
      double p = istar == 0 ? 0.0 : G[istar];
      if (P) P[(int64_t)k * (k - 1) / 2 + r] = p;
      nsum_add(&acc, p);
    }
    double Ek = nsum_get(&acc);
    E[k - 1] = Ek;
    if (EL) {
      /* Eq. 5: E[L_B] = a_k + w_k * E[max bin], E[max bin] = sum_i i*(G_k[i]-G_k[i-1]). */
      nsum m = {0.0, 0.0};
      for (int32_t i = 1; i <= B; ++i) nsum_add(&m, (double)i * (G[i] - G[i - 1]));
      EL[k - 1] = (double)a[k - 1] + (double)w[k - 1] * nsum_get(&m);
    }
    /* Step 7: argmax, ties -> smallest k (A10). */
    if (k == 1 || Ek > bestE) {
      best = k;
      bestE = Ek;
    }
  }
  return best;
}

/* O1: score every queue.  Queue q holds members [offsets[q], offsets[q+1]) in
 * (deadline, arrival, index) order; K_q = min(n_q, kmax).  Outputs:
 * E[q*kmax + k-1] (0 for k > K_q), optional P[q*kmax(kmax+1)/2 + k(k-1)/2 + r],
 * optional EL[q*kmax + k-1], best_k[q], best_E[q]. */
int32_t oracle_score(const double *F, int32_t D, int32_t B, const int64_t *a, const int64_t *w,
                     int32_t kmax, int64_t Q, const int64_t *offsets, const int64_t *deadline,
                     const int32_t *dist, const int64_t *now, double *E, double *P, double *EL,
                     int32_t *best_k, double *best_E, int32_t nthreads) {
  if (kmax < 1 || B < 1 || Q < 0) return OR_EINVAL;
  (void)D;
  set_threads(nthreads);
  const int64_t tri = (int64_t)kmax * (kmax + 1) / 2;
  int32_t err = OR_OK;
#pragma omp parallel
  {
    double *G = (double *)malloc(sizeof(double) * (B + 1));
#pragma omp for schedule(dynamic, 16)
    for (int64_t q = 0; q < Q; ++q) {
      int64_t off = offsets[q];
      int64_t n = offsets[q + 1] - off;
      int32_t K = (int32_t)(n < kmax ? n : kmax);
      double *Eq = E + q * kmax;
      for (int32_t k = 0; k < kmax; ++k) Eq[k] = 0.0;
      double *ELq = EL ? EL + q * kmax : NULL;
      if (ELq)
        for (int32_t k = 0; k < kmax; ++k) ELq[k] = 0.0;
      double *Pq = P ? P + q * tri : NULL;
      if (Pq)
        for (int64_t j = 0; j < tri; ++j) Pq[j] = 0.0;
      int32_t kb = score_window(F, B, a, w, K, deadline + off, dist + off, now[q], Eq, Pq, ELq, G);
      best_k[q] = kb;
      best_E[q] = kb ? Eq[kb - 1] : 0.0;
    }
    free(G);
  }
  return err;
}

/* O3: brute-force joint-outcome enumeration for one tiny queue.  For each k it
 * walks every outcome (x_1..x_k) in {1..B}^k, accumulates the probability of
 * each value of max_j x_j, and sets P_r(k) = sum over m of pmf_max(m) *
 * [now + a_k + w_k * m <= D_r] — the deadline test itself, not the floor
 * formula.  pmf from counts (fp64).  P packed like oracle_score.  Parallel over
 * the first outcome.  Cost sum_k B^k. */
int32_t oracle_bruteforce(const uint32_t *counts, int32_t D, int32_t B, const int64_t *a,
                          const int64_t *w, int32_t K, const int64_t *deadline, const int32_t *dist,
                          int64_t now, double *P, double *E, int32_t nthreads) {
  if (K < 0 || K > 12 || B < 1) return OR_EINVAL;
  set_threads(nthreads);
  double *pmf = (double *)malloc(sizeof(double) * (size_t)D * B);
  for (int64_t d = 0; d < D; ++d) {
    uint64_t tot = 0;
    for (int32_t i = 0; i < B; ++i) tot += counts[d * B + i];
    if (tot == 0) {
      free(pmf);
      return OR_ECOLD;
    }
    for (int32_t i = 0; i < B; ++i) pmf[d * B + i] = (double)counts[d * B + i] / (double)tot;
  }
  double *pmax = (double *)malloc(sizeof(double) * (B + 1));
  for (int32_t k = 1; k <= K; ++k) {
    for (int32_t m = 0; m <= B; ++m) pmax[m] = 0.0;
#pragma omp parallel
    {
      double *loc = (double *)calloc((size_t)B + 1, sizeof(double));
      int32_t x[16];
      double pr[17];
      int32_t mx[17];
#pragma omp for schedule(dynamic, 1)
      for (int32_t x1 = 1; x1 <= B; ++x1) {
        double p1 = pmf[(int64_t)dist[0] * B + x1 - 1];
        if (p1 == 0.0) continue;
        if (k == 1) {
          loc[x1] += p1;
          continue;
        }
        /* odometer over x_2..x_k */
        pr[1] = p1;
        mx[1] = x1;
        for (int32_t j = 2; j <= k; ++j) x[j] = 1;
        int32_t depth = 2; /* first level whose prefix must be recomputed */
        for (;;) {
          for (int32_t j = depth; j <= k; ++j) {
            pr[j] = pr[j - 1] * pmf[(int64_t)dist[j - 1] * B + x[j] - 1];
            mx[j] = mx[j - 1] > x[j] ? mx[j - 1] : x[j];
          }
          loc[mx[k]] += pr[k];
          int32_t j = k;
          while (j >= 2 && x[j] == B) x[j--] = 1;
          if (j < 2) break;
          ++x[j];
          depth = j;
        }
      }
#pragma omp critical
      for (int32_t m = 0; m <= B; ++m) pmax[m] += loc[m];
      free(loc);
    }
    double Ek = 0.0;
    for (int32_t r = 0; r < k; ++r) {
      double p = 0.0;
      for (int32_t m = 1; m <= B; ++m)
        if (now + a[k - 1] + w[k - 1] * (int64_t)m <= deadline[r]) p += pmax[m];
      P[(int64_t)k * (k - 1) / 2 + r] = p;
      Ek += p;
    }
    E[k - 1] = Ek;
  }
  free(pmax);
  free(pmf);
  return OR_OK;
}

/* ---------------------------------------------------------------------------
 * O2: trace replay (SURVEY §8(a) a7 with readings A9, A11, A15-A17).
 *
 * Per scenario (constant SLO, so deadline order = arrival order, A9):
 *   t <- first arrival; while arrivals remain or the carry is non-empty:
 *     if the carry is empty and the next arrival is later than t: t <- it
 *       (work-conserving worker, A15);
 *     scan the live queue (carry, then arrivals <= t) from the head: drop each
 *       hopeless request (P_r(1) = 0 exactly, A16) — counted `dropped` — and
 *       append the others to the window until it holds kmax members;
 *     carry <- window (even when empty);
 *     if the window is empty: continue;
 *     k* <- argmax_k E_k on the window (free mode), or the logged GPU choice
 *       (follow mode; asserted to be in the tie set T);
 *     dispatch the first k*: dur = a_k* + w_k* * max true_bin (Eq. 3-4);
 *       finished += #{t + dur <= D_r} (A11), late += the rest (A17);
 *     t <- t + dur; carry <- window[k*:].
 * Counters per scenario: total, finished, dropped, late, batches, busy_ticks,
 * span_ticks (= end time - first arrival).
 * Decision log layout (shared with the C-ABI): decision d of scenario s at
 * [arr_off[s] + s + d], terminated by 0.
 * ------------------------------------------------------------------------- */
/* Drop rules.  mode 0 (A16): r is hopeless iff P_r(1) = 0 exactly, i.e. the
 * looked-up bin i*(r,1) is 0 or F_{d_r}(tau_i*) = 0.  mode 1 (Alg. 1's drop,
 * PAPER.md:351 with EstimateBatchLatency(r, 1) = a_1 + w_1 E[bin_r], Eq. 3 and
 * Eq. 5 for a batch of one): drop iff t + a_1 + w_1 E[bin] > D_r, evaluated
 * exactly in integers as (sigma - a_1) * total < w_1 * sum_i i count_i. */
static int drop_request(const double *F, int32_t B, const int64_t *a, const int64_t *w, int64_t sigma,
                        int32_t d, int32_t mode, const int64_t *exp_num, const int64_t *exp_den) {
  if (mode == 0) {
    int64_t i1 = lookup(sigma, a[0], w[0], B);
    return (i1 == 0) || F[(int64_t)d * B + i1 - 1] == 0.0;
  }
  __int128 lhs = (__int128)(sigma - a[0]) * exp_den[d];
  __int128 rhs = (__int128)w[0] * exp_num[d];
  return lhs < rhs;
}

int32_t oracle_replay(const double *F, int32_t D, int32_t B, const int64_t *a, const int64_t *w,
                      int32_t kmax, int64_t S, const int64_t *arr_off, const int64_t *arrival,
                      const int32_t *dist, const int16_t *true_bin, const int64_t *slo,
                      int64_t *counters /* [S][7] */, const int32_t *follow_log,
                      int32_t *log_out, int64_t *tie_info /* [S][3] or NULL */, int32_t nthreads,
                      int32_t objective /* 0: E_k, 1: E_k / E[L_{B_k}] */,
                      int32_t drop_mode /* 0: hopeless (A16), 1: expected latency (Alg. 1) */,
                      const uint32_t *counts /* [D][B], needed for drop_mode 1 */,
                      const int64_t *t_start /* [S] or NULL: worker busy until then (feedback epochs) */,
                      int64_t *t_end /* [S] or NULL: end of the last batch */,
                      uint8_t *outcome /* [N] or NULL: 1 finished, 2 late, 3 dropped */) {
  if (kmax < 1 || B < 1 || S < 0) return OR_EINVAL;
  if (drop_mode == 1 && !counts) return OR_EINVAL;
  set_threads(nthreads);
  int64_t *exp_num = (int64_t *)calloc((size_t)D + 1, sizeof(int64_t));
  int64_t *exp_den = (int64_t *)calloc((size_t)D + 1, sizeof(int64_t));
  if (drop_mode == 1)
    for (int64_t d = 0; d < D; ++d)
      for (int32_t i = 0; i < B; ++i) {
        exp_num[d] += (int64_t)(i + 1) * counts[d * B + i]; /* sum_i i count_i (tau_i = i bins) */
        exp_den[d] += counts[d * B + i];
      }
#pragma omp parallel
  {
    double *G = (double *)malloc(sizeof(double) * (B + 1));
    double *E = (double *)malloc(sizeof(double) * kmax);
    double *EL = (double *)malloc(sizeof(double) * kmax);
    int64_t *win = (int64_t *)malloc(sizeof(int64_t) * kmax);
    int64_t *carry = (int64_t *)malloc(sizeof(int64_t) * kmax);
    int64_t *wdl = (int64_t *)malloc(sizeof(int64_t) * kmax);
    int32_t *wd = (int32_t *)malloc(sizeof(int32_t) * kmax);
#pragma omp for schedule(dynamic, 1)
    for (int64_t s = 0; s < S; ++s) {
      const int64_t base = arr_off[s];
      const int64_t n = arr_off[s + 1] - base;
      int64_t c_fin = 0, c_drop = 0, c_late = 0, c_bat = 0, c_busy = 0;
      int64_t ndec = 0, nties = 0, first_bad = -1;
      int64_t cursor = 0;
      int32_t ncarry = 0;
      int64_t t = t_start ? t_start[s] : INT64_MIN;
      while (cursor < n || ncarry > 0) {
        if (ncarry == 0 && arrival[base + cursor] > t) t = arrival[base + cursor];
        /* scan: carry first, then admitted arrivals */
        int32_t wc = 0;
        for (int32_t c = 0; c < ncarry; ++c) {
          int64_t r = carry[c];
          if (drop_request(F, B, a, w, arrival[base + r] + slo[s] - t, dist[base + r], drop_mode, exp_num,
                           exp_den)) {
            ++c_drop;
            if (outcome) outcome[base + r] = 3;
          } else
            win[wc++] = r;
        }
        while (wc < kmax && cursor < n && arrival[base + cursor] <= t) {
          int64_t r = cursor++;
          if (drop_request(F, B, a, w, arrival[base + r] + slo[s] - t, dist[base + r], drop_mode, exp_num,
                           exp_den)) {
            ++c_drop;
            if (outcome) outcome[base + r] = 3;
          } else
            win[wc++] = r;
        }
        ncarry = 0;
        if (wc == 0) continue;
        for (int32_t j = 0; j < wc; ++j) {
          wdl[j] = arrival[base + win[j]] + slo[s];
          wd[j] = dist[base + win[j]];
        }
        int32_t ko = score_window(F, B, a, w, wc, wdl, wd, t, E, NULL, objective ? EL : NULL, G);
        if (objective) {
          /* finish-rate objective: argmax E_k / E[L_{B_k}] (Eq. 1's 1/E[L], Eq. 5), ties -> smallest k */
          ko = 1;
          for (int32_t kk = 1; kk <= wc; ++kk) {
            E[kk - 1] = E[kk - 1] / EL[kk - 1];
            if (E[kk - 1] > E[ko - 1]) ko = kk;
          }
        }
        int32_t k = ko;
        if (follow_log) {
          int32_t kg = follow_log[base + s + ndec];
          double emax = E[ko - 1];
          /* tie band: E_k within 1e-5 k; for the rate, relative 1e-4 (E[L] error) plus the E band over E[L] */
          double band = objective ? 1e-4 * emax + 1e-5 * (double)(ko + kg) /
                                                      (kg >= 1 && kg <= wc && EL[kg - 1] < EL[ko - 1] ? EL[kg - 1]
                                                                                                     : EL[ko - 1])
                                  : 1e-5 * (double)(ko + kg);
          int ok = kg >= 1 && kg <= wc && E[kg - 1] >= emax - band;
          if (!ok && first_bad < 0) first_bad = ndec;
          if (kg != ko) ++nties;
          if (kg >= 1 && kg <= wc) k = kg;
        }
        if (log_out) log_out[base + s + ndec] = k;
        ++ndec;
        int64_t m = 0;
        for (int32_t j = 0; j < k; ++j)
          if (true_bin[base + win[j]] > m) m = true_bin[base + win[j]];
        int64_t dur = a[k - 1] + w[k - 1] * m;
        for (int32_t j = 0; j < k; ++j) {
          int fin = t + dur <= wdl[j]; /* A11: inclusive deadline */
          if (fin) ++c_fin;
          else ++c_late;
          if (outcome) outcome[base + win[j]] = fin ? 1 : 2;
        }
        ++c_bat;
        c_busy += dur;
        t += dur;
        for (int32_t j = k; j < wc; ++j) carry[ncarry++] = win[j];
      }
      if (log_out) log_out[base + s + ndec] = 0;
      if (t_end) t_end[s] = t;
      int64_t *cs = counters + s * 7;
      cs[0] = n;
      cs[1] = c_fin;
      cs[2] = c_drop;
      cs[3] = c_late;
      cs[4] = c_bat;
      cs[5] = c_busy;
      cs[6] = n > 0 ? t - arrival[base] : 0;
      if (tie_info) {
        tie_info[s * 3 + 0] = ndec;
        tie_info[s * 3 + 1] = nties;
        tie_info[s * 3 + 2] = first_bad;
      }
    }
    free(G);
    free(E);
    free(win);
    free(carry);
    free(wdl);
    free(wd);
    free(EL);
  }
  free(exp_num);
  free(exp_den);
  return OR_OK;
}
