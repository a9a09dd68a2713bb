// thresholds.cu — exact host-side thresholds of the replay policies
// (include/orloj.h, PAPER.md:345-358 drop pass, :585-593
// batch model from all distributions).  Off the critical path (computed once
// per store, like the paper's per-bs precompute) and exact: every
// quantity is an integer or a ratio of integers, so a threshold is the exact
// ceiling, never a rounded float.  A small unsigned big integer carries the
// powers F_mix^bs of the mixture CDF over a common denominator.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/orloj.h"
#include "host_util.h"

using namespace orloj::host;

namespace {

// little-endian base-2^32 unsigned integer
struct Big {
  std::vector<uint32_t> d;
  Big() = default;
  explicit Big(uint64_t v) {
    while (v) {
      d.push_back((uint32_t)v);
      v >>= 32;
    }
  }
  void trim() {
    while (!d.empty() && d.back() == 0) d.pop_back();
  }
  bool zero() const { return d.empty(); }
  size_t bits() const {
    if (d.empty()) return 0;
    size_t b = 32 * (d.size() - 1);
    for (uint32_t x = d.back(); x; x >>= 1) ++b;
    return b;
  }
};

Big add(const Big &a, const Big &b) {
  Big r;
  const size_t n = a.d.size() > b.d.size() ? a.d.size() : b.d.size();
  r.d.resize(n + 1);
  uint64_t c = 0;
  for (size_t i = 0; i < n; ++i) {
    c += (i < a.d.size() ? a.d[i] : 0ull) + (i < b.d.size() ? b.d[i] : 0ull);
    r.d[i] = (uint32_t)c;
    c >>= 32;
  }
  r.d[n] = (uint32_t)c;
  r.trim();
  return r;
}

Big sub(const Big &a, const Big &b) {  // a >= b
  Big r;
  r.d.resize(a.d.size());
  int64_t br = 0;
  for (size_t i = 0; i < a.d.size(); ++i) {
    int64_t v = (int64_t)a.d[i] - (i < b.d.size() ? (int64_t)b.d[i] : 0) - br;
    br = v < 0;
    r.d[i] = (uint32_t)(v + (br ? (1ll << 32) : 0));
  }
  r.trim();
  return r;
}

Big mul(const Big &a, uint64_t m) {
  if (a.zero() || m == 0) return Big();
  const uint32_t lo = (uint32_t)m, hi = (uint32_t)(m >> 32);
  Big r;
  r.d.assign(a.d.size() + 2, 0);
  for (int part = 0; part < 2; ++part) {
    const uint64_t f = part ? hi : lo;
    if (!f) continue;
    uint64_t c = 0;
    for (size_t i = 0; i < a.d.size(); ++i) {
      c += (uint64_t)a.d[i] * f + r.d[i + part];
      r.d[i + part] = (uint32_t)c;
      c >>= 32;
    }
    for (size_t k = a.d.size() + part; c; ++k) {
      c += r.d[k];
      r.d[k] = (uint32_t)c;
      c >>= 32;
    }
  }
  r.trim();
  return r;
}

Big mul(const Big &a, const Big &b) {
  if (a.zero() || b.zero()) return Big();
  Big r;
  r.d.assign(a.d.size() + b.d.size(), 0);
  for (size_t i = 0; i < a.d.size(); ++i) {
    uint64_t c = 0;
    for (size_t j = 0; j < b.d.size(); ++j) {
      c += (uint64_t)a.d[i] * b.d[j] + r.d[i + j];
      r.d[i + j] = (uint32_t)c;
      c >>= 32;
    }
    r.d[i + b.d.size()] = (uint32_t)c;
  }
  r.trim();
  return r;
}

Big shl(const Big &a, unsigned s) {
  if (a.zero()) return a;
  Big r;
  const unsigned w = s / 32, b = s % 32;
  r.d.assign(a.d.size() + w + 1, 0);
  for (size_t i = 0; i < a.d.size(); ++i) {
    const uint64_t v = (uint64_t)a.d[i] << b;
    r.d[i + w] |= (uint32_t)v;
    r.d[i + w + 1] |= (uint32_t)(v >> 32);
  }
  r.trim();
  return r;
}

int cmp(const Big &a, const Big &b) {
  if (a.d.size() != b.d.size()) return a.d.size() < b.d.size() ? -1 : 1;
  for (size_t i = a.d.size(); i-- > 0;)
    if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
  return 0;
}

uint64_t mod_small(const Big &a, uint64_t m) {  // m < 2^63
  unsigned __int128 r = 0;
  for (size_t i = a.d.size(); i-- > 0;) r = ((r << 32) | a.d[i]) % m;
  return (uint64_t)r;
}

Big div_small(const Big &a, uint64_t m) {  // exact or floor division by m < 2^63
  Big q;
  q.d.assign(a.d.size(), 0);
  unsigned __int128 r = 0;
  for (size_t i = a.d.size(); i-- > 0;) {
    r = (r << 32) | a.d[i];
    q.d[i] = (uint32_t)(r / m);
    r %= m;
  }
  q.trim();
  return q;
}

uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) {
    const uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// ceil(num / den) for a quotient known to be < 2^62
int64_t ceil_div(const Big &num, const Big &den) {
  uint64_t q = 0;
  for (int bit = 62; bit >= 0; --bit) {
    const uint64_t t = q | (1ull << bit);
    if (cmp(mul(den, t), num) <= 0) q = t;
  }
  return (int64_t)(q + (cmp(mul(den, q), num) < 0 ? 1 : 0));
}

orloj_status check_counts(const uint32_t *counts, int32_t D, int32_t B, std::vector<uint64_t> *tot) {
  if (!counts || D < 1 || B < 1) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "thresholds: need host counts [D][B]");
  tot->assign(D, 0);
  for (int32_t d = 0; d < D; ++d) {
    for (int32_t i = 0; i < B; ++i) (*tot)[d] += counts[(int64_t)d * B + i];
    if ((*tot)[d] == 0) return fail(ORLOJ_ERR_COLD_START, "thresholds: histogram %d has total 0", d);
  }
  return ORLOJ_OK;
}

orloj_status check_profile(const orloj_latency_profile *pr) {
  if (!pr || pr->kmax < 1 || !pr->offset_ticks || !pr->ticks_per_bin)
    return fail(ORLOJ_ERR_INVALID_ARGUMENT, "thresholds: profile missing");
  for (int k = 0; k < pr->kmax; ++k)
    if (pr->offset_ticks[k] < 0 || pr->ticks_per_bin[k] < 1 || pr->offset_ticks[k] > (1ll << 40) ||
        pr->ticks_per_bin[k] > (1ll << 40))
      return fail(ORLOJ_ERR_INVALID_ARGUMENT, "thresholds: profile entry %d out of range", k + 1);
  return ORLOJ_OK;
}

}  // namespace

extern "C" {

orloj_status orloj_expected_latency_thresholds(const uint32_t *counts, int32_t D, int32_t B,
                                               const orloj_latency_profile *profile, int64_t *thr) {
  ORLOJ_NVTX("orloj_expected_latency_thresholds");
  std::vector<uint64_t> tot;
  orloj_status st;
  if ((st = check_counts(counts, D, B, &tot))) return st;
  if ((st = check_profile(profile))) return st;
  if (!thr) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "thresholds: output NULL");
  const unsigned __int128 a1 = (unsigned __int128)profile->offset_ticks[0];
  const unsigned __int128 w1 = (unsigned __int128)profile->ticks_per_bin[0];
  for (int32_t d = 0; d < D; ++d) {
    unsigned __int128 num = 0;  // sum_i i c_i: bin i's mass at its upper edge tau_i (A1)
    for (int32_t i = 0; i < B; ++i) num += (unsigned __int128)(i + 1) * counts[(int64_t)d * B + i];
    const unsigned __int128 den = tot[d];
    thr[d] = (int64_t)(a1 + (w1 * num + den - 1) / den);
  }
  return ok();
}

orloj_status orloj_alg1_size_thresholds(const uint32_t *counts, int32_t D, int32_t B, const double *weights,
                                        const orloj_latency_profile *profile, int64_t *thr) {
  ORLOJ_NVTX("orloj_alg1_size_thresholds");
  std::vector<uint64_t> tot;
  orloj_status st;
  if ((st = check_counts(counts, D, B, &tot))) return st;
  if ((st = check_profile(profile))) return st;
  if (!thr) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "thresholds: output NULL");
  // exact mixture weights: w_d = m_d 2^{e_d} (a double is a dyadic rational), scaled by 2^{-min e}
  std::vector<Big> W(D);
  {
    int emin = 1 << 30;
    std::vector<uint64_t> m(D);
    std::vector<int> ex(D);
    bool any = false;
    for (int32_t d = 0; d < D; ++d) {
      const double x = weights ? weights[d] : 1.0;
      if (!(x >= 0.0) || x > 1e300) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "thresholds: weight %d not finite >= 0", d);
      if (x == 0.0) continue;
      int e2;
      const double fr = std::frexp(x, &e2);                  // x = fr 2^e2, fr in [0.5, 1)
      m[d] = (uint64_t)std::ldexp(fr, 53);                    // exact 53-bit mantissa
      ex[d] = e2 - 53;
      emin = ex[d] < emin ? ex[d] : emin;
      any = true;
    }
    if (!any) return fail(ORLOJ_ERR_INVALID_ARGUMENT, "thresholds: all weights are 0");
    for (int32_t d = 0; d < D; ++d)
      if (m[d]) {
        if (ex[d] - emin > 4096) return fail(ORLOJ_ERR_CAPACITY, "thresholds: weights span more than 2^4096");
        W[d] = shl(Big(m[d]), (unsigned)(ex[d] - emin));
      }
  }
  // common denominator L = lcm(totals); K_d = W_d L / tot_d; M = sum_d K_d tot_d = L sum_d W_d
  Big L(1);
  for (int32_t d = 0; d < D; ++d) {
    const uint64_t g = gcd64(mod_small(L, tot[d]), tot[d]);
    L = mul(L, tot[d] / g);
    if (L.bits() > 65536) return fail(ORLOJ_ERR_CAPACITY, "thresholds: common denominator too large");
  }
  std::vector<Big> K(D);
  Big M;
  for (int32_t d = 0; d < D; ++d) {
    if (W[d].zero()) continue;
    K[d] = mul(W[d], div_small(L, tot[d]));
    M = add(M, mul(K[d], tot[d]));
  }
  // F_mix(tau_i) = N_i / M (N_B = M)
  std::vector<Big> N(B);
  std::vector<uint64_t> cum(D, 0);
  for (int32_t i = 0; i < B; ++i) {
    Big acc;
    for (int32_t d = 0; d < D; ++d) {
      cum[d] += counts[(int64_t)d * B + i];
      if (!K[d].zero() && cum[d]) acc = add(acc, mul(K[d], cum[d]));
    }
    N[i] = acc;
  }
  // E[L_bs] = a_bs + w_bs sum_i (G_i - G_{i-1}) (i - 1/2), G_i = (N_i / M)^bs, uniform within bins (R11);
  // by parts: sum_i (G_i - G_{i-1}) (2i - 1) = (2B - 1) - 2 sum_{i<B} G_i, so over 2 M^bs:
  // X = (2B - 1) M^bs - 2 sum_{i<B} N_i^bs and thr_bs = a_bs + ceil(w_bs X / (2 M^bs)).
  std::vector<Big> P(N.begin(), N.end());  // N_i^bs
  Big Mb = M;
  for (int k = 0; k < profile->kmax; ++k) {
    if (k > 0) {
      for (int32_t i = 0; i + 1 < B; ++i) P[i] = mul(P[i], N[i]);
      Mb = mul(Mb, M);
    }
    Big S;
    for (int32_t i = 0; i + 1 < B; ++i) S = add(S, P[i]);
    const Big X = sub(mul(Mb, (uint64_t)(2 * B - 1)), mul(S, 2));
    const Big num = mul(X, (uint64_t)profile->ticks_per_bin[k]);
    thr[k] = profile->offset_ticks[k] + ceil_div(num, mul(Mb, 2));
  }
  return ok();
}

}  // extern "C"
