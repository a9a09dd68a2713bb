// replay_kernel.cuh — K3: deterministic trace replay, one warp per scenario
// (readings A9, A11, A15-A17 in DESIGN.md §3).
//
// Scenario state is (t, cursor, carry): with a constant SLO per scenario the
// deadline order equals arrival order (A9), so the live queue is exactly the
// window remainder ("carry", <= kmax entries) followed by arrivals [cursor, ...)
// with arrival <= t.  The replay is a sequential decision chain per scenario,
// so the kernel is built for latency:
//  * every member carries its "hopeless time" h_r = D_r - a_1 - w_1 m_min(d_r):
//    r is hopeless at t (P_r(1) = 0 exactly, A16) iff t > h_r — one 64-bit
//    compare (i*(r,1) >= m  <=>  sigma_r >= a_1 + w_1 m, integer-exact);
//  * the window lives in shared memory as member fields (deadline, h,
//    distribution, hidden true bin), each lane holds one of the next 32
//    arrivals in registers, refilled one decision ahead and only consumed in a
//    later decision: scanning never waits on HBM;
//  * a window of one member is dispatched without scoring (single candidate);
//  * scoring runs in blocks of REPLAY_KB candidate sizes (windows are short,
//    mostly 1-3): the block's prefix rows LG_k are built and staged back to
//    back, then every member does its lookups (REPLAY_KB-way ILP) and writes
//    P_r(k) into a per-warp [k][r] matrix; lane k-1 then sums row k with
//    128-bit loads and a short adder tree;
//  * argmax by two REDUX (max of float bits, then min k), dispatch with one
//    more REDUX (max true bin) and one ballot (finished, A11 / late, A17).
// Counters are kept warp-uniform and added to per-bucket int64 totals at the end.
//
// Segmented replay (MODE 1 + MODE 2; exact, DESIGN.md §7 "segments").  A state
// at a loop top with nothing carried and the worker free by the next arrival j
// (ncarry == 0, t <= a_j) is a *regeneration point*: the rest of the run is the
// same as a fresh replay started at arrival j (the max-plus scan and the idle
// jump both give t'_j = a_j whatever t <= a_j was, and the lookahead, the scan
// and hence every later decision depend only on (t, cursor, carry)).  MODE 1
// runs G segments of a scenario in parallel, segment g from a fresh start at
// s_g = floor(g n / G) until its first loop top with cursor >= s_{g+1} (its
// end state), recording regeneration points with their prefix counters, and
// then runs on past s_{g+1} (the extension) recording regeneration points at
// the marks segment g+1 uses, until a few records after its first one.  MODE 2
// (one warp per scenario) stitches: the true run starts at segment 0's end
// state; wherever segment g-1's extension and segment g's records share a
// regeneration point, the true run is segment g-1 up to that point and segment
// g after it, so both parts' counters (and decision logs) are taken without
// re-running anything.  Otherwise the true run is re-run from segment g-1's end
// state until it reaches one of segment g's recorded regeneration points (or
// runs through the segment).  The counters and the log are those of the plain
// replay, bit for bit; only the critical path gets shorter.
#pragma once
#include "common.cuh"
#include "priority_kernel.cuh"

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
  const int64_t *drop_thr;       // [D] or null: drop iff D_r - t < thr[d_r] (null: hopeless rule)
  // Alg. 1 policy (ALG1): thr_bs = ceil(E[L_bs]) of the all-application batch
  // model [kmax]; Eq. 1-2 priority tables [kmax][2][B+1], log E[L] [kmax], b
  const int64_t *size_thr;
  const double *prio_table;
  const double *prio_logEL;
  double prio_b;
  ProfileDev prof;
  // segmented replay (MODE 1 / 2)
  int32_t G;                      // segments per scenario
  struct ReplaySeg *seg;          // [S][G]
  int32_t *seg_log;               // scratch decision logs of segments g >= 1 (MODE 1 with a log)
  unsigned long long *seg_stats;  // [5]: decisions re-run by the stitch, segments joined, segments crossed,
                                  //      decisions in the extensions, inconsistent-size flag (zeroed by the host)
  int64_t num_arrivals;           // MODE 1 / 2: the caller's arrival_offsets[S] (sizes seg_log)
  // MODE 0 epochs (feedback loop, include/orloj.h orloj_replay_epoch): replay only
  // arrivals [s_e, s_{e+1}) of each scenario, the worker free at t_carry[s]
  // (written back at the end), per-arrival outcomes (1 finished, 2 late, 3 dropped)
  int32_t epoch, num_epochs;
  int64_t *t_carry;
  uint8_t *outcome;
};

constexpr int SEG_REC = 20;  // regeneration points recorded per list
// Records sit at marks m_0 = 0, m_{k+1} = m_k + max(8, m_k / 2) arrivals past
// the list's base: a record is the first regeneration point at or past the next
// mark.  A segment run starts empty and regenerates often at first while the
// true run may still be clearing a backlog; marks spaced geometrically keep a
// record within ~1.5x of wherever the true run regenerates, and two runs that
// have become the same run record the same points from the next mark on.
__host__ __device__ inline int64_t seg_next_mark(int64_t m) { return m + (m / 2 > 8 ? m / 2 : 8); }
// the extension past s_{g+1} stops after its first regeneration point and this many more records
#ifndef ORLOJ_SEG_EXT_AFTER
#define ORLOJ_SEG_EXT_AFTER 1
#endif
constexpr int SEG_EXT_AFTER = ORLOJ_SEG_EXT_AFTER;
// a regeneration point: arrival index, decisions and counters {finished,
// dropped, late, batches, busy} of the recording run before that point
struct SegRec {
  long long j, ndec, ctr[5];
};
struct ReplaySeg {
  int64_t t, cursor, ndec;  // end state of the segment run (first loop top with cursor >= s_{g+1})
  long long ctr[5];
  int32_t ncarry, nrec, next, pad;
  SegRec rec[SEG_REC];  // the run's regeneration points in [s_g, s_{g+1}) (marks from s_g)
  SegRec ext[SEG_REC];  // its extension past the end state (marks from s_{g+1}; running counters)
  int64_t carry_D[32], carry_h[32];
  int32_t carry_d[32], carry_tb[32];
#ifdef ORLOJ_REPLAY_TIMELINE  // diagnostic builds: %globaltimer at the item's start / end, SM id
  long long tl[4];            // first pass start / end; (segment 0 only) stitch start / end
  int32_t tl_sm[2], tl_pad[2];
#endif
};
#ifdef ORLOJ_REPLAY_TIMELINE
__device__ __forceinline__ long long tl_now() {
  long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
__device__ __forceinline__ int tl_smid() {
  int v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}
#endif

// first arrival of segment g of G over n arrivals: floor(g n / G) without overflow
__host__ __device__ inline int64_t seg_begin(int64_t n, int g, int G) {
  return g >= G ? n : (n / G) * g + (n % G) * g / G;
}
// start of segment (s, g)'s scratch decision log.  The run of segment g with
// its extension (capped at s_{g+2}) makes at most (s_{g+2} - s_g) + 32
// decisions (members are dispatched once each; only the last iteration
// consumes arrivals past the cap, at most kmax <= 32 kept), so the regions
// [off_g, off_g + s_{g+2} - s_g + 34) are disjoint: per scenario 2n + 34 G
// entries, 2N + 34 S G in all.
__host__ __device__ inline int64_t seg_log_off(int64_t arr_off_s, int64_t s, int64_t n, int g, int G) {
  return 2 * arr_off_s + seg_begin(n, g, G) + seg_begin(n, g + 1, G) - seg_begin(n, 1, G) + (s * G + g) * 34;
}

#ifndef ORLOJ_REPLAY_WARPS
#define ORLOJ_REPLAY_WARPS 4
#endif
constexpr int REPLAY_WARPS = ORLOJ_REPLAY_WARPS;  // warps (scenarios / segments) per CTA
// ORLOJ_REPLAY_STATS (diagnostic variant builds only): MODE 1 adds per-decision
// statistics to the workspace head: [5] decisions committed by the max-plus
// run path, [6] scanned decisions with a carried window, [7 + wc] windows of
// wc members after the scan (wc = 0..24, 24 = 24 or more).
#ifdef ORLOJ_REPLAY_STATS
#define ORLOJ_STAT(i, v) do { if (MODE == 1 && lane == 0) atomicAdd(p.seg_stats + (i), (unsigned long long)(v)); } while (0)
#else
#define ORLOJ_STAT(i, v) do { } while (0)
#endif
#ifndef ORLOJ_REPLAY_KB
#define ORLOJ_REPLAY_KB 2
#endif
constexpr int REPLAY_KB = ORLOJ_REPLAY_KB;  // candidate sizes per scoring block (windows are short: ~2-4)
#ifndef ORLOJ_PAIR_MAX
#define ORLOJ_PAIR_MAX 7
#endif
constexpr int PAIR_MAX = ORLOJ_PAIR_MAX;  // windows up to this size take the pair-lane path (<= 7: 28 pairs)
static_assert(PAIR_MAX >= 1 && PAIR_MAX <= 7, "pair lanes: k (k + 1) / 2 <= 32");

// Per-warp shared memory: REPLAY_KB staging rows, the window's member fields
// and the P[k][r] matrix (row stride 36 floats: conflict-free 128-bit reads).
// RATE (finish-rate objective) adds the S[k][lane] matrix of per-lane partial
// sums of G_k over the bins, for E[L_{B_k}].
template <int BPL, bool RATE = false>
struct ReplayWarpSmem {
  static constexpr int STG = 32 * BPL + 4;
  static constexpr int PSTRIDE = 36;
  static constexpr size_t BYTES = (size_t)(REPLAY_KB * STG) * 4 + 32 * (8 + 8 + 4 + 4 + 4) +
                                  (RATE ? 2 : 1) * 32 * PSTRIDE * 4 + 16;  // + segment-run state (MODE 1)
  __host__ __device__ static constexpr size_t bytes() { return BYTES; }
};

// CTA shared memory: store [D][B] floats, hopeless thresholds [D] int64 (padded), warps.
__host__ __device__ inline size_t replay_head_bytes(int D, int B) {
  return (((size_t)D * B * 4 + 15) & ~(size_t)15) + (size_t)((D + 1) & ~1) * 8 + 32 * 2 * 16;
}

#ifndef ORLOJ_REPLAY_MIN_BLOCKS
#define ORLOJ_REPLAY_MIN_BLOCKS 8
#endif

// MODE 0: plain replay, one warp per scenario.  MODE 1: speculative segments,
// one warp per (scenario, segment).  MODE 2: stitch, one warp per scenario.
template <int BPL, bool RATE, bool ALG1 = false, int MODE = 0>
__global__ void __launch_bounds__(REPLAY_WARPS * 32, MODE == 2 ? 2 : ORLOJ_REPLAY_MIN_BLOCKS)
replay_kernel(const __grid_constant__ ReplayParams p) {
  constexpr int STG = ReplayWarpSmem<BPL, RATE>::STG;
  constexpr int PST = ReplayWarpSmem<BPL, RATE>::PSTRIDE;

  extern __shared__ __align__(16) float s_dyn[];
  const int D = p.D, B = p.B;
  float *s_store = s_dyn;                                                   // [D][B]
  int64_t *s_thr = reinterpret_cast<int64_t *>(s_store + (size_t)D * B);   // [D]: a_1 + w_1 m_min(d)
  int4 *s_pair = reinterpret_cast<int4 *>(s_thr + ((D + 1) & ~1));          // [32][2] pair-lane table
  char *s_warp = reinterpret_cast<char *>(s_dyn) + replay_head_bytes(D, B);
  const int lane = (int)opaque_u32(threadIdx.x & 31);  // pinned: not re-read from SR_TID in the loop
  const int wid = threadIdx.x >> 5;
  char *my = s_warp + wid * ReplayWarpSmem<BPL, RATE>::bytes();
  float *stg_p = reinterpret_cast<float *>(my) + 4;                          // REPLAY_KB rows, stride STG
  // the loop addresses shared memory through 32-bit shared-space arrays (common.cuh SArr)
  const uint32_t sb = smem_base(s_dyn);
  const uint32_t mb0 =
      opaque_u32(sb + (uint32_t)replay_head_bytes(D, B) + (uint32_t)wid * (uint32_t)ReplayWarpSmem<BPL, RATE>::bytes());
  const SArr<float> sto{sb};                                                 // store [D][B]
  const SArr<int64_t> thr{opaque_u32(sb + (uint32_t)D * B * 4)};             // [D]: a_1 + w_1 m_min(d)
  const uint32_t a_pair = opaque_u32(thr.a + (uint32_t)((D + 1) & ~1) * 8);  // [32][2] int4
  const SArr<float> stg{mb0 + 16};                                            // REPLAY_KB rows, stride STG
  const uint32_t a_win = mb0 + REPLAY_KB * STG * 4;
  const SArr<int64_t> w_dl{a_win};               // window deadlines
  const SArr<int64_t> w_h{a_win + 256};          // window hopeless times
  const SArr<int32_t> w_d{a_win + 512};          // window distributions
  const SArr<int32_t> w_tb{a_win + 640};         // window true bins
  const SArr<int32_t> w_ix{a_win + 768};         // window arrival indices (MODE 0 with per-arrival outcomes)
  const SArr<float> Pm{a_win + 896};             // P[k-1][r], stride PST
  const SArr<float> Sm{a_win + 896 + 32 * PST * 4};  // RATE only: per-lane partial sum_{i<B} G_k(tau_i), [k-1][lane]
  // MODE 1 (cold, warp-uniform; kept out of registers): base arrival of the
  // current record list, records in it, extension flag
  const SArr<int64_t> sm_mark_base{a_win + 896 + (RATE ? 2 : 1) * 32 * PST * 4};
  const SArr<int32_t> sm_nrec{a_win + 896 + (RATE ? 2 : 1) * 32 * PST * 4 + 8};
  const SArr<int32_t> sm_ext{a_win + 896 + (RATE ? 2 : 1) * 32 * PST * 4 + 12};

  // Pair lanes for windows of 2..PAIR_MAX members (most scored windows): lane p
  // scores candidate size pk and member pr, p = pk (pk - 1) / 2 + pr - 1, with
  // size pk's lookup constants; as a gatherer, lane k-1 sums the pair lanes
  // pk (pk - 1) / 2 + [0, k) of its size.  [lane][0] = {pk, pr - 1, gather base},
  // [lane][1] = lookup constants of pk (kept in shared memory, not registers).
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    int k = 1;
    while (k * (k + 1) / 2 <= l) ++k;  // lanes >= 28: k = 8 (idle)
    s_pair[2 * l] = make_int4(k, l - k * (k - 1) / 2, l * (l + 1) / 2, 0);
    s_pair[2 * l + 1] = k <= p.prof.kmax ? make_int4(p.prof.a2[k - 1], p.prof.wB2[k - 1], (int)p.prof.mag[k - 1],
                                                     (int)p.prof.sh[k - 1])
                                         : make_int4(0, 0, 0, 0);
  }
  // stage the (small) store; hopeless threshold a_1 + w_1 m_min(d) per distribution
  for (int e = threadIdx.x; e < D * B; e += blockDim.x) s_store[e] = p.log2F[e];
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    int m = B;
    for (int i = B - 1; i >= 0; --i)
      if (s_store[d * B + i] != -INFINITY) m = i + 1;
    s_thr[d] = ALG1 ? p.size_thr[0]  // Alg. 1 l.10-13: infeasible for every bs iff infeasible for bs = 1
                    : p.drop_thr ? p.drop_thr[d] : (int64_t)p.prof.a[0] + (int64_t)p.prof.w[0] * m;
  }
  if (lane < REPLAY_KB) stg_p[lane * STG - 1] = -INFINITY;
  __syncthreads();

  if constexpr (MODE != 0) {
    // the scratch logs are sized from the caller's num_arrivals: a trace with
    // more arrivals would write past them — refuse the whole call, flag it
    if (p.arr_off[p.S] - p.arr_off[0] > p.num_arrivals) {
      if (blockIdx.x == 0 && threadIdx.x == 0) p.seg_stats[4] = 1;
      return;
    }
  }
  const int64_t u = (int64_t)blockIdx.x * REPLAY_WARPS + wid;
  int64_t s = u;
  int g = 0;  // MODE 1: this warp's segment; MODE 2: the segment being stitched
  if constexpr (MODE == 1) {
    if (u >= p.S * p.G) return;
    g = (int)(u / p.S);  // segment-major items: a block's warps replay the same segment of 4 scenarios
    s = u - (int64_t)g * p.S;
  } else {
    if (s >= p.S) return;
  }

  const int kmax = p.prof.kmax;
  int64_t base = p.arr_off[s];
  int64_t n = p.arr_off[s + 1] - base;
  uint8_t *oc = nullptr;  // MODE 0: per-arrival outcomes (indexed like arr / dis / tbs)
  if constexpr (MODE == 0) {
    if (p.num_epochs > 1) {  // epoch e: arrivals [s_e, s_{e+1}) of the scenario
      const int64_t b0 = seg_begin(n, p.epoch, p.num_epochs);
      base += b0;
      n = seg_begin(n, p.epoch + 1, p.num_epochs) - b0;
    }
    if (p.outcome) oc = p.outcome + base;
  }
  // per-scenario indices and counts are 32-bit (include/orloj.h: a scenario
  // holds fewer than 2^31 - 64 arrivals; a violated precondition is a fault)
  if (n > 0x7fffffbfll) __trap();
  const int32_t ni = (int32_t)n;
  const int64_t slo = p.slo[s];
  const int64_t *arr = p.arrival + base;
  const int32_t *dis = p.dist + base;
  const int16_t *tbs = p.true_bin + base;
  // RATE: lane k-1 evaluates E[L_{B_k}] with a_k, w_k of its own candidate size
  const float my_a = RATE ? (float)p.prof.a[lane] : 0.f;
  const float my_w = RATE ? (float)p.prof.w[lane] : 0.f;
  // ALG1: lane bs-1 holds thr_bs and the lookup constants of size bs
  const int64_t my_thr = (ALG1 && lane < kmax) ? p.size_thr[lane] : INT64_MAX;
  const int4 my_lk = (ALG1 && lane < kmax) ? make_int4(p.prof.a2[lane], p.prof.wB2[lane], (int)p.prof.mag[lane],
                                                       (int)p.prof.sh[lane])
                                           : make_int4(0, 0, 0, 0);
  const int32_t my_wk = (ALG1 && lane < kmax) ? p.prof.w[lane] : 0;
  const int32_t my_ak = (ALG1 && lane < kmax) ? p.prof.a[lane] : 0;

  int64_t t = INT64_MIN;
  if constexpr (MODE == 0)
    if (p.t_carry) t = p.t_carry[s];  // the worker is busy until then (INT64_MIN: free)
  int32_t cursor = 0;
  int32_t seg_end = INT32_MAX;  // MODE 1: stop (s_{g+1}, then the extension cap); MODE 2: s_{g+1} of the stitched g
  int32_t rec_at = INT32_MAX;  // MODE 1: record the first regeneration point at or past this arrival
  ReplaySeg *sg = nullptr;               // MODE 1: this segment; MODE 2: the scenario's segments
  int32_t *mylog = p.log ? p.log + base + s : nullptr;
  if constexpr (MODE == 1) {
    cursor = (int32_t)seg_begin(n, g, p.G);
    if (g > 0) rec_at = cursor;  // segment 0's records are never matched
    if (lane == 0) {
      sm_mark_base.st(0, cursor);
      sm_nrec.st(0, 0);
      sm_ext.st(0, 0);
    }
    __syncwarp();
    if (g + 1 < p.G) seg_end = (int32_t)seg_begin(n, g + 1, p.G);
    sg = opaque_ptr(p.seg + s * p.G + g);  // used only in the (cold) segment hooks
#ifdef ORLOJ_REPLAY_TIMELINE
    if (lane == 0) {
      sg->tl[0] = tl_now();
      sg->tl_sm[0] = tl_smid();
    }
#endif
    if (g > 0) mylog = p.seg_log ? p.seg_log + seg_log_off(base, s, n, g, p.G) : nullptr;
  }
  // window slots start as valid entries (distribution 0, bin 1): the scoring
  // reads every lane's slot and masks the non-members afterwards
  w_dl.st(lane, 0);
  w_h.st(lane, 0);
  w_d.st(lane, 0);
  w_tb.st(lane, 1);
  __syncwarp();
  // lookahead: lane l holds arrivals[cursor + l] (arrival INT64_MAX beyond the trace)
  int64_t ua = INT64_MAX;
  int ud = 0, ut = 0;
  auto reload = [&]() {
    const int32_t idx = cursor + lane;
    ua = INT64_MAX;
    if (idx < ni) {
      ua = arr[idx];
      ud = dis[idx];
      ut = tbs[idx];
    }
  };
  reload();
  int ncarry = 0, carry_off = 0;
  uint32_t c_fin = 0, c_drop = 0, c_late = 0, c_bat = 0;  // < 2^32: counts within one scenario
  long long c_busy = 0;
  int32_t ndec = 0;
  int nrec = 0;  // MODE 1: records in the current list; MODE 2: match pointer into segment g's records
  int64_t taken = 0;  // MODE 2: decisions taken over from segment runs (the rest were re-run here)
  int joined = 0, crossed = 0;

  // MODE 1: end state of the segment run
  auto save_end = [&]() {
    if (lane < ncarry) {
      sg->carry_D[lane] = w_dl.ld(carry_off + lane);
      sg->carry_h[lane] = w_h.ld(carry_off + lane);
      sg->carry_d[lane] = w_d.ld(carry_off + lane);
      sg->carry_tb[lane] = w_tb.ld(carry_off + lane);
    }
    if (lane == 0) {
      sg->t = t;
      sg->cursor = cursor;
      sg->ndec = ndec;
      sg->ctr[0] = c_fin;
      sg->ctr[1] = c_drop;
      sg->ctr[2] = c_late;
      sg->ctr[3] = c_bat;
      sg->ctr[4] = c_busy;
      sg->ncarry = ncarry;
      sg->nrec = nrec;
    }
  };
  // MODE 2: decision log of segment gg's run (segment 0 wrote the true log)
  auto seg_src_log = [&](int gg) -> const int32_t * {
    return gg == 0 ? p.log + base + s : p.seg_log + seg_log_off(base, s, n, gg, p.G);
  };
  // MODE 2: append segment gg's decisions [from, to) and its counters between two of its points
  auto take = [&](int gg, long long from, long long to, const long long *c0, const long long *c1) {
    if (mylog) {
      const int32_t *src = seg_src_log(gg);
      for (long long i = from + lane; i < to; i += 32) mylog[ndec + i - from] = src[i];
    }
    c_fin += (uint32_t)(c1[0] - c0[0]);
    c_drop += (uint32_t)(c1[1] - c0[1]);
    c_late += (uint32_t)(c1[2] - c0[2]);
    c_bat += (uint32_t)(c1[3] - c0[3]);
    c_busy += c1[4] - c0[4];
    ndec += (int32_t)(to - from);
    taken += to - from;
  };
  // MODE 2: load segment gg's end state into the registers / window (the true state)
  auto materialize = [&](const ReplaySeg *e) {
    t = e->t;
    cursor = (int32_t)e->cursor;
    ncarry = e->ncarry;
    carry_off = 0;
    __syncwarp();
    if (lane < ncarry) {
      w_dl.st(lane, e->carry_D[lane]);
      w_h.st(lane, e->carry_h[lane]);
      w_d.st(lane, e->carry_d[lane]);
      w_tb.st(lane, e->carry_tb[lane]);
    }
    __syncwarp();
    reload();
  };
  // MODE 2: the true run is at segment g-1's end state (not loaded): while the
  // extension of segment g-1 and the records of segment g share a regeneration
  // point, the true run is segment g-1's extension up to it and segment g's run
  // from it — join without re-running anything.  Returns true once the last
  // segment is joined (the true run ends at its end state).
  auto lazy_walk = [&]() -> bool {
    while (g < p.G) {
      const ReplaySeg *pe = sg + g - 1, *e = sg + g;
      const int ne = pe->next, nr = e->nrec;
      const long long ja = lane < ne ? pe->ext[lane].j : -1;
      const long long jb = lane < nr ? e->rec[lane].j : -2;
      int hit = -1;
      for (int b2 = 0; b2 < nr; ++b2) {
        const long long x = __shfl_sync(FULL, jb, b2);
        if (x == ja && hit < 0) hit = b2;
      }
      const unsigned hm = __ballot_sync(FULL, hit >= 0);
      if (hm == 0) return false;
      const int ia = __ffs(hm) - 1;  // lists increase: the first common point
      const int ib = __shfl_sync(FULL, hit, ia);
      take(g - 1, pe->ndec, pe->ext[ia].ndec, pe->ctr, pe->ext[ia].ctr);
      take(g, e->rec[ib].ndec, e->ndec, e->rec[ib].ctr, e->ctr);
      ++joined;
      ++g;
    }
    return true;
  };
  if constexpr (MODE == 2) {
    // segment 0 ran from the true start: the true run is at its end state
    sg = opaque_ptr(p.seg + s * p.G);
#ifdef ORLOJ_REPLAY_TIMELINE
    if (lane == 0) {
      sg->tl[2] = tl_now();
      sg->tl_sm[1] = tl_smid();
    }
#endif
    ndec = (int32_t)sg[0].ndec;  // segment 0 wrote its decisions into the true log
    taken = ndec;
    c_fin = (uint32_t)sg[0].ctr[0];
    c_drop = (uint32_t)sg[0].ctr[1];
    c_late = (uint32_t)sg[0].ctr[2];
    c_bat = (uint32_t)sg[0].ctr[3];
    c_busy = sg[0].ctr[4];
    g = 1;
    if (lazy_walk()) {  // joined everything: the true run ends at the last segment's end state
      t = sg[p.G - 1].t;
      cursor = ni;
    } else {
      materialize(sg + g - 1);
      seg_end = g + 1 < p.G ? (int32_t)seg_begin(n, g + 1, p.G) : INT32_MAX;
    }
  }

  // consume m (< 32) arrivals from the lookahead: shift by m lanes, refill the
  // tail from HBM (used from the next decision on)
  auto advance = [&](int m) {
    cursor += m;
    const int src = (lane + m) & 31;
    const int64_t sa = __shfl_sync(FULL, ua, src);
    const int sd = __shfl_sync(FULL, ud, src);
    const int st = __shfl_sync(FULL, ut, src);
    if (lane + m < 32) {
      ua = sa;
      ud = sd;
      ut = st;
    } else {
      const int32_t idx = cursor + lane;
      ua = INT64_MAX;
      if (idx < ni) {
        ua = arr[idx];
        ud = dis[idx];
        ut = tbs[idx];
      }
    }
  };
  const int64_t a1 = p.prof.a[0], w1 = p.prof.w[0];
  // the max-plus scan runs on 32-bit offsets from the first lookahead arrival
  // when 32 batch durations (each <= a_1 + w_1 B) and the lookahead's arrival
  // offsets stay below 2^29 (exact: every value below 2^30 + 2^29, no wrap)
  const bool scan32 = 32 * (a1 + w1 * (int64_t)B) < (1ll << 29);

  while (cursor < ni || ncarry > 0) {
    if constexpr (MODE == 1) {
      if (cursor >= seg_end) {  // first loop top past the segment: its end state, then the extension
        if (sm_ext.ld(0)) break;
        nrec = sm_nrec.ld(0);
        save_end();
        rec_at = seg_end;
        __syncwarp();
        if (lane == 0) {
          sm_ext.st(0, 1);
          sm_mark_base.st(0, seg_end);
          sm_nrec.st(0, 0);
        }
        __syncwarp();
        seg_end = (int32_t)seg_begin(n, g + 2, p.G);
        // every extension iteration starts below s_{g+2}, which bounds the
        // scratch log (seg_log_off); a run already past it has no extension
        if (cursor >= seg_end) break;
      }
      if (cursor >= rec_at && ncarry == 0) {
        const int64_t a0 = __shfl_sync(FULL, ua, 0);
        if (a0 != INT64_MAX && t <= a0) {  // regeneration point at arrival `cursor`: record it
          const int nr = sm_nrec.ld(0);
          const bool ext = sm_ext.ld(0);
          const int64_t mb = sm_mark_base.ld(0);
          const long long v = lane == 0 ? cursor : lane == 1 ? ndec : lane == 2 ? c_fin : lane == 3 ? c_drop
                              : lane == 4 ? c_late : lane == 5 ? c_bat : c_busy;
          if (lane < 7) reinterpret_cast<long long *>(ext ? &sg->ext[nr] : &sg->rec[nr])[lane] = v;
          int64_t m = rec_at - mb;
          while (m <= cursor - mb) m = seg_next_mark(m);
          rec_at = nr + 1 < SEG_REC && mb + m < INT32_MAX ? (int32_t)(mb + m) : INT32_MAX;
          __syncwarp();
          if (lane == 0) sm_nrec.st(0, nr + 1);
          __syncwarp();
          if (ext && nr + 1 > SEG_EXT_AFTER) break;
        }
      }
    }
    if constexpr (MODE == 2) {
      if (cursor >= seg_end) {  // the true run crossed segment g without meeting it: next segment
        ++crossed;
        ++g;
        nrec = 0;
        seg_end = g + 1 < p.G ? (int32_t)seg_begin(n, g + 1, p.G) : INT32_MAX;
        continue;
      }
      if (g < p.G && ncarry == 0) {
        const int64_t a0 = __shfl_sync(FULL, ua, 0);
        if (a0 != INT64_MAX && t <= a0) {  // true run regenerates at arrival `cursor`
          const ReplaySeg *e = sg + g;
          const int nr = e->nrec;
          while (nrec < nr && e->rec[nrec].j < cursor) ++nrec;
          if (nrec < nr && e->rec[nrec].j == cursor) {  // segment g regenerated here too: same run from now on
            take(g, e->rec[nrec].ndec, e->ndec, e->rec[nrec].ctr, e->ctr);
            ++joined;
            ++g;
            nrec = 0;
            if (lazy_walk()) {
              t = sg[p.G - 1].t;
              break;
            }
            materialize(sg + g - 1);
            seg_end = g + 1 < p.G ? (int32_t)seg_begin(n, g + 1, p.G) : INT32_MAX;
            continue;
          }
        }
      }
    }
    // ---- 0. runs of single-member windows (max-plus scan) -----------------
    // With nothing carried, arrival j of the lookahead is a window of one iff
    // it is not hopeless at its decision time t'_j = max(T_{j-1}, a_j) and the
    // next arrival comes later (a_{j+1} > t'_j); its batch then ends at
    // T_j = t'_j + d_j, d_j = a_1 + w_1 bin_j.  T_j = g_j(T_{j-1}) with
    // g_j(x) = max(x + d_j, a_j + d_j): maps (P, Q): x -> max(x + P, Q) compose
    // associatively, (P, Q) then (P', Q') = (P + P', max(Q + P', Q')), so a
    // warp scan yields up to 31 consecutive decisions at once; the leading run
    // of lanes meeting both conditions is committed, exactly as the sequential
    // loop would (window of one: k* = 1, no scoring).
    if (ncarry == 0) {
      const bool va = ua != INT64_MAX;
      const int64_t hj = va ? ua + slo - thr.ld(ud) : INT64_MIN;
      const int64_t an = __shfl_down_sync(FULL, ua, 1);
      // lane 0 decides for arrival `cursor` (its own registers: no broadcasts), one ballot
      const int64_t t0 = ua > t ? ua : t;
      const bool ok0 = __ballot_sync(FULL, lane == 0 && va && an > t0 && t0 <= hj) != 0u;
      if (ok0) {  // warp-uniform
        const int64_t dj = a1 + w1 * ut;
        int64_t P, Qv;
        const int64_t base = __shfl_sync(FULL, ua, 0);  // lane 0 is a real arrival (ok0)
        if (scan32 && __all_sync(FULL, !va || ua - base < (1ll << 29))) {
          // the same scan on 32-bit offsets (values equal to the 64-bit scan's)
          int32_t P32 = va ? (int32_t)dj : 0, Q32 = va ? (int32_t)(ua - base) + (int32_t)dj : INT32_MIN;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int32_t Pp = __shfl_up_sync(FULL, P32, off);
            const int32_t Qp = __shfl_up_sync(FULL, Q32, off);
            if (lane >= off) {
              Q32 = max(Qp + P32, Q32);
              P32 += Pp;
            }
          }
          P = P32;
          Qv = base + Q32;  // >= base + Q of lane 0: a real value in every lane
        } else {
          P = va ? dj : 0;
          Qv = va ? ua + dj : INT64_MIN;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int64_t Pp = __shfl_up_sync(FULL, P, off);
            const int64_t Qp = __shfl_up_sync(FULL, Qv, off);
            if (lane >= off) {
              const int64_t q2 = Qp + P;
              Qv = q2 > Qv ? q2 : Qv;
              P += Pp;
            }
          }
        }
        const int64_t Tj = t + P > Qv ? t + P : Qv;  // t may be INT64_MIN: t + P does not overflow
        const int64_t tpj = Tj - dj;
        const bool ok = lane < 31 && va && an > tpj && tpj <= hj;
        const int m = __ffs(~__ballot_sync(FULL, ok)) - 1;  // >= 1 (lane 0 passed ok0)
        const unsigned fm = __ballot_sync(FULL, lane < m && Tj <= ua + slo);
        if (oc && lane < m) oc[cursor + lane] = ((fm >> lane) & 1u) ? 1 : 2;
        c_fin += __popc(fm);
        c_late += m - __popc(fm);
        c_bat += m;
        c_busy += __shfl_sync(FULL, P, m - 1);
        t = __shfl_sync(FULL, Tj, m - 1);
        if (mylog && lane < m) mylog[ndec + lane] = 1;
        ORLOJ_STAT(5, m);
        ndec += m;
        advance(m);
        continue;
      }
    }
    const int64_t next_arr = __shfl_sync(FULL, ua, 0);
    if (ncarry == 0 && next_arr > t) t = next_arr;  // idle worker: jump to the next arrival (A15)
    // ---- 1. scan -------------------------------------------------------
    int wc = 0;
    ORLOJ_STAT(6, ncarry > 0 ? 1 : 0);
    if (ncarry > 0) {
      const bool valid = lane < ncarry;
      int64_t Dr = 0, hr = 0;
      int dr = 0, tr = 0, ir = 0;
      if (valid) {
        Dr = w_dl.ld(carry_off + lane);
        hr = w_h.ld(carry_off + lane);
        dr = w_d.ld(carry_off + lane);
        tr = w_tb.ld(carry_off + lane);
        if (oc) ir = w_ix.ld(carry_off + lane);
      }
      const bool keep = valid && t <= hr;
      const unsigned vm = __ballot_sync(FULL, valid);
      const unsigned km = __ballot_sync(FULL, keep);
      c_drop += __popc(vm & ~km);
      if (oc && valid && !keep) oc[ir] = 3;
      __syncwarp();
      if (keep) {
        const int slot = __popc(km & ((1u << lane) - 1u));
        w_dl.st(slot, Dr);
        w_h.st(slot, hr);
        w_d.st(slot, dr);
        w_tb.st(slot, tr);
        if (oc) w_ix.st(slot, ir);
      }
      wc = __popc(km);
    }
    while (wc < kmax) {
      const bool valid = ua <= t;  // arrivals are sorted: valid lanes form a prefix
      const unsigned vm = __ballot_sync(FULL, valid);
      if (vm == 0) break;
      const int64_t uh = ua + slo - thr.ld(ud);  // hopeless time (computed here: refilled lanes' loads
      const bool keep = valid && t <= uh;        // are never consumed in the decision that issued them)
      const unsigned km = __ballot_sync(FULL, keep);
      const int need = kmax - wc;
      unsigned consumed = vm;
      if (__popc(km) >= need) {
        // lane of the need-th kept member: its inclusive kept-rank equals need
        const unsigned le = (lane == 31) ? FULL : ((1u << (lane + 1)) - 1u);
        const unsigned at = __ballot_sync(FULL, keep && __popc(km & le) == need);
        const int pos = __ffs(at) - 1;
        consumed = pos == 31 ? FULL : ((1u << (pos + 1)) - 1u);
      }
      const unsigned kc = km & consumed;
      c_drop += __popc(vm & consumed & ~km);
      if (oc && ((vm & consumed & ~km) >> lane) & 1u) oc[cursor + lane] = 3;
      if ((kc >> lane) & 1u) {
        const int slot = wc + __popc(kc & ((1u << lane) - 1u));
        w_dl.st(slot, ua + slo);
        w_h.st(slot, uh);
        w_d.st(slot, ud);
        w_tb.st(slot, ut);
        if (oc) w_ix.st(slot, (int32_t)(cursor + lane));
      }
      wc += __popc(kc);
      const int nc = __popc(consumed);
      if (nc == 32) {  // whole lookahead consumed: reload all of it, scan on
        cursor += 32;
        const int32_t idx = cursor + lane;
        ua = INT64_MAX;
        if (idx < ni) {
          ua = arr[idx];
          ud = dis[idx];
          ut = tbs[idx];
        }
        continue;
      }
      advance(nc);
      break;
    }
    ncarry = 0;
    carry_off = 0;
    wc = warp_uniform(wc);
    ORLOJ_STAT(7 + (wc < 24 ? wc : 24), 1);
    __syncwarp();
    if (wc == 0) continue;

    // ---- 2. score the window ---------------------------------------------
    // window fields of every lane (slots >= wc hold stale entries: each use below
    // is masked by mem / sel or indexes members only)
    const bool mem = lane < wc;
    const int64_t Dr = w_dl.ld(lane);
    const int32_t sig = sigma2(Dr - t);
    const int dr = w_d.ld(lane);
    const int tb = w_tb.ld(lane);

    int kstar = 1;  // a window of one has a single candidate: no scoring needed
    uint32_t selm = 1u;  // ALG1: the popped members (window positions)
    if (ALG1 && wc > 1) {  // warp-uniform
      // Alg. 1 l.14-20: Q_bs = {r : t + E[L_bs] <= D_r} is a suffix of
      // the deadline-ordered window; lane bs-1 finds its first member by binary search
      int lo = 0, hi = wc;
      const int64_t need = my_thr == INT64_MAX ? INT64_MAX : t + my_thr;  // beyond kmax: never feasible
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (w_dl.ld(mid) < need || my_thr == INT64_MAX) lo = mid + 1;
        else hi = mid;
      }
      const bool feas = lane < kmax && wc - lo >= lane + 1;  // |Q_bs| >= bs
      // candidate: earliest D_{Q_bs}, ties -> larger bs (SURVEY A/Design reading of P:296-297)
      const uint64_t dq = feas ? (uint64_t)(w_dl.ld(lo) - t) : ~0ull;  // >= 0 when feasible
      const uint32_t mh = __reduce_min_sync(FULL, (uint32_t)(dq >> 32));
      const uint32_t ml = __reduce_min_sync(FULL, (uint32_t)(dq >> 32) == mh ? (uint32_t)dq : 0xffffffffu);
      kstar = (int)__reduce_max_sync(FULL, (feas && dq == (((uint64_t)mh << 32) | ml)) ? (uint32_t)(lane + 1) : 0u);
      const int first = __shfl_sync(FULL, lo, kstar - 1);
      // PopBatch(Q_kstar): the kstar highest Eq. 1-2 priorities, ties -> earlier member
      const int4 lk = make_int4(__shfl_sync(FULL, my_lk.x, kstar - 1), __shfl_sync(FULL, my_lk.y, kstar - 1),
                                __shfl_sync(FULL, my_lk.z, kstar - 1), __shfl_sync(FULL, my_lk.w, kstar - 1));
      const int32_t wk = __shfl_sync(FULL, my_wk, kstar - 1);
      const bool inq = mem && lane >= first;
      uint32_t key = 0u;
      if (inq) {
        const double *tab = p.prio_table + (size_t)(kstar - 1) * 2 * (B + 1);
        const float lp = prio_elem_global(tab, p.prio_logEL[kstar - 1], B, lk, wk, sig, -p.prio_b * (double)(Dr - t),
                                          (float)p.prio_b);
        key = lp != lp ? 1u : fkey(lp == 0.0f ? 0.0f : lp);  // p = 0 (-inf) stays poppable: fkey(-inf) > 0
      }
      int rank = 0;
      for (int j = 0; j < wc; ++j) {
        const uint32_t kj = __shfl_sync(FULL, key, j);
        rank += (kj > key || (kj == key && j < lane)) ? 1 : 0;
      }
      selm = __ballot_sync(FULL, inq && rank < kstar);
    }
    if (!ALG1 && wc > 1) {   // warp-uniform
    float E = 0.f;
    if (!RATE && wc <= PAIR_MAX) {
      // ---- 2'. small window: lanes over (k, r) pairs -----------------------
      // LG_k at the pair's own lookup bin, summed over members j <= k in the
      // block path's order (0 + x_1 + ... + x_k), then 2^LG (0 at bin 0) — the
      // same fp32 values as the block path, and E_k from the same adder tree.
      const int4 pq = lds_v4s32(a_pair + 32u * lane), plk = lds_v4s32(a_pair + 32u * lane + 16u);
      const int pk = pq.x;
      const int sr = __shfl_sync(FULL, sig, pq.y);
      const int bi = lookup_bin(sr, plk.x, plk.y, (uint32_t)plk.z, (uint32_t)plk.w);
      const int bo = bi > 0 ? bi - 1 : 0;
      float lgp = 0.f;
#pragma unroll
      for (int j = 0; j < PAIR_MAX; ++j) {
        if (j >= wc) break;  // warp-uniform
        const float x = sto.ld(__shfl_sync(FULL, dr, j) * B + bo);
        if (j < pk) lgp += x;
      }
      const float pv = (bi > 0 && pk <= wc) ? ex2_approx(lgp) : 0.f;
      // gather through shared memory (the P matrix area, [k-1][8]): pair lane
      // (k, r) writes P_r(k) to slot (k-1) 8 + r and a zero to the mirrored
      // slot (7-k) 8 + 7-r, which no pair owns (r' = 7 - r >= k' = 8 - k): all
      // 56 slots are rewritten every time, and lane k-1 reads its 8 as quads
      if (lane < 28) {
        Pm.st((pk - 1) * 8 + pq.y, pv);
        Pm.st((7 - pk) * 8 + 7 - pq.y, 0.f);
      }
      __syncwarp();
      float x[8];
      Pm.ldv<4>(8 * lane, *reinterpret_cast<float(*)[4]>(x));
      if (wc > 4) Pm.ldv<4>(8 * lane + 4, *reinterpret_cast<float(*)[4]>(x + 4));  // warp-uniform
      else x[4] = x[5] = x[6] = x[7] = 0.f;
      const float acc0 = (x[0] + x[1]) + (x[2] + x[3]);
      E = wc <= 4 ? acc0 : acc0 + ((x[4] + x[5]) + (x[6] + x[7]));
    } else {
    float lg[BPL];
#pragma unroll
    for (int b = 0; b < BPL; ++b) lg[b] = 0.f;
    const bool vok = lane * BPL < B;
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += REPLAY_KB) {  // unrolled: profile entries are immediate constants
      if (k0 >= wc) break;                        // warp-uniform
      if (k0 > 0) __syncwarp();                   // previous block's gathers are done
#pragma unroll
      for (int i = 0; i < REPLAY_KB; ++i) {
        const int d = __shfl_sync(FULL, dr, (k0 + i) & 31);  // beyond wc: harmless id 0
        if (vok) {
          float x[BPL];
          sto.ldv<BPL>(d * B + lane * BPL, x);
#pragma unroll
          for (int e = 0; e < BPL; ++e) lg[e] += x[e];
        }
        stg.stv<BPL>(i * STG + lane * BPL, lg);
        if constexpr (RATE) {
          // this lane's share of sum_{i<B} G_k(tau_i) (bins tau_1 .. tau_{B-1})
          float part = 0.f;
#pragma unroll
          for (int e = 0; e < BPL; ++e)
            if (lane * BPL + e < B - 1) part += ex2_approx(lg[e]);
          Sm.st(((k0 + i) & 31) * PST + lane, part);
        }
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < REPLAY_KB; ++i) {
        const int kk = k0 + i;  // k - 1 (rows at or beyond wc are computed but never read)
        const int bi = lookup_bin(sig, p.prof.a2[kk], p.prof.wB2[kk], p.prof.mag[kk], p.prof.sh[kk]);
        const float pr = ex2_approx(stg.ld(i * STG + bi - 1));
        Pm.st((kk & 31) * PST + lane, lane <= kk ? pr : 0.f);
      }
    }
    __syncwarp();
    // E_k = sum_{r<k} P[k-1][r] in lane k-1: 128-bit row loads, adder tree
    if (mem) {
      const int nj = (wc + 3) >> 2;  // warp-uniform: quads holding members r < wc
      float acc[8];
      if (nj == 1) {  // windows of <= 4: the tree below reduces to its first quad, bit for bit
        float x[4];
        Pm.ldv<4>(lane * PST, x);
        acc[0] = (x[0] + x[1]) + (x[2] + x[3]);
        E = acc[0];
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[j] = 0.f;
          if (j < nj && 4 * j <= lane) {
            float x[4];
            Pm.ldv<4>(lane * PST + 4 * j, x);
            acc[j] = (x[0] + x[1]) + (x[2] + x[3]);
          }
        }
        E = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      }
      if constexpr (RATE) {
        // finish rate E_k / E[L_{B_k}], E[L_{B_k}] = a_k + w_k (B - sum_{i<B} G_k(tau_i))  (Eq. 5)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float x[4];
          Sm.ldv<4>(lane * PST + 4 * j, x);
          acc[j] = (x[0] + x[1]) + (x[2] + x[3]);
        }
        const float S = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        const float EL = my_a + my_w * ((float)B - S);
        E = E / EL;
      }
    }
    }  // block path
    // ---- 3. argmax + dispatch ----------------------------------------------
    const uint32_t mx = __reduce_max_sync(FULL, mem ? __float_as_uint(E) : 0u);
    kstar = (int)__reduce_min_sync(FULL, (mem && __float_as_uint(E) == mx) ? (uint32_t)lane : 32u) + 1;
    }
    const bool sel = ALG1 ? ((selm >> lane) & 1u) != 0u : lane < kstar;
    const int mbin = (int)__reduce_max_sync(FULL, sel ? (uint32_t)tb : 0u);
    const int64_t dur = ALG1 ? (int64_t)__shfl_sync(FULL, my_ak, kstar - 1) +
                                   (int64_t)__shfl_sync(FULL, my_wk, kstar - 1) * mbin
                             : (int64_t)p.prof.a[kstar - 1] + (int64_t)p.prof.w[kstar - 1] * mbin;
    const unsigned fm = __ballot_sync(FULL, sel && t + dur <= Dr);
    const int ix = (oc && mem) ? w_ix.ld(lane) : 0;
    if (oc && sel) oc[ix] = ((fm >> lane) & 1u) ? 1 : 2;
    c_fin += __popc(fm);
    c_late += kstar - __popc(fm);
    c_bat += 1;
    c_busy += dur;
    t += dur;
    if (mylog && lane == 0) mylog[ndec] = ALG1 ? (int32_t)selm : kstar;
    ++ndec;
    ncarry = wc - kstar;
    carry_off = kstar;
    if (ALG1 && ncarry > 0) {
      // the unpopped members stay pending in deadline order: compact in place
      const int64_t hr = mem ? w_h.ld(lane) : 0;
      const unsigned km = __ballot_sync(FULL, mem && !sel);
      __syncwarp();
      if (mem && !sel) {
        const int slot = __popc(km & ((1u << lane) - 1u));
        w_dl.st(slot, Dr);
        w_h.st(slot, hr);
        w_d.st(slot, dr);
        w_tb.st(slot, tb);
        if (oc) w_ix.st(slot, ix);
      }
      carry_off = 0;
    }
    __syncwarp();
  }
  if constexpr (MODE == 1) {
    const bool ext = sm_ext.ld(0);
    nrec = sm_nrec.ld(0);
    if (!ext) save_end();  // ended before s_{g+1} (last segment, or the trace ran out)
    if (lane == 0) {
      sg->next = ext ? nrec : 0;
      if (ext) atomicAdd(p.seg_stats + 3, (unsigned long long)(ndec - sg->ndec));
#ifdef ORLOJ_REPLAY_TIMELINE
      sg->tl[1] = tl_now();
#endif
    }
    return;
  }
  if constexpr (MODE == 2) {
    if (lane == 0) {
#ifdef ORLOJ_REPLAY_TIMELINE
      p.seg[s * p.G].tl[3] = tl_now();
#endif
      atomicAdd(p.seg_stats + 0, (unsigned long long)(ndec - taken));
      atomicAdd(p.seg_stats + 1, (unsigned long long)joined);
      atomicAdd(p.seg_stats + 2, (unsigned long long)crossed);
    }
  }
  if (lane == 0) {
    if (mylog) mylog[ndec] = 0;
    if constexpr (MODE == 0)
      if (p.t_carry) p.t_carry[s] = t;
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
