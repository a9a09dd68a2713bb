/*
 * orloj.h — C ABI of the B200-native Orloj batch-scoring library (liborloj.so).
 *
 * Orloj (arXiv 2209.00159) schedules batches of requests whose execution time
 * is a random variable known only through an empirical histogram per
 * application (PAPER.md:241-255 problem statement, :377-383 per-application
 * tracking).  This library evaluates, on the GPU and for very many independent
 * queues at once, the paper's batch execution-time model on every candidate
 * batch = every deadline-ordered prefix of a queue:
 *
 *   batch time     L_{B_k} = a_k + w_k * max_{j<=k} X_j          Eq. 3-4 (:479-491),
 *                                                                 Eq. 9 CDF form (:537-541)
 *   CDF of the max G_k(tau_i) = prod_{j<=k} F_{d_j}(tau_i)        Eq. 6 (:503-507), Eq. 8 (:512-535)
 *   finish prob.   P_r(k) = Pr(t + L_{B_k} <= D_r) = G_k(tau_{i*}) step SLO cost (:411-419)
 *                  i*(r,k) = clamp(floor((D_r - t - a_k) / w_k), 0, B)
 *   objective      E_k = sum_{r<=k} P_r(k), k* = smallest argmax  (:419-421)
 *   optional       E[L_{B_k}] = a_k + w_k * E[max bin]             Eq. 5 (:493-502)
 *
 * and replays request traces through the resulting decision rule (admit, drop
 * hopeless, pick, dispatch non-preemptively).
 *
 * Conventions (all entry points):
 *  - Every call returns an orloj_status; 0 = OK.  On failure, orloj_last_error()
 *    returns a thread-local message describing the last error on this thread.
 *  - Time is int64 "ticks" (1 tick = 1 us in the shipped workloads); only
 *    differences (D_r - t) enter the arithmetic, so absolute timestamps may be
 *    large (PAPER.md:612-623 overflow discussion).
 *  - Bins: a store has B bins, bin i (1..B) standing for tau_i = i * Delta, the
 *    upper bin edge (mass "discrete at upper edges", reading A1).
 *  - Buffers marked "device" are CUDA device pointers (e.g. torch CUDA tensor
 *    storage); "host" are host pointers ("pinned host" where the call copies
 *    asynchronously).  The caller owns every buffer.  The hot calls
 *    (score / pick / replay) never allocate, keep no global mutable state,
 *    and only enqueue work on `stream` (a cudaStream_t passed as void*; NULL =
 *    legacy default stream).  Calls on distinct streams are independent.
 *  - O(1) argument errors are detected and returned synchronously, before any
 *    work is enqueued.  Faults inside kernels surface as ORLOJ_ERR_CUDA at the
 *    next call or stream synchronisation (CUDA convention).  Expensive O(N)
 *    input checks live in orloj_validate_* (synchronous, not hot).
 */
#ifndef ORLOJ_H
#define ORLOJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORLOJ_ABI_VERSION 5  /* 5: orloj_score_model.plan, orloj_score_model_prepare */
#define ORLOJ_MAX_KMAX 256        /* candidate batch sizes per queue (score / pick) */
#define ORLOJ_MAX_BINS 256        /* bins per histogram (score / pick) */
#define ORLOJ_REPLAY_MAX_KMAX 32  /* window size in replay */
#define ORLOJ_REPLAY_MAX_BINS 128 /* bins per histogram in replay */

typedef enum {
  ORLOJ_OK = 0,
  ORLOJ_ERR_INVALID_ARGUMENT = 1, /* bad pointer / size / profile (non-monotone, w_k < 1, ...) */
  ORLOJ_ERR_COLD_START = 2,       /* a histogram has total count 0 */
  ORLOJ_ERR_UNSORTED = 3,         /* queue / trace order violated (validation only) */
  ORLOJ_ERR_CAPACITY = 4,         /* beyond built limits (kmax, B, 2^30-tick horizon, store size) */
  ORLOJ_ERR_CUDA = 5,             /* CUDA runtime / launch error */
  ORLOJ_ERR_OOM = 6               /* scratch allocation failed (validation / store build only) */
} orloj_status;

/* Thread-local message of the last failing call on this thread ("" if none). */
const char *orloj_last_error(void);

/* ORLOJ_ABI_VERSION of the loaded library. */
int32_t orloj_abi_version(void);

/* ---------------------------------------------------------------------------
 * Histogram / CDF store.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t num_dists;     /* D >= 1 */
  int32_t num_bins;      /* B: multiple of 4, 4 <= B <= ORLOJ_MAX_BINS */
  int64_t bin_ticks;     /* Delta > 0 (informational: kernels work in bin units via the profile) */
  const float *log2_cdf; /* device [D][B] row-major, 16-byte aligned:
                            element [d][i-1] = log2 F_d(tau_i) rounded to fp32 (RN);
                            -inf where F = 0; [d][B-1] == 0.0f exactly (F_d(tau_B) = 1). */
} orloj_store;

/* Build log2_cdf rows from integer counts: F_d(tau_i) = cum_i / total_d in fp64,
 * log2 in fp64, rounded once to fp32.  counts: device uint32 [D][B]; out: device
 * float [D][B] (caller-allocated, 16-byte aligned).  Rows may be built in chunks
 * by offsetting both pointers.  Synchronises `stream` (off the hot path: the
 * paper's profiler runs off the critical path) and may allocate
 * 4 bytes of scratch.  Errors: INVALID_ARGUMENT (sizes / alignment),
 * COLD_START (some row has total 0; rows already written are left as written),
 * CUDA, OOM. */
orloj_status orloj_store_build(const uint32_t *counts, int32_t num_dists, int32_t num_bins,
                               float *log2_cdf_out, void *stream);

/* Online profiler: accumulate sampled
 * solo execution times into the integer histogram counts a store is built
 * from.  Sample j (distribution dist_id[j], solo time solo_ticks[j] >= 0) adds
 * 1 to counts[d][i-1] with i = clamp(ceil(solo / bin_ticks), 1, B) — bin i
 * holds (tau_{i-1}, tau_i] ("discrete at upper edges", A1; longer times fold
 * into bin B).  counts: device uint32 [D][B], ADDED to (atomics); the window
 * reset of the paper is a memset of counts by the caller, followed by
 * orloj_store_build.  Async on `stream`.  Errors: INVALID_ARGUMENT (sizes,
 * bin_ticks <= 0), CUDA.  Samples with dist_id outside [0, D) are ignored. */
orloj_status orloj_histogram_accumulate(const int32_t *dist_id, const int64_t *solo_ticks, int64_t num_samples,
                                        int64_t bin_ticks, uint32_t *counts, int32_t num_dists, int32_t num_bins,
                                        void *stream);

/* ---------------------------------------------------------------------------
 * Latency profile: Eq. 3 generalised to a monotone integer table (A3).
 * A batch of k whose slowest member lies in bin m runs a_k + w_k * m ticks.
 * Eq. 3 (l_B = c0 + c1 k l) is the preset a_k = round(c0), w_k = round(c1 k Delta).
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t kmax;                 /* 1 <= kmax <= ORLOJ_MAX_KMAX (replay: <= ORLOJ_REPLAY_MAX_KMAX) */
  const int64_t *offset_ticks;  /* host [kmax]: a_k >= 0, non-decreasing in k */
  const int64_t *ticks_per_bin; /* host [kmax]: w_k >= 1, non-decreasing in k */
} orloj_latency_profile;
/* The table is copied into kernel parameters at each call (host pointers need
 * only be valid during the call).  Monotonicity (A14) is required
 * (INVALID_ARGUMENT otherwise): it makes P_r(k+1) <= P_r(k) hold bit-exactly.
 * Horizon: a_kmax + w_kmax * B must be <= 2^30 - 1 ticks (~17.9 min at 1 us
 * ticks; CAPACITY otherwise), so bin lookups run in exact 32-bit integer
 * arithmetic on doubled slacks. */

/* ---------------------------------------------------------------------------
 * Queues (release time, deadline = release + SLO, and an
 * execution-time distribution through the application id, :377-383).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t num_queues;            /* Q >= 0 */
  const int64_t *queue_offsets;  /* device [Q+1], CSR: queue q = members [off[q]-off[0], off[q+1]-off[0])
                                    of the member arrays (off[0] may be any base, e.g. a chunk of a
                                    larger queue set) */
  const int64_t *arrival_ticks;  /* device [N] release times, or NULL; read only by validation (tie order) */
  const int64_t *deadline_ticks; /* device [N]; per queue ordered by (deadline, arrival, index) (A9) */
  const int32_t *dist_id;        /* device [N], 0 <= dist_id < store.num_dists */
  const int64_t *now_ticks;      /* device [Q]: decision time t of each queue */
} orloj_queues;
/* score / pick take each queue as given: candidates are its first
 * K_q = min(n_q, kmax) members; hopeless members simply score P = 0. */

/* Score every candidate batch of every queue.
 *   expected_finish      device float [Q][kmax]: E_k at [q][k-1]; entries k > K_q are 0.
 *   finish_prob          device float [Q][kmax(kmax+1)/2] or NULL: P_r(k) at
 *                        [q][k(k-1)/2 + r], r = 0..k-1 (0-based member), k = 1..kmax;
 *                        entries with k > K_q are left untouched.
 *   expected_batch_ticks device float [Q][kmax] or NULL: E[L_{B_k}] (Eq. 5); 0 for k > K_q.
 * Accuracy: |P - P_exact| <= 1e-5, |E_k - E_exact| <= 1e-5 k.
 * Errors: INVALID_ARGUMENT, CAPACITY (B > 256, kmax > 256, horizon), CUDA. */
orloj_status orloj_score_batches(const orloj_store *store, const orloj_latency_profile *profile,
                                 const orloj_queues *queues, float *expected_finish,
                                 float *finish_prob, float *expected_batch_ticks, void *stream);

/* Pick the batch size of every queue: k* = argmax_k E_k,
 * ties -> smallest k (A10).  best_k: device int32 [Q] (0 iff the queue is
 * empty); best_expected: device float [Q] (E_{k*}; 0 for empty queues).
 * Same kernel as score_batches with a fused warp-reduction epilogue. */
orloj_status orloj_pick_batch(const orloj_store *store, const orloj_latency_profile *profile,
                              const orloj_queues *queues, int32_t *best_k, float *best_expected,
                              void *stream);

/* End-to-end variant of orloj_pick_batch for queues that live in (pinned) host
 * memory: enqueues H2D copies of the queue arrays into `workspace`, the pick
 * kernel and D2H copies of the results, all on `stream`; the caller
 * synchronises.  Host arrays must stay valid until the stream reaches the
 * copies.  queue_offsets_host follows the orloj_queues convention (any base),
 * so a caller can pipeline chunks of one queue set on several streams, each
 * with its own workspace, to overlap copies with compute.  workspace: device, >= orloj_pick_batch_host_workspace(Q, N) bytes,
 * 256-byte aligned.  Small calls ((Q+1)*8 + 12 N + 8 Q <= 64 KiB, e.g. one
 * scheduling decision) whose six host arrays are all pinned and mapped into the
 * device address space (cudaHostAlloc / registered memory under UVA) take a
 * zero-copy path: the kernel reads the queues and writes the results in host
 * memory over PCIe (one launch, no copies; workspace unused and may be NULL);
 * the results are valid once the stream is synchronised. */
size_t orloj_pick_batch_host_workspace(int64_t num_queues, int64_t num_members);
orloj_status orloj_pick_batch_host(const orloj_store *store, const orloj_latency_profile *profile,
                                   int64_t num_queues, const int64_t *queue_offsets_host,
                                   const int64_t *deadline_ticks_host, const int32_t *dist_id_host,
                                   const int64_t *now_ticks_host, int32_t *best_k_host,
                                   float *best_expected_host, void *workspace,
                                   size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Trace replay (readings A9, A11, A15-A17).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t num_scenarios;           /* S >= 0 */
  const int64_t *arrival_offsets;  /* device [S+1], CSR over arrivals */
  const int64_t *arrival_ticks;    /* device [N], non-decreasing within a scenario */
  const int32_t *dist_id;          /* device [N] */
  const int16_t *true_bin;         /* device [N], 1..B: hidden execution time, used only at dispatch */
  const int64_t *slo_ticks;        /* device [S] >= 0: deadline = arrival + slo (constant per scenario) */
  const int32_t *bucket;           /* device [S], 0 <= bucket < num_buckets */
  int32_t num_buckets;             /* >= 1 */
} orloj_trace;

typedef struct {
  int64_t total;      /* arrivals */
  int64_t finished;   /* completed with end <= deadline (A11) */
  int64_t dropped;    /* dropped as hopeless: P_r(1) = 0 (A16) */
  int64_t late;       /* dispatched, completed after the deadline (A17) */
  int64_t batches;    /* decisions = dispatched batches */
  int64_t busy_ticks; /* sum of batch durations */
  int64_t span_ticks; /* end of last batch - first arrival */
} orloj_counters;

/* Replay every scenario on a single non-preemptive worker.  Per scenario, in
 * this order, until every arrival is handled: (1) if nothing is queued, jump to
 * the next arrival (work-conserving, A15); (2) scan the live queue (window
 * remainder first, then arrivals <= t) from the head, dropping each hopeless
 * request and collecting the others into a window of <= kmax (A16); (3) pick
 * k* on the window exactly as orloj_pick_batch; (4) dispatch the first k*:
 * dur = a_k* + w_k* * max true_bin; finished / late by the deadline; (5) t += dur.
 * per_bucket: device [num_buckets]; counters are ADDED (atomics), so zero them
 * first.  decision_log: device int32 [N + S] or NULL; decision d of scenario s
 * is written at [arrival_offsets[s] + s + d], followed by a 0.
 * Limits: kmax <= 32, B <= 128, D*B*4 <= 64 KiB (CAPACITY otherwise); every
 * scenario holds fewer than 2^31 - 64 arrivals (per-scenario indices and counts
 * are 32-bit in the kernel; orloj_validate_trace checks it, and a replay that
 * meets a longer scenario faults: ORLOJ_ERR_CUDA at the next synchronisation). */
orloj_status orloj_replay_trace(const orloj_store *store, const orloj_latency_profile *profile,
                                const orloj_trace *trace, orloj_counters *per_bucket,
                                int32_t *decision_log, void *stream);

/* Replay policy variants (the Alg. 1 ingredients,
 * PAPER.md:306-373).  objective: ORLOJ_OBJ_EXPECTED_FINISH picks argmax E_k
 * (the default of orloj_replay_trace); ORLOJ_OBJ_FINISH_RATE picks argmax
 * E_k / E[L_{B_k}] — expected finishes per tick of worker time, the 1/E[L]
 * factor of Eq. 1 with E[L_{B_k}] from Eq. 5 (:493-502); ties
 * -> smallest k.  drop_threshold_ticks: device int64 [num_dists] or NULL.  A
 * request of distribution d is dropped at time t iff D_r - t < thr[d]; NULL
 * means the hopeless rule thr[d] = a_1 + w_1 m_min(d) (P_r(1) = 0, A16).  The
 * Alg. 1 drop "t + EstimateBatchLatency(r, 1) > D_r" is
 * thr[d] = a_1 + ceil(w_1 E[bin_d]) (an integer the caller computes from the
 * histogram counts).  Thresholds are assumed non-negative and fixed per replay
 * (dropping stays permanent only if thr[d] <= a_1 + w_1 B). */
/* ORLOJ_OBJ_ALG1 replays the paper's scheduler iteration (Alg. 1)
 * over the window (the kmax earliest-deadline pending requests, A9):
 *   drop (l.10-13): r leaves every Q_bs iff t + E[L_bs] > D_r for all bs, i.e.
 *     D_r - t < thr_1 (E[L_bs] is non-decreasing in bs);
 *   Q_bs = {r : D_r - t >= thr_bs}, thr_bs = ceil(E[L_bs]) of the
 *     all-application batch model (integer ticks, so the test is exact);
 *   candidate (l.14-19): among bs with |Q_bs| >= bs the earliest D_{Q_bs}, ties ->
 *     larger bs (the prose "overall earliest deadline" reading of l.15);
 *   PopBatch (l.20): the bs members of Q_bs with the highest Eq. 1-2 priority
 *     (orloj_priority_table tables, ties -> earlier member); the rest stay pending.
 * The decision log then holds, per decision, the bit mask of popped window
 * positions (bit r = r-th earliest-deadline pending member). */
typedef enum { ORLOJ_OBJ_EXPECTED_FINISH = 0, ORLOJ_OBJ_FINISH_RATE = 1, ORLOJ_OBJ_ALG1 = 2 } orloj_objective;
typedef struct {
  int32_t objective;                   /* orloj_objective */
  const int64_t *drop_threshold_ticks; /* device [num_dists] or NULL (hopeless rule); NULL for ALG1 */
  /* ALG1 only (NULL / 0 otherwise): */
  const int64_t *size_threshold_ticks;  /* device [kmax]: thr_bs = ceil(E[L_bs]), non-decreasing, >= 0 */
  const double *priority_table;         /* device [kmax][2][B+1] (orloj_priority_table, num_sizes = kmax) */
  const double *priority_log_expected;  /* device [kmax] */
  double priority_b_per_tick;           /* the b the tables were built with */
} orloj_replay_policy;
orloj_status orloj_replay_trace_ex(const orloj_store *store, const orloj_latency_profile *profile,
                                   const orloj_trace *trace, const orloj_replay_policy *policy,
                                   orloj_counters *per_bucket, int32_t *decision_log, void *stream);

/* Exact thresholds for the replay policies (host arrays; synchronous host
 * computation, no device work; off the critical path like the paper's per-bs
 * precompute).  counts: host uint32 [D][B], every row with a
 * positive total (COLD_START otherwise).  Both are exact ceilings of exact
 * rationals (no floating point):
 *  - orloj_expected_latency_thresholds: thr[d] = a_1 + ceil(w_1 sum_i i c_{d,i} /
 *    sum_i c_{d,i}) — EstimateBatchLatency(r, 1) of Alg. 1's drop under
 *    the E_k scorer's model (A1: a batch of one whose member sits in bin m runs
 *    a_1 + w_1 m), the drop_threshold_ticks of ORLOJ_OBJ_EXPECTED_FINISH /
 *    FINISH_RATE replays.  thr: host int64 [D].
 *  - orloj_alg1_size_thresholds: thr_bs = ceil(E[L_bs]) for bs = 1..kmax under
 *    Alg. 1's batch model (R10/R11: bs i.i.d. draws from the weighted mixture
 *    of all applications, each bin's mass uniform within it as in Eq. 2):
 *    E[L_bs] = a_bs + w_bs sum_i (G_i - G_{i-1}) (i - 1/2), G_i = F_mix(tau_i)^bs —
 *    the size_threshold_ticks of ORLOJ_OBJ_ALG1.  weights: host double [D] (>= 0,
 *    not all 0; each taken as the exact dyadic rational it is) or NULL
 *    (uniform).  thr: host int64 [kmax].  CAPACITY if the common denominator
 *    of the mixture exceeds 2^65536.
 * The two readings of a bin's mass (upper edge vs uniform) differ on purpose:
 * each threshold belongs to the model its policy scores with. */
orloj_status orloj_expected_latency_thresholds(const uint32_t *counts, int32_t num_dists, int32_t num_bins,
                                               const orloj_latency_profile *profile, int64_t *thr);
orloj_status orloj_alg1_size_thresholds(const uint32_t *counts, int32_t num_dists, int32_t num_bins,
                                        const double *weights, const orloj_latency_profile *profile,
                                        int64_t *thr);

/* Segmented replay: the same replay (every counter and decision-log entry
 * identical to orloj_replay_trace_ex, bit for bit) with a shorter critical
 * path.  Each scenario's arrivals are cut into `segments` equal ranges
 * s_g = floor(g n / segments); one warp per (scenario, segment) replays range g
 * from an empty queue and records where its run *regenerates* (at a decision
 * point nothing is pending and the worker is free by the next arrival j: from
 * there on the run equals a fresh replay started at j, whatever came before);
 * a second pass continues the true run from segment 0 and, in each later
 * segment, switches to the segment's own run at the first regeneration point
 * both pass through (or runs through the segment itself when there is none).
 * The scenarios' sequential decision chains (A9, A15: one worker, non-
 * preemptive) are what bounds the replay on many SMs; segments split them.
 * segments: 1..ORLOJ_REPLAY_MAX_SEGMENTS (1 = orloj_replay_trace_ex; workspace
 * may then be NULL).  num_arrivals: arrival_offsets[S] (sizes the workspace).
 * workspace: caller-owned, 256-byte aligned device memory of at least
 * orloj_replay_seg_workspace(S, num_arrivals, segments, decision_log != NULL)
 * bytes; contents are scratch except its first 40 bytes, which hold int64
 * diagnostics of the call once it completes: {decisions the second pass re-ran,
 * segments joined at a common regeneration point, segments run through,
 * decisions the first pass made past the segment ends, size error}.  The
 * workspace is sized from num_arrivals: if arrival_offsets[S] exceeds it the
 * kernels do nothing (counters and log untouched) and set the size-error word
 * to 1 (the check needs the device offsets, so it cannot be synchronous).
 * policy: as orloj_replay_trace_ex (NULL: the
 * default expected-finish policy).  Errors: INVALID_ARGUMENT for a bad segment
 * count or a missing / short / misaligned workspace, else as
 * orloj_replay_trace_ex. */
#define ORLOJ_REPLAY_MAX_SEGMENTS 4096
size_t orloj_replay_seg_workspace(int64_t num_scenarios, int64_t num_arrivals, int32_t segments,
                                  int32_t with_log);
orloj_status orloj_replay_trace_seg(const orloj_store *store, const orloj_latency_profile *profile,
                                    const orloj_trace *trace, const orloj_replay_policy *policy,
                                    int32_t segments, int64_t num_arrivals, void *workspace,
                                    size_t workspace_bytes, orloj_counters *per_bucket,
                                    int32_t *decision_log, void *stream);

/* ---------------------------------------------------------------------------
 * Long-term feedback loop: "finished
 * requests are sampled and sent to the profiler to evaluate individually. The
 * execution time data will then be asynchronously picked up and accumulated
 * by the scheduler periodically ... resets its profiling memory every once in
 * a while."  Reading R15: a replay is cut into epochs; the
 * store is static during an epoch (A18); at the end of an epoch the sampled
 * completed requests' solo times (their hidden true bins) are added to the
 * profiling window, every row whose window holds >= min_samples samples is
 * rebuilt, and the window is reset every window_epochs epochs.  An epoch
 * boundary is a batching barrier (an epoch's arrivals are all handled before
 * the next epoch's are admitted); the worker's busy time carries over.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t epoch;              /* 0 <= epoch < num_epochs */
  int32_t num_epochs;         /* >= 1: epoch e of scenario s = its arrivals [s_e, s_{e+1}), s_e = floor(e n_s / num_epochs) */
  int64_t *worker_free_ticks; /* device int64 [S] or NULL: read at the start (the worker is busy until then;
                                 INT64_MIN = free), overwritten with the end of the scenario's last batch */
  uint8_t *outcome;           /* device uint8 [N] or NULL: every arrival of the epoch gets 1 (finished),
                                 2 (late) or 3 (dropped); other entries are untouched */
} orloj_replay_epoch;
/* orloj_replay_trace_ex over one epoch (plain kernel).  Counters count the
 * epoch's arrivals (span_ticks = end of its last batch - its first arrival).
 * decision_log: device int32 [N + S] or NULL; decision d of the epoch of
 * scenario s at [arrival_offsets[s] + s + s_e + d], followed by a 0 (give each
 * epoch its own log buffer to keep all of them).  policy NULL = default. */
orloj_status orloj_replay_trace_epoch(const orloj_store *store, const orloj_latency_profile *profile,
                                      const orloj_trace *trace, const orloj_replay_policy *policy,
                                      const orloj_replay_epoch *epoch, orloj_counters *per_bucket,
                                      int32_t *decision_log, void *stream);
/* Profiler: arrival j with outcome[j] in {1, 2} (completed: "finished
 * requests") and sample_mask[j] != 0 (sample_mask NULL = every one)
 * adds 1 to counts[dist_id[j]][true_bin[j] - 1] — its solo execution time,
 * which the replay knows as the hidden true bin.  counts: device uint32 [D][B],
 * ADDED to.  Async.  Errors: INVALID_ARGUMENT, CAPACITY (D*B > 2^30), CUDA. */
orloj_status orloj_profile_outcomes(const int32_t *dist_id, const int16_t *true_bin, const uint8_t *outcome,
                                    const uint8_t *sample_mask, int64_t num_arrivals, uint32_t *counts,
                                    int32_t num_dists, int32_t num_bins, void *stream);
/* Refresh: rows d whose counts total >= max(1, min_samples) are rebuilt as
 * orloj_store_build does (same arithmetic, bit for bit); the other rows of
 * log2_cdf are left as they are (the previous profile stays in use until the
 * window has enough samples; no COLD_START).  Async, no allocation. */
orloj_status orloj_store_refresh(const uint32_t *counts, int32_t num_dists, int32_t num_bins, uint32_t min_samples,
                                 float *log2_cdf, void *stream);
typedef struct {
  int32_t num_epochs;          /* E >= 1 */
  int32_t window_epochs;       /* W >= 1: the window counts are zeroed after epochs W-1, 2W-1, ... */
  uint32_t min_samples;        /* >= 1 */
  const uint8_t *sample_mask;  /* device uint8 [N] or NULL: which completed requests the profiler evaluates */
} orloj_feedback;
size_t orloj_replay_feedback_workspace(int64_t num_scenarios, int64_t num_arrivals, int32_t num_dists,
                                       int32_t num_bins);
/* The whole loop, natively: for e = 0..E-1 { orloj_replay_trace_epoch(e) with
 * the worker time carried; orloj_profile_outcomes into the window;
 * orloj_store_refresh of `store` in place; reset the window if (e+1) % W == 0 }.
 * store->log2_cdf is REWRITTEN (it must be writable device memory; its
 * initial rows are the prior profile).  per_epoch_bucket: device [E][num_buckets]
 * counters, ADDED to.  window_counts_out: device uint32 [D][B] or NULL: the
 * window the last refresh used.  decision_logs: device int32 [E][N + S] or
 * NULL (epoch e's log at offset e (N + S), layout as orloj_replay_trace_epoch).
 * workspace: >= orloj_replay_feedback_workspace(S, N, D, B) bytes, 256-byte
 * aligned.  Synchronises `stream` once at the start (reads arrival_offsets[S]);
 * otherwise async.  Errors: as the calls it makes. */
orloj_status orloj_replay_feedback(const orloj_store *store, const orloj_latency_profile *profile,
                                   const orloj_trace *trace, const orloj_replay_policy *policy,
                                   const orloj_feedback *feedback, void *workspace, size_t workspace_bytes,
                                   orloj_counters *per_epoch_bucket, uint32_t *window_counts_out,
                                   int32_t *decision_logs, void *stream);

/* ---------------------------------------------------------------------------
 * Eq. 1-2 priority scores and PopBatch (PAPER.md:423-455,
 * :585-593, Alg. 1 :306-373).
 *
 * Batch latency of size bs (1..num_sizes): a batch of bs requests drawn from
 * the mixture of all application distributions (weights) has its
 * latency in bin i = (l1, l2] = (a_bs + w_bs (i-1), a_bs + w_bs i] with
 * probability pm_i = F_mix(tau_i)^bs - F_mix(tau_{i-1})^bs (Eq. 3-4, Eq. 6
 * i.i.d., A1 grid), uniform within the bin (the histogram of Eq. 2, frequency
 * h_i = pm_i / w_bs).  The priority of a request with slack sigma = D_r - t is
 * Eq. 1 with the step cost (c = 1) and an Exp(b) delay, summed per bin as
 * Eq. 2:
 *   p = (1 / E[L_bs]) sum_i { (h_i/b)(e^{b l2} - e^{b l1}) e^{-b sigma}   l2 <= sigma
 *                             (h_i/b)(1 - e^{-b (sigma - l1)})            l1 < sigma < l2
 *                             0                                           sigma <= l1 }
 * with E[L_bs] = sum_i pm_i (l1 + l2) / 2.  Scores are returned as log p
 * (fp32; -inf when no outcome meets the deadline).
 * ------------------------------------------------------------------------- */
/* Build the per-size tables (off the critical path; synchronous).
 * log_table: device double [num_sizes][2][B+1]; [s][0][i] = log of the
 * full-bin sum over bins 1..i divided by e^{-b sigma} (-inf at i = 0),
 * [s][1][i] = log(h_i / b) (-inf when pm_i = 0 and at i = 0).  log_expected:
 * device double [num_sizes], log E[L_bs].  weights: device float [D] (>= 0,
 * not all 0) or NULL (uniform).  b_per_tick > 0 with b_per_tick * w_bs small
 * enough that e^{b w} is finite (b w < 709).  num_sizes <= profile.kmax. */
orloj_status orloj_priority_table(const orloj_store *store, const orloj_latency_profile *profile,
                                  int32_t num_sizes, const float *weights, double b_per_tick,
                                  double *log_table, double *log_expected, void *stream);
/* log p for every queue member and batch size: device float [num_sizes][N]
 * (size-major), N = queue_offsets[Q] - queue_offsets[0].  Uses only
 * queue_offsets, deadline_ticks and now_ticks.  Async on stream.  The call
 * re-bases the fp64 tables into an fp32 table per block and picks one of two
 * arithmetic tiers on the host (a fitted polynomial for 1 - e^{-bx} when it
 * holds to 2^-23 over the profile's bin widths, else a series / ex2 form);
 * both meet |d log p| <= 1e-6 + 2^-22 |log p|.  A table
 * larger than the shared-memory budget (num_sizes x (B+2) entries above
 * ~88 KiB) is re-based into a stream-ordered scratch allocation instead. */
orloj_status orloj_priority_scores(const orloj_store *store, const orloj_latency_profile *profile,
                                   int32_t num_sizes, double b_per_tick, const double *log_table,
                                   const double *log_expected, const orloj_queues *queues, float *log_priority,
                                   void *stream);
/* Piecewise-step cost: a request misses deadline D_r + offset[s]
 * at cumulative cost cost[s]; the cost function decomposes into single steps at
 * D_r + offset[s] with cost cost[s] - cost[s-1] (cost[-1] = 0), and the
 * priority is the sum of the single-step priorities (Eq. 2 each, same E[L]).
 * offset_ticks: host int64 [num_steps], strictly increasing, |offset| <= 2^40;
 * cost: host double [num_steps], strictly increasing from > 0; 1 <= num_steps
 * <= 8.  Copied at the call (no ownership kept). */
typedef struct {
  int32_t num_steps;
  const int64_t *offset_ticks;
  const double *cost;
} orloj_cost_steps;
/* orloj_priority_scores with a piecewise-step cost per request (same layout);
 * steps = {1, {0}, {1.0}} reproduces orloj_priority_scores.  Async. */
orloj_status orloj_priority_scores_steps(const orloj_store *store, const orloj_latency_profile *profile,
                                         int32_t num_sizes, double b_per_tick, const double *log_table,
                                         const double *log_expected, const orloj_queues *queues,
                                         const orloj_cost_steps *steps, float *log_priority, void *stream);
/* PopBatch: per queue q, the (up to) batch_size[q] <= 32 members with the
 * highest log p for that size (ties -> earlier member; -inf and NaN never
 * chosen), among the first 256 members; log_priority is the [num_sizes][N]
 * output of orloj_priority_scores.  selected: device int32 [Q][32],
 * member index within the queue, highest priority first, -1 after the last
 * (a batch_size outside [1, num_sizes] selects nothing).  Async on stream. */
orloj_status orloj_pop_batch(const orloj_queues *queues, const float *log_priority, int32_t num_sizes,
                             const int32_t *batch_size, int32_t *selected, void *stream);

/* ---------------------------------------------------------------------------
 * Scoring-model variants: the expected finish count
 *   E_k = sum_{r<=k} sum_s dc_s P(t + L_{B_k} <= D_r + offset_s)
 * for k = 1..K (K = min(n_q, kmax), kmax <= 32, B <= 128) with
 *   - duration_ticks: device int64 [kmax][B+1]; dur[k-1][m] = duration of a
 *     batch of k whose slowest member sits at bin position m (m = 0..B; bin i
 *     spans positions (i-1, i]); non-decreasing in m (Eq. 3 is a_k + w_k m;
 *     any grid, e.g. log-spaced, is a table);
 *   - interpolate = 0: every bin's mass at its upper edge (A1): P = G_k(i*),
 *     i* = #{m >= 1 : dur[k-1][m] <= x};  interpolate = 1: each member's
 *     position uniform within its bin (linear CDF inside bins) and
 *     the duration linear between grid positions: with dur[m] <= x < dur[m+1],
 *     u = (x - dur[m]) / (dur[m+1] - dur[m]),
 *     P = prod_j (F_j(m) + u (F_j(m+1) - F_j(m))), F_j(0) = 0; x >= dur[B] -> 1;
 *   - a piecewise-step cost: num_steps (0 = one unit step at
 *     offset 0, else 1..8) host arrays step_offset_ticks (strictly increasing)
 *     and step_cost (cumulative, strictly increasing from > 0); dc_s = c_s - c_{s-1}.
 * expected_finish: device float [Q][kmax] (entries k > K are 0); best_k /
 * best_expected: device [Q] or NULL (argmax, ties -> smallest k; 0 for empty
 * queues).  Async. */
typedef struct {
  int32_t kmax;
  const int64_t *duration_ticks;
  int32_t interpolate;
  int32_t num_steps;
  const int64_t *step_offset_ticks;
  const double *step_cost;
  const void *plan; /* device ORLOJ_SCORE_MODEL_PLAN_BYTES from orloj_score_model_prepare for this
                       duration table (reused across calls), or NULL: analysed on every call */
} orloj_score_model;
orloj_status orloj_score_model_batches(const orloj_store *store, const orloj_queues *queues,
                                       const orloj_score_model *model, float *expected_finish, int32_t *best_k,
                                       float *best_expected, void *stream);

/* Analyse a duration table once (async on `stream`): for each size k, whether
 * its row is an arithmetic grid dur[m] = dur[0] + w m (Eq. 3; w >= 1,
 * dur[0] >= 0, dur[0] + w B < 2^30), and if so the constants of the main
 * scorer's exact integer lookup (floor((x - dur[0]) / w) by a division magic)
 * that orloj_score_model_batches then uses instead of a binary search over the
 * row -- the same bin, so the same results.  plan: device buffer of
 * ORLOJ_SCORE_MODEL_PLAN_BYTES (caller-owned; valid while the table is
 * unchanged).  model->plan is ignored here. */
#define ORLOJ_SCORE_MODEL_PLAN_BYTES 512
orloj_status orloj_score_model_prepare(const orloj_score_model *model, int32_t num_bins, void *plan, void *stream);

/* ---------------------------------------------------------------------------
 * Validation (synchronous, O(N), not hot; may allocate a few bytes of scratch).
 * ------------------------------------------------------------------------- */
/* rows non-decreasing, <= 0, no NaN, [d][B-1] == 0.0f.  INVALID_ARGUMENT otherwise. */
orloj_status orloj_validate_store(const orloj_store *store, void *stream);
/* offsets monotone from 0; dist ids in range (INVALID_ARGUMENT); per-queue
 * (deadline, arrival, index) order (UNSORTED; arrival used when non-NULL). */
orloj_status orloj_validate_queues(const orloj_store *store, const orloj_queues *queues, void *stream);
/* offsets monotone from 0, ids / bins / buckets in range, slo >= 0, fewer than
 * 2^31 - 64 arrivals per scenario (INVALID_ARGUMENT); arrivals non-decreasing
 * per scenario (UNSORTED). */
orloj_status orloj_validate_trace(const orloj_store *store, const orloj_trace *trace, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ORLOJ_H */
