/*
 * augsched.h — C ABI of libaugsched, a B200-native (sm_100a) implementation of
 * the per-iteration scheduling pass of AugServe (arXiv 2512.04013).
 *
 * Citations: "P:n" is line n of the paper's text; "Eq.k" follows the
 * order of \begin{equation} there (Eq.4 = P:479 ... Eq.32 = P:741); "Rk" is a
 * reading fixed in DESIGN.md where the paper is silent.
 *
 * What one scheduling step computes (Algorithm 1), per instance:
 *   1. Stage I on arrivals: policy argmin of Eq.4-8, value V1 of Eq.9-15.
 *   2. Stage II on returned calls: V2 of Eq.16-22 and V_final of Eq.23-25;
 *      route Preserve->running, Swap->swapped, Discard->waiting.
 *   3. Token limit: Eq.27-32 on the KV ledger, clamped to
 *      [floor(beta_low*target_max), floor(beta_high*target_max)].
 *   4. Score: key = orderable_u32(fp32(V - alpha*(now-last)*T)) (Eq.26, R1, R3).
 *   5. Order: running => swapped => waiting, each ascending by key, ties by
 *      request id (R2, R16).
 *   6. Admit the prefix whose preceding demand is below the limit, with a
 *      partial last chunk (P:1225-1229 + chunked prefill P:1102, R17).
 *   7. Rare memory resolution: demote Preserve-paused KV, then evict from the
 *      tail of the order (R20).
 * augsched_simulate additionally runs the engine model (R21-R24) and the
 * metrics to completion.
 *
 * Conventions
 *   - Every call returns an int status: AUGSCHED_OK (0) or a negative code; no
 *     C++ exception crosses the ABI; augsched_last_error() gives a
 *     thread-local message for the last non-zero status.
 *   - Time is integer: iterations (uint64) and microsecond ticks (uint64).
 *     Token counts are integers; values/scores are IEEE binary64 computed
 *     without FMA contraction, converted once to fp32 for the key (R3).
 *   - A handle owns every device buffer it allocates and issues all work on the
 *     CUDA stream given at creation (a cudaStream_t, e.g. a torch stream's
 *     pointer; NULL = legacy default stream).  Calls are asynchronous with
 *     respect to the host unless documented otherwise.  A handle may move
 *     between threads but must not be used by two threads at once.
 *   - Device-side faults (a state violation seen by a kernel) are latched in a
 *     device error word and returned by the next call that synchronizes
 *     (augsched_sync, augsched_simulate with AUGSCHED_HOST_RESULTS) as
 *     AUGSCHED_E_STATE.
 */
#ifndef AUGSCHED_H_
#define AUGSCHED_H_

#include <stdint.h>

#if defined(__GNUC__)
#define AUGSCHED_API __attribute__((visibility("default")))
#else
#define AUGSCHED_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------- */
#define AUGSCHED_OK 0
#define AUGSCHED_E_INVALID (-1)       /* bad argument or configuration */
#define AUGSCHED_E_CAPACITY (-2)      /* a queue/slot/trace exceeds the handle's capacity */
#define AUGSCHED_E_CUDA (-3)          /* a CUDA runtime error (message has the name) */
#define AUGSCHED_E_STATE (-4)         /* a record violates the request state machine */
#define AUGSCHED_E_OOM (-5)           /* device allocation failed */
#define AUGSCHED_E_UNIMPLEMENTED (-6)

/* ---- policies and ranking/budget modes ----------------------- */
#define AUGSCHED_PRESERVE 0
#define AUGSCHED_SWAP 1
#define AUGSCHED_DISCARD 2

#define AUGSCHED_RANK_AUGSERVE 0      /* value order of Eq.26 */
#define AUGSCHED_RANK_FCFS 1          /* key = 0: order (tier, id) (R33) */
#define AUGSCHED_RANK_RANDOM 2        /* random scheduling of P:266-273: a fresh shuffle every
                                         iteration, key = hi32(mix(mix(rank_seed<<32 | id) ^ t))
                                         with mix = the SplitMix64 output function (reading B8) */
#define AUGSCHED_RANK_AUGSERVE_TI 3   /* time-invariant form of Eq.26 (reading B12):
                                         key = orderable_u32(fp32(V + alpha*(last*T))); between two events
                                         it ranks like V - alpha*(now-last)*T in exact arithmetic, and a
                                         waiting request's key never changes, so augsched_step on a
                                         single-instance handle keeps the order incrementally (merge of the
                                         changed entries into the previous order) */
#define AUGSCHED_BUDGET_DYNAMIC 0     /* Eq.27-32 + clamp */
#define AUGSCHED_BUDGET_STATIC 1      /* fixed l_static tokens */
#define AUGSCHED_POLICY_ARGMIN 0      /* Eq.7-8 */
#define AUGSCHED_POLICY_PRESERVE 1    /* forced policy (baseline emulation) */
#define AUGSCHED_POLICY_SWAP 2
#define AUGSCHED_POLICY_DISCARD 3

/* Per-instance sweep parameters (one serving instance = one queue set). */
typedef struct augsched_instance_params {
  uint32_t target_max;       /* target_max of P:749; also N^fwd_max in Eq.6/9/17/18 (R9); >= 1 */
  uint32_t l_static;         /* static token limit when budget_mode == STATIC */
  double alpha;              /* anti-starvation coefficient of Eq.26, value units per second; >= 0 */
  uint64_t slo_ttft_ticks;   /* TTFT SLO in µs (1 s) */
  uint32_t slo_norm_num;     /* normalized-latency SLO = num/den x T^fwd (10/1) */
  uint32_t slo_norm_den;
  uint32_t ranking;          /* AUGSCHED_RANK_* */
  uint32_t budget_mode;      /* AUGSCHED_BUDGET_* */
  uint32_t policy_mode;      /* AUGSCHED_POLICY_* */
  uint32_t rank_seed;        /* seed of AUGSCHED_RANK_RANDOM (ignored otherwise) */
} augsched_instance_params;

/* System constants (SPEC SimConfig). */
typedef struct augsched_config {
  uint64_t m_per_token;      /* M: KV bytes per token; >= 1 */
  uint64_t g_total;          /* G_total bytes (Eq.30) */
  uint64_t g_model, g_runtime, g_safety;  /* G_fixed = sum (Eq.29); G_fixed < G_total */
  uint64_t t_fwd_ticks;      /* T^fwd in µs; >= 1 */
  uint32_t s_in, s_out;      /* S^fwd_in / S^fwd_out tokens per iteration; >= 1 */
  uint32_t gamma_num, gamma_den;  /* gamma of Eq.31 = num/den in [0, 1]; den >= 1 */
  double beta_low, beta_high;     /* clamp factors, 0 <= beta_low <= beta_high */
  augsched_instance_params defaults;  /* used when create() gets per_inst == NULL */
} augsched_config;

/* ---- simulation inputs (all arrays in one memory space, see flags) --------
 * CSR trace set: trace k owns requests [req_off[k], req_off[k+1]) in arrival
 * order; request r owns segments [seg_off[r], seg_off[r] + n_seg[r]).  A
 * segment is a decode phase of gen_true tokens followed (except the last) by
 * a tool call of dur_true µs that returns ret_len tokens.
 * gen_pred / dur_pred are the predictor's outputs.  Arrival
 * ticks must be nondecreasing within a trace; gen_true >= 1 (R29).           */
typedef struct augsched_trace {
  const uint32_t* req_off;   /* [n_traces + 1] */
  const uint64_t* arr_tick;  /* [n_req] arrival time, µs */
  const uint32_t* l_pre;     /* [n_req] prompt tokens L^pre (>= 1) */
  const uint32_t* seg_off;   /* [n_req] */
  const uint32_t* n_seg;     /* [n_req] in [1, 255] (simulate reports E_INVALID otherwise) */
  const uint32_t* gen_true;  /* [n_seg_total] */
  const uint32_t* gen_pred;  /* [n_seg_total] predicted L^out */
  const uint32_t* dur_true;  /* [n_seg_total] call duration µs (ignored for last segment) */
  const float* dur_pred;     /* [n_seg_total] predicted T^api, seconds */
  const uint32_t* ret_len;   /* [n_seg_total] returned tokens R (ignored for last) */
  uint32_t n_traces;
  uint32_t n_req;            /* total requests (length of per-request arrays) */
  uint32_t n_seg_total;      /* total segments */
  uint32_t reserved;
} augsched_trace;

/* ---- table-driven workload generator --------------------
 * W1/W2/W3 traces drawn on the device, identical to the host twin
 * tracegen/tablegen.py: u = mix(mix(seed << 32 | trace) ^ (request << 12 |
 * field)) with mix = the SplitMix64 output function; continuous
 * distributions through 4,096-level quantile tables (index u >> 52); integer
 * draws from u >> 32 (see tracegen/tablegen.py for every field).           */
typedef struct augsched_gen_tables {
  const double* gap;         /* [4096] unit-mean inter-arrival quantiles (exponential or gamma) */
  const uint32_t* prompt;    /* [4096] prompt tokens */
  const uint32_t* gen;       /* [4096] decoded tokens per segment */
  const uint32_t* dur;       /* [4][4096] call duration (µs) per tool class */
  const uint32_t* ret;       /* [4][4096] returned tokens per tool class */
  const double* noise;       /* [4096] multiplicative duration-prediction noise */
  uint32_t cls_th[3];        /* cumulative class-share thresholds on u >> 32 */
  uint32_t calls_lo[4], calls_hi[4];
  uint32_t edges[8], mids[8];/* bucket predictor: edges and reported midpoints */
  uint32_t acc_th;           /* predictor hit iff u >> 32 < acc_th */
  uint32_t nocall_th;        /* request without calls iff u >> 32 < nocall_th */
  uint32_t oracle_pred;      /* 1: predictions = truth */
  uint32_t reserved;
} augsched_gen_tables;

typedef struct augsched_gen_spec {
  uint32_t seed, n_traces, n_max, reserved;
  uint64_t horizon_ticks;    /* 0: W2 (exactly n_max requests per trace); else W1/W3 cut */
  const double* scale;       /* device [n_traces]: 1e6 / (rate of trace k, req/s) */
} augsched_gen_spec;

/* Per-instance result record of augsched_simulate (fixed size, byte-comparable). */
enum {
  AUGSCHED_R_NREQ = 0, AUGSCHED_R_ARRIVED, AUGSCHED_R_COMPLETED, AUGSCHED_R_SLO_OK,
  AUGSCHED_R_SLO_OK_5X, AUGSCHED_R_BUSY_STEPS, AUGSCHED_R_DECISIONS, AUGSCHED_R_EVICTIONS,
  AUGSCHED_R_DEMOTIONS, AUGSCHED_R_CALLS_PRESERVE, AUGSCHED_R_CALLS_SWAP,
  AUGSCHED_R_CALLS_DISCARD, AUGSCHED_R_RETURNS, AUGSCHED_R_TOKENS, AUGSCHED_R_FINAL_T,
  AUGSCHED_R_MAKESPAN, AUGSCHED_R_SUM_TTFT, AUGSCHED_R_SUM_E2E, AUGSCHED_R_SUM_GEN,
  AUGSCHED_R_ADMITTED, AUGSCHED_R_ERR, AUGSCHED_R_MAXQ,
  AUGSCHED_R_INCOMPLETE,  /* requests not finished when the run stopped (R28) */
  AUGSCHED_R_RSV23,
  AUGSCHED_R_NFIELD
};
#define AUGSCHED_NBIN 160   /* integer log-linear bins: v<16 -> v; else 16+4(e-4)+2 mantissa bits */
typedef struct augsched_result {
  uint64_t f[AUGSCHED_R_NFIELD];
  uint32_t hist_ttft[AUGSCHED_NBIN];   /* TTFT in µs */
  uint32_t hist_norm[AUGSCHED_NBIN];   /* floor(e2e µs / generated tokens) */
} augsched_result;

/* simulate flags */
#define AUGSCHED_HOST_TRACES 1u   /* traces + inst_trace_id are host pointers: copied in (timed) */
#define AUGSCHED_HOST_RESULTS 2u  /* results is a host pointer: copied out, call synchronizes */
#define AUGSCHED_RESUME 4u        /* continue from the handle's state instead of t = 0 */

/* ---- step mode (the scheduler as a library) ------------------------------
 * Record kinds enqueued between steps; processed at the start of the next
 * augsched_step in the order CALL/FINISH (engine events of the last forward),
 * snapshot, RETURN (Stage II), NEW/IMPORT (Stage I / restore).             */
#define AUGSCHED_K_NEW 1      /* id empty -> waiting; la = l_pre, lb = gen_pred, ta = dur_pred, flags bit0 = has call */
#define AUGSCHED_K_RETURN 2   /* id paused -> routed; la = returned tokens R, lb = next gen_pred, ta = next dur_pred, bit0 = next call */
#define AUGSCHED_K_CALL 3     /* id running & decode-ready -> paused with S~ (R13); ta = dur_pred of the call */
#define AUGSCHED_K_FINISH 4   /* id active -> empty, KV released */
#define AUGSCHED_K_IMPORT 5   /* id empty -> given state: flags bits4-6 status (1 run,2 swap,3 wait,4 paused),
                                 bits 8-9 applied policy, bit 12 stage II; la/lb/lc/ta value features
                                 (stage I: L, O, -, A; stage II: Lt, R, O', A'); last/ctx/kv/cpu/pend token state */
typedef struct augsched_record_soa {
  const uint32_t* kind;
  const uint32_t* id;      /* slot index < max_active_per_instance */
  const uint32_t* la;
  const uint32_t* lb;
  const uint32_t* lc;
  const float* ta;
  const uint32_t* flags;
  const uint32_t* last;
  const uint32_t* ctx;
  const uint32_t* kv;
  const uint32_t* cpu;
  const uint32_t* pend;
} augsched_record_soa;

/* Outputs of one step: device pointers owned by the handle, valid until the
 * next call on it.  Per instance i the queue segment is
 * [i*max_active, i*max_active + n_active[i]) of order/grant/key.
 *
 * admitted[i] is the length of the admission prefix: the entries j of the
 * order with P_{j-1} < B that Algorithm 1 adds to the batch (P:1225-1229,
 * R17), counted BEFORE memory resolution (R20).  A tail eviction can cancel
 * a grant inside the prefix, so grant[j] may be 0 for j < admitted[i]; the
 * batch to run is {order[j] : j < admitted[i], grant[j] > 0}.  augsched_step
 * writes grant[j] = 0 for every admitted[i] <= j < n_active[i].
 * tier_off[3*i + k] is the position (within instance i's segment) where
 * tier k (0 running, 1 swapped, 2 waiting, R16) starts; tier k
 * ends where tier k+1 starts, tier 2 at n_active[i].                      */
typedef struct augsched_step_out {
  const int64_t* budget;     /* [n_instances] token limit N_max of this step */
  const uint32_t* n_active;  /* [n_instances] |running u swapped u waiting| */
  const uint32_t* admitted;  /* [n_instances] admission-prefix length (see above) */
  const uint32_t* order;     /* slot ids in scheduling order */
  const uint32_t* grant;     /* tokens granted to order[j] this step (0 if none or cancelled) */
  const uint32_t* key;       /* orderable u32 of the fp32 score of order[j] */
  const uint32_t* tier_off;  /* [3 * n_instances] per-tier segment starts (augsched_step only;
                                NULL from augsched_step_prefix) */
} augsched_step_out;

typedef struct augsched_handle augsched_t;

/* Create a handle for n_instances independent instances with room for
 * max_active_per_instance requests each (simulate: >= the longest trace and
 * <= 65535; step: slots per instance).  per_inst: host array of n_instances
 * params or NULL (cfg->defaults for all).  Validates S:43-45: quantities > 0,
 * 0 <= gamma <= 1, beta_low <= beta_high, G_fixed < G_total, alpha >= 0.
 * device: CUDA ordinal; cuda_stream: cudaStream_t (borrowed, not owned).
 * Returns OK, E_INVALID, E_OOM or E_CUDA. */
AUGSCHED_API int augsched_create(const augsched_config* cfg, const augsched_instance_params* per_inst,
                    uint32_t n_instances, uint32_t max_active_per_instance, int device,
                    void* cuda_stream, augsched_t** out);

/* Queue n records for `instance` (step mode).  recs_on_device = 0: host
 * arrays, copied before return; 1: device arrays that must stay valid until
 * the handle's stream passes this call.  Host-side capacity check:
 * E_CAPACITY if the pending queue would exceed max_active_per_instance * 4
 * records; E_INVALID for a bad kind/id.  State violations are detected on
 * the device and reported as E_STATE by a later synchronizing call. */
AUGSCHED_API int augsched_enqueue(augsched_t* h, uint32_t instance, const augsched_record_soa* recs, uint32_t n,
                     int recs_on_device);

/* One scheduling step at iteration now_iter for every instance (steps 1-7
 * above, then last = now for granted requests and the granted batch's token
 * accounting: swap-in, recompute, prefill/assimilate, decode).  Fills `out`
 * with device pointers.  Asynchronous.  The order is the unique sorted order
 * of (tier, key, slot) (R2); when the previous call on the
 * handle was also augsched_step, the handle starts from its own copy of that
 * order and merges the slots changed since (records, grants, evictions) into
 * it -- for time-invariant keys always, for R3 / FCFS keys after checking
 * that the unchanged ones are still in order -- and sorts otherwise; the
 * outputs are the same either way. */
AUGSCHED_API int augsched_step(augsched_t* h, uint64_t now_iter, augsched_step_out* out);

/* The same decision round as augsched_step (identical grants, limits, queue
 * sizes and state updates), producing the order only for the admitted
 * prefix: order/key/grant are valid for positions [0, admitted) of each
 * instance; later positions are not written.  Every queued request has
 * demand >= 1, so the admitted prefix lies within the first min(B, n)
 * entries of the order, and they are found by selection instead of a full
 * sort when the handle's largest token limit is <= 8192:
 *   - one instance: one cooperative kernel (one launch per call): a
 *     streaming pass keeps the words at or below the current word of an
 *     anchor slot chosen by the previous call (exact whenever their count
 *     lies in [min(B, n), 8192]; otherwise a histogram pass and a collect
 *     pass), then one CTA sorts and admits them.  The kernel needs every
 *     SM's share of the grid resident at once (cooperative launch);
 *   - several instances whose slots fit in shared memory: one CTA per
 *     instance, the same anchored filter per instance, else a radix select.
 * Any other handle runs augsched_step.  Asynchronous. */
AUGSCHED_API int augsched_step_prefix(augsched_t* h, uint64_t now_iter, augsched_step_out* out);

/* Export instance `instance`'s slot state to host memory (synchronizes the
 * handle's stream): slots[6*x .. 6*x+5] = status (0 empty, 1 running,
 * 2 swapped, 3 waiting, 4 paused), applied policy (AUGSCHED_PRESERVE/SWAP/
 * DISCARD; 2 for an empty slot), ctx, kv, cpu, pend of slot x (the token
 * state an IMPORT record carries); ledger[0..1] = A (KV of non-paused
 * requests) and P (KV of Preserve-paused requests), Eq.27-28.  Either
 * pointer may be NULL.  Records still pending are not applied.  Returns OK,
 * E_INVALID or E_CUDA (a latched device fault is left for augsched_sync). */
AUGSCHED_API int augsched_step_export(augsched_t* h, uint32_t instance, int32_t* slots, int64_t* ledger);

/* ---- sharded single queue --------------------------------
 * One global queue whose slots are split over G ranks (one GPU each): rank
 * r's handle is a single-instance handle (all ranks: the same config,
 * parameters and max_active) holding global slots
 * [r * max_active, (r + 1) * max_active).  Every queued request has demand
 * >= 1, so the global admission prefix (Algorithm 1's fill loop)
 * lies within the union of every shard's first min(B, n_r) order entries;
 * the shards exchange only those (and, for the rare R20 resolution, their
 * KV holders) once per step.  A step is three calls around two collectives
 * the caller runs over its process group (rank-major, e.g. NCCL):
 *   1. augsched_shard_begin(h, now, ledger): this step's CALL / FINISH
 *      records, their C_other (Eq.5, R13) taken from the GLOBAL ledger the
 *      last commit left; ledger = device int64[2] <- this shard's (A, P)
 *      after them.
 *        -> all-reduce(SUM) of ledger over the ranks: ledger_sum[0] is the
 *           global S1 snapshot A_snap
 *   2. augsched_shard_offer(h, ledger_sum, offer): RETURN / NEW / IMPORT
 *      records against A_snap (Stage I/II policy predictions, R7/R12);
 *      this shard's order (as augsched_step) and its offer: a device buffer
 *      of augsched_shard_offer_bytes(h) bytes (header with the shard's
 *      ledger, its first min(n_r, cap >= every limit) order entries
 *      {packed word tier:2 | key:32 | local slot:30, demand, kv}, its
 *      queued slots holding KV, its Preserve-paused slots).
 *        -> all-gather of the offers (rank-major, G * offer bytes)
 *   3. augsched_shard_commit(h, offers, G, rank, out): the limit B from
 *      the global ledger (Eq.27-32), the merge of the offers, the global
 *      admission prefix (R17), memory pressure resolved over the gathered
 *      holders (R20), this shard's part applied (grants, last = now,
 *      evictions, demotions) and the global ledger for the next step.  out: the global prefix
 *      (order = global slot ids, grant, key) of length admitted[0], B in
 *      budget[0], the global queue size in n_active[0] (device pointers
 *      valid until the next call).  E_CAPACITY (latched, returned by
 *      augsched_sync) if a shard had more KV holders than its offer holds and
 *      the step needed them.  Asynchronous. */
AUGSCHED_API uint64_t augsched_shard_offer_bytes(const augsched_t* h);
AUGSCHED_API int augsched_shard_begin(augsched_t* h, uint64_t now_iter, int64_t* ledger);
AUGSCHED_API int augsched_shard_offer(augsched_t* h, const int64_t* ledger_sum, void* offer);
AUGSCHED_API int augsched_shard_commit(augsched_t* h, const void* offers, uint32_t n_ranks, uint32_t rank,
                                       augsched_step_out* out);

/* Run every instance's simulation (Algorithm 1 + engine model + metrics) until
 * all its requests finished or its iteration counter reaches max_iters.
 * inst_trace_id[i] selects instance i's trace.  results: n_instances records.
 * flags: AUGSCHED_HOST_TRACES / AUGSCHED_HOST_RESULTS / AUGSCHED_RESUME.
 * Without HOST_RESULTS the call is asynchronous and results must be a
 * device buffer.  E_CAPACITY if a trace is longer than the handle allows.
 * The per-request checks (n_seg in [1, 255], segment lists inside the
 * segment arrays) run on the device before the simulation: a violation
 * latches E_INVALID, returned by the synchronizing call (this one with
 * HOST_RESULTS, else augsched_sync), and no instance is simulated.
 * max_iters <= 2^32 (E_INVALID otherwise). */
AUGSCHED_API int augsched_simulate(augsched_t* h, const augsched_trace* traces, const uint32_t* inst_trace_id,
                      uint64_t max_iters, augsched_result* results, uint32_t flags);

/* Generate n_traces traces on the device into `out` (device arrays allocated
 * by the caller: req_off [n_traces + 1], per-request arrays [req_cap],
 * per-segment arrays [seg_cap]; `tables` points to device tables).  Sets
 * out->n_traces / n_req / n_seg_total (the call synchronizes the handle's
 * stream to read the totals).  E_CAPACITY if the traces need more than
 * req_cap requests or seg_cap segments; E_INVALID for bad arguments. */
AUGSCHED_API int augsched_generate(augsched_t* h, const augsched_gen_spec* spec, const augsched_gen_tables* tables,
                      augsched_trace* out, uint32_t req_cap, uint32_t seg_cap);

/* Wait for the handle's stream; returns a latched device error (E_STATE) if
 * any, once: the latch is cleared when it is reported. */
AUGSCHED_API int augsched_sync(augsched_t* h);

/* Number of kernel launches issued by this handle since creation. */
AUGSCHED_API uint64_t augsched_launch_count(const augsched_t* h);

/* Synchronize and free everything.  Safe on NULL. */
AUGSCHED_API void augsched_destroy(augsched_t* h);

/* Thread-local message for the last non-zero status ("" if none). */
AUGSCHED_API const char* augsched_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* AUGSCHED_H_ */
