// Persistent per-instance simulation kernel (K8 of SURVEY §2.4), fusing
// intake (Stage I/II), the token-limit update, scoring, ordering, admission,
// memory resolution, engine advance and metrics for one instance per CTA.
//
// Ordering without a sort: the per-step outputs that feed the simulation only
// depend on WHICH entries fall in the admitted prefix of the (tier, key, id)
// order and on the single partially-granted entry (R17), and, under memory
// pressure, on which tail entries are evicted (R20).  Both are weighted
// order statistics: the admitted prefix ends at the first entry whose
// cumulative demand reaches the limit B, the evicted tail at the first entry
// (from the back) whose cumulative kv+grant reaches the deficit.  They are
// found exactly by an MSD radix select over the unique 50-bit composite key
// (tier << 48 | key << 16 | id) with demand-weighted shared-memory
// histograms (warp-aggregated with __match_any_sync / __reduce_add_sync).
// augsched_step, whose API returns the full order, uses the sort kernels.
#pragma once
#include <cstdint>
#include "augsched.h"
#include "model.cuh"

namespace augsched {

#ifndef AUGSCHED_SIM_NT
#define AUGSCHED_SIM_NT 32
#endif
// One warp per CTA by default: an instance's per-step barriers are then
// warp-local, and many more instances are resident per SM.
constexpr int SIM_NT = AUGSCHED_SIM_NT;
constexpr int SIM_RB = SIM_NT >= 256 ? 8 : 5;   // radix bits of the fallback select
#ifndef AUGSCHED_SIM_CAND
#define AUGSCHED_SIM_CAND 64
#endif
constexpr int SIM_CAND = AUGSCHED_SIM_CAND;      // small-candidate list capacity
#ifndef AUGSCHED_SIM_MINB
#define AUGSCHED_SIM_MINB 32
#endif
#ifndef AUGSCHED_SIM_UNROLL
#define AUGSCHED_SIM_UNROLL 2
#endif
constexpr int SIM_MINB = AUGSCHED_SIM_MINB;   // resident instances (warps) per SM the registers are bounded for
constexpr int SIM_UNROLL = AUGSCHED_SIM_UNROLL;  // queue entries in flight per thread in the key pass
constexpr int SIM_NW = SIM_NT / 32;
// One-warp instances per CTA.  Above 1 the CTA's instances advance in step
// (one CTA barrier per iteration) so its warps run the same phase of the
// step at the same time and share the instruction stream (the step's code
// far exceeds the SM's 32 KB instruction cache).
#ifndef AUGSCHED_SIM_WPC
#define AUGSCHED_SIM_WPC 16
#endif
constexpr int SIM_WPC = AUGSCHED_SIM_WPC;
static_assert(SIM_WPC == 1 || SIM_NT == 32, "several instances per CTA need one-warp instances");
constexpr int KBITS = 50;                 // tier(2) | key(32) | id(16)
constexpr uint64_t KMASK = (1ull << KBITS) - 1;
constexpr uint64_t KEVICT = 1ull << 63;   // marks an evicted entry in the K array
constexpr int HOLE_CAP = 64;              // serial hole filling up to this many removals

// Trace set as the kernel sees it (device pointers).
struct DevTrace {
  const uint32_t* req_off;
  const uint64_t* arr_tick;
  const uint32_t* l_pre;
  const uint32_t* seg_off;
  const uint32_t* n_seg;
  const uint32_t* gen_true;
  const uint32_t* gen_pred;
  const uint32_t* dur_true;
  const float* dur_pred;
  const uint32_t* ret_len;
};

// Per-instance persistent header (resumable simulation).
struct InstHdr {
  uint64_t t;
  int64_t A, P;           // KV ledger in tokens: active, Preserve-paused
  uint64_t min_ret;       // min return tick over the paused list
  uint64_t w2;            // demand total of the W list
  uint32_t next_arr, n_r, n_w, n_pz, n_fin;
  uint32_t started;
  // W list layout (sim.cu "sorted W list"): sorted main [wh, ws) with mh
  // holes, unsorted tail [ws, we), in buffer wbuf
  uint32_t wh, ws, we, mh, wbuf, tclean;
};

// Mutable state of one request, packed in one 32-byte sector so the engine
// advance of a granted entry is a single gather (two 16-byte loads).
struct __align__(32) ReqState {
  int32_t ctx;         // context tokens (prompt + generated + returned so far)
  int32_t kv;          // tokens whose KV is on the GPU
  int32_t cpu;         // tokens swapped out to host memory (Swap policy)
  int32_t pend;        // tokens to prefill / assimilate (prompt or returned R)
  uint32_t meta;       // seg:8 | status:4 | pol:4 | n_seg:8
  uint32_t ft;         // first-token iteration (t+1 >= 1; 0 = none)
  uint32_t lastc;      // last-scheduled iteration while paused (R14)
  uint32_t left;       // tokens still to decode in the current segment
};

// Scoring record of one queued request (one 16-byte vector load).
struct __align__(16) QEnt {
  double V;            // value (Stage I / II / final), fixed between events
  uint32_t last;       // last-scheduled iteration (R14)
  uint32_t e;          // request id | tier << 30
};

// Handle-owned per-instance arena (stride = max_active entries per instance).
struct Arena {
  // cold state by request id
  ReqState* rs;
  uint64_t* ret;       // return tick of the outstanding call
  // queue lists by position (tier-split): R = running u swapped (tier 0/1),
  // W = waiting (tier 2); scoring record + demand.  W has two buffers of
  // w_stride entries per instance (instance i, buffer b at
  // (2 i + b) * w_stride): the sorted-W rebuild writes the other buffer.
  QEnt* r_q;
  uint32_t* r_dem;
  QEnt* w_q;
  uint32_t* w_dem;
  // paused list by position
  uint32_t* pz_id;
  // per-step scratch: keys / weights of the R list (and of W when a step
  // needs them materialised); secondary selections (demotion, eviction)
  uint64_t* kscr;
  uint32_t* wscr;
  uint64_t* kscr2;
  uint32_t* wscr2;
};

struct SimParams {
  augsched_config cfg;
  int64_t cap;                               // floor((G_total - G_fixed)/M)
  DevTrace tr;
  const augsched_instance_params* ip;        // [n_inst]
  const uint32_t* inst_trace;                // [n_inst]
  Arena ar;
  InstHdr* hdr;                              // [n_inst]
  augsched_result* acc;                      // [n_inst] handle-owned accumulators
  augsched_result* out;                      // [n_inst] caller's results (device)
  uint64_t max_iters;
  uint32_t n_inst, max_active;
  uint32_t w_stride;                         // entries per W buffer (2 * max_active)
  uint32_t* work;                            // work-stealing counter
  uint32_t* err;                             // device error word
};

// Entries per W buffer: the sorted W list leaves removed entries as holes
// and appends at the tail, so a buffer holds twice the live capacity before
// a rebuild compacts it (sim.cu, w_rebuild).
__host__ __device__ inline uint32_t sim_w_stride(uint32_t max_active) { return 2u * max_active; }

__device__ __forceinline__ uint32_t meta_seg(uint32_t m) { return m & 0xFF; }
__device__ __forceinline__ uint32_t meta_st(uint32_t m) { return (m >> 8) & 0xF; }
__device__ __forceinline__ uint32_t meta_pol(uint32_t m) { return (m >> 12) & 0xF; }
__device__ __forceinline__ uint32_t meta_nseg(uint32_t m) { return (m >> 16) & 0xFF; }
__device__ __forceinline__ uint32_t make_meta(uint32_t seg, uint32_t st, uint32_t pol, uint32_t nseg) {
  return (seg & 0xFF) | (st << 8) | (pol << 12) | ((nseg & 0xFF) << 16);
}
__device__ __forceinline__ uint32_t meta_with(uint32_t m, uint32_t st, uint32_t pol) {
  return (m & 0xFFFF00FFu) | (st << 8) | (pol << 12);
}

}  // namespace augsched
