// augsched_step: the scheduler as a library over per-instance slot arrays.
// One step (Algorithm 1, for every instance at once):
//   [records]  CALL/FINISH -> snapshot -> RETURN (Stage II) / NEW (Stage I) / IMPORT
//   keys       Eq.26 key per slot + token limit (Eq.27-32) + digit histograms
//              of every sort pass; writes one packed u64 per slot:
//              tier:2 | key:32 | slot:30 (most significant first)
//   sort       stable LSD radix sort of (instance, tier, key) with the slot
//              id carried in the low bits: 8+8+8 key bits, then a 10-bit
//              digit (top key byte + tier), then instance bytes; one kernel
//              per digit with a two-level (group / tile) aggregate look-back
//   admit      one block per instance: prefix scan of demand over the order
//              (R17), demotion + tail eviction when the grants exceed free
//              KV (R20), then last = now and the granted batch's token
//              accounting
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "augsched.h"
#include "model.cuh"

namespace augsched {

constexpr int STEP_MAX_PASS = 8;
constexpr int STEP_RB_MAX = 10;                 // widest digit (bins = 1 << bits)
constexpr int STEP_HIST_WORDS = 4096;          // bins over all passes (<= 8), or the prefix digit
#ifndef AUGSCHED_PF_BITS
#define AUGSCHED_PF_BITS 12
#endif
constexpr int PF_BITS = AUGSCHED_PF_BITS;       // prefix step: top digit (tier:2 + key top bits)
constexpr uint32_t PF_SCAP = 8192;              // prefix step: admitted-prefix capacity (max limit)
constexpr uint32_t PF_CCAP = 16384;             // prefix step: crossing-bucket entries kept on chip
constexpr size_t PF_MULTI_SMEM = 200 * 1024;    // prefix step, several instances: shared memory per CTA

struct PassDesc {
  int src;    // 0: `bits` bits of the packed key at `shift`; 2: byte of the instance index
  int shift;
  int bits;
  int hoff;   // offset of this pass's bins in the histogram array
};

struct StepState {
  bool ready = false;
  uint32_t n_inst = 0, max_active = 0;
  size_t N = 0;
  // slot state
  uint32_t* st = nullptr;      // status (bits 0-3) | applied policy << 4
  double* V = nullptr;
  uint32_t* last = nullptr;
  int32_t *ctx = nullptr, *kv = nullptr, *cpu = nullptr, *pend = nullptr;
  long long *A = nullptr, *P = nullptr, *Aevt = nullptr, *Asnap = nullptr, *need = nullptr;
  Coef* coef = nullptr;
  // pending records (device SoA; ids converted to global slot indices)
  uint32_t *r_kind = nullptr, *r_id = nullptr, *r_la = nullptr, *r_lb = nullptr, *r_lc = nullptr,
           *r_flags = nullptr, *r_last = nullptr, *r_ctx = nullptr, *r_kv = nullptr,
           *r_cpu = nullptr, *r_pend = nullptr;
  float* r_ta = nullptr;
  uint32_t r_cap = 0, r_n = 0;
  uint64_t last_now = 0;         // last `now` passed to a step (time must not run backwards)
  uint64_t shard_now = 0;        // sharded queue (f4): the iteration of the step in progress
  const int64_t* shard_ledger = nullptr;
  uint32_t shard_batch = 0;      // the record batch split over shard_begin / shard_offer
  long long* gA = nullptr;       // [2] global (A, P) after the last commit
  bool have_now = false;
  // duplicate-record detection: per slot, the winning record of the batch in
  // each record phase (CALL/FINISH; RETURN/NEW/IMPORT), key
  // (~batch << 32) | prio << 31 | index, atomicMin
  unsigned long long *claimA = nullptr, *claimB = nullptr;
  uint32_t rec_batch = 0;        // batches processed so far
  // outputs
  long long* budget = nullptr;
  uint32_t *n_active = nullptr, *admitted = nullptr, *order = nullptr, *grant = nullptr,
           *key = nullptr, *flag = nullptr;
  uint32_t* tcnt = nullptr;      // [4 * n_inst] per-tier queue counts of the full step (zeroed each step)
  uint32_t* tier_off = nullptr;  // [3 * n_inst] per-tier segment starts (full step output)
  uint32_t* gdirty = nullptr;    // [n_inst] grant[] positions [0, gdirty) may hold grants of earlier steps
  // sort scratch
  unsigned long long *k0 = nullptr, *k1 = nullptr;   // packed tier:2 | key:32 | slot:30
  unsigned long long* lb_status = nullptr;           // [tiles][1 << STEP_RB_MAX] tile aggregates
  unsigned long long* lb_gstatus = nullptr;          // [groups][1 << STEP_RB_MAX] group aggregates
  uint32_t G = 1;                                    // tiles per look-back group
  uint32_t* ghist = nullptr;      // [STEP_HIST_WORDS]
  uint32_t* tile_ctr = nullptr;   // [STEP_MAX_PASS]
  unsigned long long epoch = 0;
  int npass = 0;
  PassDesc passes[STEP_MAX_PASS];
  uint32_t n_tiles = 0;
  uint32_t* zbuf = nullptr;       // [n_inst | STEP_HIST_WORDS | STEP_MAX_PASS | 4], zeroed every step
  uint32_t* pf_cnt = nullptr;     // prefix step: [|A|, |C|]
  unsigned long long *pf_A = nullptr, *pf_C = nullptr;   // prefix step candidates (packed words)
  uint32_t* gslot = nullptr;      // prefix step: grant by slot during resolution (kept zero)
  unsigned long long* pf_theta = nullptr;   // prefix step: anchor word and slot (kept across steps)
  unsigned long long* pf_H = nullptr;       // prefix step: holder list (resolution candidates)
  uint32_t* wkv = nullptr;                  // sticky flag: KV held outside running / swapped / Preserve-paused
  uint32_t* pf_nact = nullptr;              // prefix step: queue-size words, alternating by epoch
  uint32_t pf_epoch = 0;                    // prefix step: calls so far (epoch tag of the kernel's flags)
  bool pf_dirty = false;                    // a full step ran since: counters need one clear
  int pf_grid = 0;                // prefix step: co-resident CTAs of the cooperative kernel
  int coop_grid = 0;              // full step, one instance: CTAs of the cooperative kernel (0: not used)
  // time-invariant keys (ranking 3, one instance): the order is kept across
  // steps; a step merges the slots changed since the last one into it
  bool ti = false;
  bool vi = false;                // the same for value (R3) / FCFS keys: words recomputed, order checked
  bool ti_valid = false;          // tiw holds the previous full step's sorted words
  uint32_t ti_ep = 0;             // step epoch (dirty marks)
  unsigned long long *tiw = nullptr, *tiw2 = nullptr;   // [N] sorted words (current, next)
  uint32_t* ti_n = nullptr;       // [1] entries in tiw
  uint32_t* dmark = nullptr;      // [N] epoch of the slot's last change
  uint32_t* dlist = nullptr;      // [2][TI_DCAP] changed slots by epoch parity
  uint32_t* dcnt = nullptr;       // [2] their counts
  unsigned long long* ubuf = nullptr;   // [N] the unchanged words, compacted
  uint32_t* ti_misc = nullptr;    // [4] per-call scratch: |D| after filtering, tier counts of D
  uint32_t* ti_gcnt = nullptr;    // [TI_DCAP + 1] unchanged words per rank among the changed ones
  // batched full step (full_multi_kernel): each instance's order is kept
  // across steps and the next step merges what changed into it
  bool minc = false;
  bool minc_valid = false;        // mord holds the previous full step's order of every instance
  uint32_t* mord = nullptr;       // [N] order by instance (local slots)
  uint32_t* mord_n = nullptr;     // [n_inst] its length
  unsigned long long* coop_bar = nullptr;   // its grid-barrier counter (monotone)
  unsigned long long coop_bar_base = 0;     // the counter's value at the next call's start
  uint32_t* coop_hist = nullptr;            // [4][coop_grid][512] per-CTA digit histograms
  bool pf_spec = true;            // prefix step: speculative pass (off when any instance shuffles)
  uint32_t max_limit = 0;         // largest token limit any instance can get
  size_t zwords = 0;
  int sms = 148;
  void* alloc_list[64];
  int n_alloc = 0;
};

int step_ensure(StepState& st, uint32_t n_inst, uint32_t max_active, cudaStream_t s,
                const augsched_config& cfg, const augsched_instance_params* d_ip, uint64_t* launches);
int step_enqueue(StepState& st, uint32_t inst, const augsched_record_soa* r, uint32_t n, int on_dev,
                 cudaStream_t s, uint32_t* d_err, uint64_t* launches);
int step_run_prefix(StepState& st, const augsched_config& cfg, int64_t cap,
                    const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
                    augsched_step_out* out, cudaStream_t s, uint64_t* launches);
int step_run(StepState& st, const augsched_config& cfg, int64_t cap,
             const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
             augsched_step_out* out, cudaStream_t s, uint64_t* launches);
size_t step_shard_offer_bytes(const StepState& st);
int step_shard_begin(StepState& st, const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
                     int64_t* ledger, cudaStream_t s, uint64_t* launches);
int step_shard_offer(StepState& st, const augsched_config& cfg, int64_t cap, const augsched_instance_params* d_ip,
                     uint32_t* d_err, const int64_t* ledger_sum, void* offer, cudaStream_t s, uint64_t* launches);
int step_shard_commit(StepState& st, const augsched_config& cfg, int64_t cap, const augsched_instance_params* d_ip,
                      uint32_t* d_err, const int64_t* ledger_sum, const void* offers, uint32_t n_ranks,
                      uint32_t rank, augsched_step_out* out, cudaStream_t s, uint64_t* launches);
void step_free(StepState& st);
int set_error(int code, const char* msg);

}  // namespace augsched
