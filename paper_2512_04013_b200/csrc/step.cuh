// augsched_step: the scheduler as a library over per-instance slot arrays.
// One step (Algorithm 1, for every instance at once):
//   [records]  CALL/FINISH -> snapshot -> RETURN (Stage II) / NEW (Stage I) / IMPORT
//   keys       Eq.26 key per slot + token limit (Eq.27-32) + digit histograms
//   sort       stable LSD radix sort of (instance, tier, key) with slot-id
//              payload, one kernel per 8-bit digit, decoupled look-back
//   admit      block prefix scan of demand over each instance's order (R17)
//   resolve    demotion + tail eviction when the grants exceed free KV (R20)
//   apply      last = now and the granted batch's token accounting
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "augsched.h"
#include "model.cuh"

namespace augsched {

constexpr int STEP_MAX_PASS = 8;

struct PassDesc {
  int src;    // 0: byte of the u32 key, 1: tier (payload >> 30), 2: byte of the instance index
  int shift;
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
  // outputs
  long long* budget = nullptr;
  uint32_t *n_active = nullptr, *admitted = nullptr, *order = nullptr, *grant = nullptr,
           *key = nullptr, *flag = nullptr;
  // sort scratch
  uint32_t *k0 = nullptr, *v0 = nullptr, *k1 = nullptr, *v1 = nullptr;
  unsigned long long* lb_status = nullptr;
  uint32_t* ghist = nullptr;      // [STEP_MAX_PASS][256]
  uint32_t* tile_ctr = nullptr;   // [STEP_MAX_PASS]
  unsigned long long epoch = 0;
  int npass = 0;
  PassDesc passes[STEP_MAX_PASS];
  uint32_t n_tiles = 0;
  void* alloc_list[64];
  int n_alloc = 0;
};

int step_ensure(StepState& st, uint32_t n_inst, uint32_t max_active, cudaStream_t s,
                const augsched_config& cfg, const augsched_instance_params* d_ip, uint64_t* launches);
int step_enqueue(StepState& st, uint32_t inst, const augsched_record_soa* r, uint32_t n, int on_dev,
                 cudaStream_t s, uint32_t* d_err, uint64_t* launches);
int step_run(StepState& st, const augsched_config& cfg, int64_t cap,
             const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
             augsched_step_out* out, cudaStream_t s, uint64_t* launches);
void step_free(StepState& st);
int set_error(int code, const char* msg);

}  // namespace augsched
