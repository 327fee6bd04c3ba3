// augsched_step: the scheduler as a library over per-instance slot arrays.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "augsched.h"

namespace augsched {

struct StepState {
  bool ready = false;
  uint32_t n_inst = 0, max_active = 0;
};

int step_ensure(StepState& st, uint32_t n_inst, uint32_t max_active, cudaStream_t s);
int step_enqueue(StepState& st, uint32_t inst, const augsched_record_soa* r, uint32_t n, int on_dev,
                 cudaStream_t s, uint64_t* launches);
int step_run(StepState& st, const augsched_config& cfg, int64_t cap,
             const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
             augsched_step_out* out, cudaStream_t s, uint64_t* launches);
void step_free(StepState& st);
int set_error(int code, const char* msg);

}  // namespace augsched
