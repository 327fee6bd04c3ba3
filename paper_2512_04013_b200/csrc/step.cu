#include "step.cuh"
namespace augsched {
int step_ensure(StepState& st, uint32_t n_inst, uint32_t max_active, cudaStream_t) {
  st.n_inst = n_inst; st.max_active = max_active; return AUGSCHED_OK;
}
int step_enqueue(StepState&, uint32_t, const augsched_record_soa*, uint32_t, int, cudaStream_t, uint64_t*) {
  return set_error(AUGSCHED_E_UNIMPLEMENTED, "step mode not built yet");
}
int step_run(StepState&, const augsched_config&, int64_t, const augsched_instance_params*, uint32_t*,
             uint64_t, augsched_step_out*, cudaStream_t, uint64_t*) {
  return set_error(AUGSCHED_E_UNIMPLEMENTED, "step mode not built yet");
}
void step_free(StepState&) {}
}  // namespace augsched
