// Host side of libaugsched: handle lifetime, validation, device memory and
// launches.  All entry points are extern "C" (include/augsched.h); errors are
// returned as status codes with a thread-local message, never as exceptions.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>
#include "augsched.h"
#include "sim.cuh"
#include "step.cuh"

namespace augsched {
size_t sim_smem_bytes();
const void* sim_kernel_ptr();
cudaError_t launch_sim(const SimParams& p, int grid, size_t smem, cudaStream_t st);
int launch_generate(const augsched_gen_tables& tb, const augsched_gen_spec& sp, const augsched_trace& out,
                    uint32_t req_cap, uint32_t seg_cap, uint32_t* scratch, uint32_t* totals, uint32_t* err,
                    cudaStream_t s);
}  // namespace augsched

using namespace augsched;

namespace {

__global__ void validate_requests_kernel(const uint32_t* seg_off, const uint32_t* n_seg, uint32_t n_req,
                                         uint32_t n_seg_total, uint32_t* err, uint32_t* work) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_req) return;
  const uint32_t ns = n_seg[r];
  if (ns < 1 || ns > 255 || (uint64_t)seg_off[r] + ns > n_seg_total) {
    atomicOr(err, 4u);
    atomicMax(work, 0x80000000u);   // the simulate kernel finds no instance to run
  }
}

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      if (e_ == cudaErrorMemoryAllocation) {                                        \
        cudaGetLastError();                                                         \
        return fail(AUGSCHED_E_OOM, "%s: %s", #expr, cudaGetErrorString(e_));       \
      }                                                                             \
      return fail(AUGSCHED_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));        \
    }                                                                               \
  } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc(reinterpret_cast<void**>(p), (n ? n : 1) * sizeof(T));
}

}  // namespace

struct augsched_handle {
  augsched_config cfg{};
  uint32_t n_inst = 0, max_active = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t cap = 0;
  std::vector<void*> allocs;
  augsched_instance_params* d_ip = nullptr;
  uint32_t* d_err = nullptr;
  uint32_t* d_work = nullptr;
  uint64_t launches = 0;
  // simulate state
  Arena ar{};
  InstHdr* d_hdr = nullptr;
  augsched_result* d_acc = nullptr;
  bool sim_ready = false;
  int sim_grid = 0;
  size_t sim_smem = 0;
  // host-trace staging (AUGSCHED_HOST_TRACES)
  void* d_trace_buf = nullptr;
  size_t d_trace_cap = 0;
  uint32_t* d_inst_trace = nullptr;
  // workload generator scratch
  uint32_t* gen_scratch = nullptr;
  size_t gen_scratch_words = 0;
  // step mode
  StepState st{};
  bool step_ready = false;

  template <class T>
  int alloc(T** p, size_t n) {
    cudaError_t e = dalloc(p, n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(e == cudaErrorMemoryAllocation ? AUGSCHED_E_OOM : AUGSCHED_E_CUDA,
                  "cudaMalloc(%zu bytes): %s", n * sizeof(T), cudaGetErrorString(e));
    }
    allocs.push_back(*p);
    return AUGSCHED_OK;
  }
};

namespace {

int validate_params(const augsched_instance_params& p, uint32_t i) {
  if (p.target_max < 1) return fail(AUGSCHED_E_INVALID, "instance %u: target_max must be >= 1", i);
  if (!(p.alpha >= 0.0) || !std::isfinite(p.alpha))
    return fail(AUGSCHED_E_INVALID, "instance %u: alpha must be finite and >= 0", i);
  if (p.slo_norm_den < 1) return fail(AUGSCHED_E_INVALID, "instance %u: slo_norm_den must be >= 1", i);
  if (p.ranking > 3 || p.budget_mode > 1 || p.policy_mode > 3)
    return fail(AUGSCHED_E_INVALID, "instance %u: bad ranking/budget_mode/policy_mode", i);
  if (p.l_static > (1u << 26)) return fail(AUGSCHED_E_INVALID, "instance %u: l_static too large", i);
  return AUGSCHED_OK;
}

int validate_cfg(const augsched_config& c) {
  if (c.m_per_token < 1 || c.t_fwd_ticks < 1 || c.s_in < 1 || c.s_out < 1 || c.gamma_den < 1)
    return fail(AUGSCHED_E_INVALID, "m_per_token, t_fwd_ticks, s_in, s_out, gamma_den must be >= 1");
  if (c.gamma_num > c.gamma_den) return fail(AUGSCHED_E_INVALID, "gamma must be in [0, 1]");
  if (!(c.beta_low >= 0.0) || !(c.beta_high >= c.beta_low) || !std::isfinite(c.beta_high))
    return fail(AUGSCHED_E_INVALID, "need 0 <= beta_low <= beta_high");
  const uint64_t fixed = c.g_model + c.g_runtime + c.g_safety;
  if (fixed < c.g_model || fixed >= c.g_total)
    return fail(AUGSCHED_E_INVALID, "G_model + G_runtime + G_safety must be < G_total");
  return AUGSCHED_OK;
}

int ensure_sim(augsched_t* h) {
  if (h->sim_ready) return AUGSCHED_OK;
  if (h->max_active > 65535)
    return fail(AUGSCHED_E_CAPACITY, "simulate needs max_active_per_instance <= 65535 (got %u)",
                h->max_active);
  const size_t N = (size_t)h->n_inst * h->max_active;
  Arena& a = h->ar;
  int rc;
  if ((rc = h->alloc(&a.rs, N)) || (rc = h->alloc(&a.ret, N)) || (rc = h->alloc(&a.r_q, N)) ||
      (rc = h->alloc(&a.r_dem, N)) || (rc = h->alloc(&a.w_q, N)) || (rc = h->alloc(&a.w_dem, N)) ||
      (rc = h->alloc(&a.pz_id, N)) ||
      (rc = h->alloc(&a.kscr, N)) || (rc = h->alloc(&a.wscr, N)) ||
      (rc = h->alloc(&a.kscr2, N)) || (rc = h->alloc(&a.wscr2, N)) ||
      (rc = h->alloc(&h->d_hdr, h->n_inst)) || (rc = h->alloc(&h->d_acc, h->n_inst)))
    return rc;
  // shared-memory queue capacity and persistent grid
  h->sim_smem = sim_smem_bytes();
  CUDA_TRY(cudaFuncSetAttribute(sim_kernel_ptr(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)h->sim_smem));
  int per_sm = 0, sms = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sim_kernel_ptr(), SIM_NT * SIM_WPC,
                                                         h->sim_smem));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  if (per_sm < 1) return fail(AUGSCHED_E_CUDA, "simulate kernel does not fit on an SM");
  h->sim_grid = per_sm * sms;
  h->sim_ready = true;
  return AUGSCHED_OK;
}

}  // namespace

extern "C" {

const char* augsched_last_error(void) { return g_err; }

uint64_t augsched_launch_count(const augsched_t* h) { return h ? h->launches : 0; }

int augsched_create(const augsched_config* cfg, const augsched_instance_params* per_inst,
                    uint32_t n_instances, uint32_t max_active_per_instance, int device,
                    void* cuda_stream, augsched_t** out) {
  g_err[0] = 0;
  if (!cfg || !out) return fail(AUGSCHED_E_INVALID, "cfg and out must be non-NULL");
  *out = nullptr;
  if (n_instances < 1 || max_active_per_instance < 1)
    return fail(AUGSCHED_E_INVALID, "n_instances and max_active_per_instance must be >= 1");
  int rc = validate_cfg(*cfg);
  if (rc) return rc;
  std::vector<augsched_instance_params> ip(n_instances);
  uint32_t max_limit = 0;
  bool any_random = false, all_ti = true, all_vi = true;
  for (uint32_t i = 0; i < n_instances; ++i) {
    ip[i] = per_inst ? per_inst[i] : cfg->defaults;
    if ((rc = validate_params(ip[i], i))) return rc;
    const double hi = std::floor(cfg->beta_high * (double)ip[i].target_max);
    if (hi > (double)(1u << 26)) return fail(AUGSCHED_E_INVALID, "instance %u: token limit too large", i);
    const uint32_t lim = ip[i].budget_mode == AUGSCHED_BUDGET_STATIC ? ip[i].l_static : (uint32_t)hi;
    max_limit = lim > max_limit ? lim : max_limit;
    any_random = any_random || ip[i].ranking == AUGSCHED_RANK_RANDOM;
    all_ti = all_ti && ip[i].ranking == AUGSCHED_RANK_AUGSERVE_TI;
    all_vi = all_vi && (ip[i].ranking == AUGSCHED_RANK_AUGSERVE || ip[i].ranking == AUGSCHED_RANK_FCFS);
  }
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(AUGSCHED_E_INVALID, "bad device %d", device);
  CUDA_TRY(cudaSetDevice(device));
  augsched_t* h = new (std::nothrow) augsched_t();
  if (!h) return fail(AUGSCHED_E_OOM, "host allocation failed");
  h->cfg = *cfg;
  h->n_inst = n_instances;
  h->max_active = max_active_per_instance;
  h->st.max_limit = max_limit;
  h->st.pf_spec = !any_random;   // a fresh shuffle every iteration leaves no anchor
  h->st.ti = all_ti && n_instances == 1;   // incremental full order (reading B12, f1)
#ifndef AUGSCHED_NO_VI
  h->st.vi = all_vi && n_instances == 1;   // the same for R3 / FCFS keys, order checked every step
#endif
  h->device = device;
  h->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  h->cap = (int64_t)((cfg->g_total - (cfg->g_model + cfg->g_runtime + cfg->g_safety)) /
                     cfg->m_per_token);
  if ((rc = h->alloc(&h->d_ip, n_instances)) || (rc = h->alloc(&h->d_err, 1)) ||
      (rc = h->alloc(&h->d_work, 1))) {
    augsched_destroy(h);
    return rc;
  }
  cudaError_t e = cudaMemcpyAsync(h->d_ip, ip.data(), sizeof(augsched_instance_params) * n_instances,
                                  cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->d_err, 0, sizeof(uint32_t), h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    augsched_destroy(h);
    return fail(AUGSCHED_E_CUDA, "create: %s", cudaGetErrorString(e));
  }
  *out = h;
  return AUGSCHED_OK;
}

void augsched_destroy(augsched_t* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  for (void* p : h->allocs) cudaFree(p);
  if (h->d_trace_buf) cudaFree(h->d_trace_buf);
  if (h->gen_scratch) cudaFree(h->gen_scratch);
  step_free(h->st);
  delete h;
}

int augsched_generate(augsched_t* h, const augsched_gen_spec* spec, const augsched_gen_tables* tables,
                      augsched_trace* out, uint32_t req_cap, uint32_t seg_cap) {
  if (!h || !spec || !tables || !out || !spec->scale) return fail(AUGSCHED_E_INVALID, "generate: NULL argument");
  if (spec->n_traces < 1 || spec->n_max < 1) return fail(AUGSCHED_E_INVALID, "generate: empty spec");
  for (int c = 0; c < 4; ++c)
    if (tables->calls_lo[c] > tables->calls_hi[c] || tables->calls_hi[c] > 254)
      return fail(AUGSCHED_E_INVALID, "generate: calls per request of class %d outside [lo, 254]", c);
  const void* ptrs[] = {tables->gap, tables->prompt, tables->gen, tables->dur, tables->ret, tables->noise,
                        out->req_off, out->arr_tick, out->l_pre, out->seg_off, out->n_seg, out->gen_true,
                        out->gen_pred, out->dur_true, out->dur_pred, out->ret_len};
  for (const void* q : ptrs)
    if (!q) return fail(AUGSCHED_E_INVALID, "generate: NULL table or output array");
  CUDA_TRY(cudaSetDevice(h->device));
  const size_t words = 4 * (size_t)spec->n_traces + 2 + 2;
  if (words > h->gen_scratch_words) {
    if (h->gen_scratch) cudaFree(h->gen_scratch);
    h->gen_scratch = nullptr;
    h->gen_scratch_words = 0;
    CUDA_TRY(cudaMalloc(&h->gen_scratch, words * sizeof(uint32_t)));
    h->gen_scratch_words = words;
  }
  uint32_t* totals = h->gen_scratch + words - 2;
  CUDA_TRY(cudaMemsetAsync(h->d_err, 0, sizeof(uint32_t), h->stream));
  h->launches += launch_generate(*tables, *spec, *out, req_cap, seg_cap, h->gen_scratch, totals, h->d_err,
                                 h->stream);
  CUDA_TRY(cudaGetLastError());
  uint32_t tot[2] = {0, 0}, err = 0;
  CUDA_TRY(cudaMemcpyAsync(tot, totals, sizeof(tot), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(&err, h->d_err, sizeof(err), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (err & 2u) return fail(AUGSCHED_E_CAPACITY, "generate: %u requests / %u segments exceed %u / %u",
                            tot[0], tot[1], req_cap, seg_cap);
  out->n_traces = spec->n_traces;
  out->n_req = tot[0];
  out->n_seg_total = tot[1];
  return AUGSCHED_OK;
}

int augsched_sync(augsched_t* h) {
  if (!h) return fail(AUGSCHED_E_INVALID, "NULL handle");
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  uint32_t err = 0;
  CUDA_TRY(cudaMemcpy(&err, h->d_err, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) CUDA_TRY(cudaMemset(h->d_err, 0, sizeof(err)));   // reported once
  if (err & 1u) return fail(AUGSCHED_E_STATE, "a record violated the request state machine");
  if (err & 2u) return fail(AUGSCHED_E_CAPACITY, "a trace is longer than max_active_per_instance");
  if (err & 4u) return fail(AUGSCHED_E_INVALID, "a request has n_seg outside [1, 255]");
  if (err & 8u) return fail(AUGSCHED_E_STATE, "an invariant of SURVEY 8(c).4 failed (AUGSCHED_DEBUG build)");
  return AUGSCHED_OK;
}

int augsched_simulate(augsched_t* h, const augsched_trace* traces, const uint32_t* inst_trace_id,
                      uint64_t max_iters, augsched_result* results, uint32_t flags) {
  if (!h || !traces || !inst_trace_id || !results)
    return fail(AUGSCHED_E_INVALID, "simulate: NULL argument");
  if (flags & ~(AUGSCHED_HOST_TRACES | AUGSCHED_HOST_RESULTS | AUGSCHED_RESUME))
    return fail(AUGSCHED_E_INVALID, "simulate: unknown flags 0x%x", flags);
  if (max_iters > (1ull << 32))   // last-scheduled iterations are stored as u32 (R14)
    return fail(AUGSCHED_E_INVALID, "simulate: max_iters %llu > 2^32", (unsigned long long)max_iters);
  CUDA_TRY(cudaSetDevice(h->device));
  int rc = ensure_sim(h);
  if (rc) return rc;
  DevTrace tr{traces->req_off, traces->arr_tick, traces->l_pre, traces->seg_off, traces->n_seg,
              traces->gen_true, traces->gen_pred, traces->dur_true, traces->dur_pred,
              traces->ret_len};
  const uint32_t* d_tid = inst_trace_id;
  if (flags & AUGSCHED_HOST_TRACES) {
    // validate on the host while the arrays are visible, then stage them
    const uint32_t nt = traces->n_traces, nr = traces->n_req, ns = traces->n_seg_total;
    if (traces->req_off[nt] != nr) return fail(AUGSCHED_E_INVALID, "req_off[n_traces] != n_req");
    for (uint32_t i = 0; i < h->n_inst; ++i) {
      const uint32_t k = inst_trace_id[i];
      if (k >= nt) return fail(AUGSCHED_E_INVALID, "instance %u: trace id %u out of range", i, k);
      if (traces->req_off[k + 1] - traces->req_off[k] > h->max_active)
        return fail(AUGSCHED_E_CAPACITY, "instance %u: trace %u has %u requests > max_active %u",
                    i, k, traces->req_off[k + 1] - traces->req_off[k], h->max_active);
    }
    // the per-request segment checks run on the device (validate_requests_kernel)
    const size_t b_req_off = sizeof(uint32_t) * (nt + 1), b64 = sizeof(uint64_t) * nr,
                 b32r = sizeof(uint32_t) * nr, b32s = sizeof(uint32_t) * ns,
                 btid = sizeof(uint32_t) * h->n_inst;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t need = al(b_req_off) + al(b64) + 3 * al(b32r) + 5 * al(b32s) + al(btid);
    if (need > h->d_trace_cap) {
      if (h->d_trace_buf) cudaFree(h->d_trace_buf);
      h->d_trace_buf = nullptr;
      h->d_trace_cap = 0;
      CUDA_TRY(cudaMalloc(&h->d_trace_buf, need));
      h->d_trace_cap = need;
    }
    char* b = static_cast<char*>(h->d_trace_buf);
    auto put = [&](const void* src, size_t n) -> void* {
      void* d = b;
      if (n) cudaMemcpyAsync(d, src, n, cudaMemcpyHostToDevice, h->stream);
      b += al(n);
      return d;
    };
    tr.req_off = (const uint32_t*)put(traces->req_off, b_req_off);
    tr.arr_tick = (const uint64_t*)put(traces->arr_tick, b64);
    tr.l_pre = (const uint32_t*)put(traces->l_pre, b32r);
    tr.seg_off = (const uint32_t*)put(traces->seg_off, b32r);
    tr.n_seg = (const uint32_t*)put(traces->n_seg, b32r);
    tr.gen_true = (const uint32_t*)put(traces->gen_true, b32s);
    tr.gen_pred = (const uint32_t*)put(traces->gen_pred, b32s);
    tr.dur_true = (const uint32_t*)put(traces->dur_true, b32s);
    tr.dur_pred = (const float*)put(traces->dur_pred, b32s);
    tr.ret_len = (const uint32_t*)put(traces->ret_len, b32s);
    d_tid = (const uint32_t*)put(inst_trace_id, btid);
    CUDA_TRY(cudaGetLastError());
  }
  augsched_result* d_out = results;
  if (flags & AUGSCHED_HOST_RESULTS) d_out = h->d_acc;  // copied out below
  if (!(flags & AUGSCHED_RESUME)) {
    CUDA_TRY(cudaMemsetAsync(h->d_hdr, 0, sizeof(InstHdr) * h->n_inst, h->stream));
    CUDA_TRY(cudaMemsetAsync(h->d_acc, 0, sizeof(augsched_result) * h->n_inst, h->stream));
  }
  CUDA_TRY(cudaMemsetAsync(h->d_work, 0, sizeof(uint32_t), h->stream));
  if (traces->n_req) {
    // segment lists inside the arrays, n_seg in [1, 255] (meta holds 8 bits);
    // a violation latches E_INVALID and leaves the simulation no work
    validate_requests_kernel<<<(traces->n_req + 255) / 256, 256, 0, h->stream>>>(
        tr.seg_off, tr.n_seg, traces->n_req, traces->n_seg_total, h->d_err, h->d_work);
    h->launches += 1;
  }
  SimParams p{};
  p.cfg = h->cfg;
  p.cap = h->cap;
  p.tr = tr;
  p.ip = h->d_ip;
  p.inst_trace = d_tid;
  p.ar = h->ar;
  p.hdr = h->d_hdr;
  p.acc = h->d_acc;
  p.out = d_out;
  p.max_iters = max_iters;
  p.n_inst = h->n_inst;
  p.max_active = h->max_active;
  p.work = h->d_work;
  p.err = h->d_err;
  const uint32_t ctas = (h->n_inst + SIM_WPC - 1) / SIM_WPC;   // SIM_WPC instances in flight per CTA
  const int grid = (int)(ctas < (uint32_t)h->sim_grid ? ctas : (uint32_t)h->sim_grid);
  CUDA_TRY(launch_sim(p, grid, h->sim_smem, h->stream));
  h->launches += 1;
  if (flags & AUGSCHED_HOST_RESULTS) {
    CUDA_TRY(cudaMemcpyAsync(results, h->d_acc, sizeof(augsched_result) * h->n_inst,
                             cudaMemcpyDeviceToHost, h->stream));
    return augsched_sync(h);
  }
  return AUGSCHED_OK;
}

int augsched_enqueue(augsched_t* h, uint32_t instance, const augsched_record_soa* recs, uint32_t n,
                     int recs_on_device) {
  if (!h || !recs) return fail(AUGSCHED_E_INVALID, "enqueue: NULL argument");
  if (instance >= h->n_inst) return fail(AUGSCHED_E_INVALID, "enqueue: bad instance %u", instance);
  CUDA_TRY(cudaSetDevice(h->device));
  int rc = step_ensure(h->st, h->n_inst, h->max_active, h->stream, h->cfg, h->d_ip, &h->launches);
  if (rc) return rc;
  return step_enqueue(h->st, instance, recs, n, recs_on_device, h->stream, h->d_err, &h->launches);
}

// Iteration indices are stored as u32 last-scheduled times (R14), so `now`
// must be < 2^32, and time must not run backwards (Eq.26's wait now - last
// is unsigned).
static int check_now(augsched_t* h, uint64_t now, const char* who) {
  if (now >= (1ull << 32)) return fail(AUGSCHED_E_INVALID, "%s: now_iter %llu >= 2^32", who, (unsigned long long)now);
  if (h->st.have_now && now < h->st.last_now)
    return fail(AUGSCHED_E_INVALID, "%s: now_iter %llu < previous %llu", who, (unsigned long long)now,
                (unsigned long long)h->st.last_now);
  h->st.have_now = true;
  h->st.last_now = now;
  return AUGSCHED_OK;
}

int augsched_step_prefix(augsched_t* h, uint64_t now_iter, augsched_step_out* out) {
  if (!h || !out) return fail(AUGSCHED_E_INVALID, "step_prefix: NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  int rc = step_ensure(h->st, h->n_inst, h->max_active, h->stream, h->cfg, h->d_ip, &h->launches);
  if (rc) return rc;
  if ((rc = check_now(h, now_iter, "step_prefix"))) return rc;
  return step_run_prefix(h->st, h->cfg, h->cap, h->d_ip, h->d_err, now_iter, out, h->stream, &h->launches);
}

int augsched_step(augsched_t* h, uint64_t now_iter, augsched_step_out* out) {
  if (!h || !out) return fail(AUGSCHED_E_INVALID, "step: NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  int rc = step_ensure(h->st, h->n_inst, h->max_active, h->stream, h->cfg, h->d_ip, &h->launches);
  if (rc) return rc;
  if ((rc = check_now(h, now_iter, "step"))) return rc;
  return step_run(h->st, h->cfg, h->cap, h->d_ip, h->d_err, now_iter, out, h->stream, &h->launches);
}

int augsched_step_export(augsched_t* h, uint32_t instance, int32_t* slots, int64_t* ledger) {
  if (!h) return fail(AUGSCHED_E_INVALID, "step_export: NULL handle");
  if (instance >= h->n_inst) return fail(AUGSCHED_E_INVALID, "step_export: bad instance %u", instance);
  CUDA_TRY(cudaSetDevice(h->device));
  int rc = step_ensure(h->st, h->n_inst, h->max_active, h->stream, h->cfg, h->d_ip, &h->launches);
  if (rc) return rc;
  const uint32_t MA = h->max_active;
  const size_t off = (size_t)instance * MA;
  if (slots) {
    std::vector<uint32_t> st(MA);
    std::vector<int32_t> ctx(MA), kv(MA), cpu(MA), pend(MA);
    CUDA_TRY(cudaMemcpyAsync(st.data(), h->st.st + off, 4 * (size_t)MA, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx.data(), h->st.ctx + off, 4 * (size_t)MA, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaMemcpyAsync(kv.data(), h->st.kv + off, 4 * (size_t)MA, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaMemcpyAsync(cpu.data(), h->st.cpu + off, 4 * (size_t)MA, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaMemcpyAsync(pend.data(), h->st.pend + off, 4 * (size_t)MA, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    for (uint32_t x = 0; x < MA; ++x) {
      const uint32_t sv = st[x] & 15;
      slots[6 * (size_t)x + 0] = (int32_t)sv;
      slots[6 * (size_t)x + 1] = sv == ST_NONE ? AUGSCHED_DISCARD : (int32_t)((st[x] >> 4) & 3);
      slots[6 * (size_t)x + 2] = ctx[x];
      slots[6 * (size_t)x + 3] = kv[x];
      slots[6 * (size_t)x + 4] = cpu[x];
      slots[6 * (size_t)x + 5] = pend[x];
    }
  }
  if (ledger) {
    long long ap[2];
    CUDA_TRY(cudaMemcpyAsync(&ap[0], h->st.A + instance, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaMemcpyAsync(&ap[1], h->st.P + instance, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    ledger[0] = ap[0];
    ledger[1] = ap[1];
  }
  return AUGSCHED_OK;   // a latched device fault is left for augsched_sync
}

uint64_t augsched_shard_offer_bytes(const augsched_t* h) {
  return h ? (uint64_t)step_shard_offer_bytes(h->st) : 0ull;
}

int augsched_shard_begin(augsched_t* h, uint64_t now_iter, int64_t* ledger) {
  if (!h || !ledger) return fail(AUGSCHED_E_INVALID, "shard_begin: NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  int rc = step_ensure(h->st, h->n_inst, h->max_active, h->stream, h->cfg, h->d_ip, &h->launches);
  if (rc) return rc;
  if ((rc = check_now(h, now_iter, "shard_begin"))) return rc;
  h->st.shard_ledger = nullptr;
  return step_shard_begin(h->st, h->d_ip, h->d_err, now_iter, ledger, h->stream, &h->launches);
}

int augsched_shard_offer(augsched_t* h, const int64_t* ledger_sum, void* offer) {
  if (!h || !ledger_sum || !offer) return fail(AUGSCHED_E_INVALID, "shard_offer: NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  return step_shard_offer(h->st, h->cfg, h->cap, h->d_ip, h->d_err, ledger_sum, offer, h->stream, &h->launches);
}

int augsched_shard_commit(augsched_t* h, const void* offers, uint32_t n_ranks, uint32_t rank,
                          augsched_step_out* out) {
  if (!h || !offers || !out) return fail(AUGSCHED_E_INVALID, "shard_commit: NULL argument");
  if (!h->st.shard_ledger) return fail(AUGSCHED_E_INVALID, "shard_commit: no shard_offer in this step");
  CUDA_TRY(cudaSetDevice(h->device));
  const int rc = step_shard_commit(h->st, h->cfg, h->cap, h->d_ip, h->d_err, h->st.shard_ledger, offers, n_ranks,
                                   rank, out, h->stream, &h->launches);
  h->st.shard_ledger = nullptr;
  return rc;
}

}  // extern "C"

// error helper shared with step.cu
namespace augsched {
int set_error(int code, const char* msg) { return fail(code, "%s", msg); }
}  // namespace augsched
