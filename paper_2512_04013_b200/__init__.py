"""augsched: B200-native AugServe scheduler hot path (arXiv 2512.04013).

Thin Python binding over the C ABI of libaugsched.so (include/augsched.h):
argument marshalling only.  Every step of the scheduling path runs in the
library's sm_100a kernels; PyTorch supplies device memory, the CUDA stream and
(for multi-GPU runs) torch.distributed.  There is no CPU fallback: if the
shared library or a CUDA device is missing, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libaugsched.so")

OK, E_INVALID, E_CAPACITY, E_CUDA, E_STATE, E_OOM, E_UNIMPLEMENTED = 0, -1, -2, -3, -4, -5, -6
HOST_TRACES, HOST_RESULTS, RESUME = 1, 2, 4
K_NEW, K_RETURN, K_CALL, K_FINISH, K_IMPORT = 1, 2, 3, 4, 5

RESULT_FIELDS = [
    "n_requests", "arrived", "completed", "slo_ok", "slo_ok_5x", "busy_steps", "decisions",
    "evictions", "demotions", "calls_preserve", "calls_swap", "calls_discard", "returns",
    "tokens_granted", "final_t", "makespan_iter", "sum_ttft_ticks", "sum_e2e_ticks",
    "sum_gen_tokens", "admitted", "err", "max_queue", "incomplete", "rsv23",
]
NBIN = 160
RESULT_DTYPE = np.dtype([("f", np.uint64, (len(RESULT_FIELDS),)), ("hist_ttft", np.uint32, (NBIN,)),
                         ("hist_norm", np.uint32, (NBIN,))])
EXPORTS = ["augsched_create", "augsched_enqueue", "augsched_step", "augsched_step_prefix", "augsched_simulate",
           "augsched_generate", "augsched_step_export", "augsched_shard_offer_bytes", "augsched_shard_begin",
           "augsched_shard_offer", "augsched_shard_commit",
           "augsched_sync", "augsched_launch_count", "augsched_destroy", "augsched_last_error"]


class InstanceParams(C.Structure):
    _fields_ = [("target_max", C.c_uint32), ("l_static", C.c_uint32), ("alpha", C.c_double),
                ("slo_ttft_ticks", C.c_uint64), ("slo_norm_num", C.c_uint32),
                ("slo_norm_den", C.c_uint32), ("ranking", C.c_uint32), ("budget_mode", C.c_uint32),
                ("policy_mode", C.c_uint32), ("rank_seed", C.c_uint32)]


class Config(C.Structure):
    _fields_ = [("m_per_token", C.c_uint64), ("g_total", C.c_uint64), ("g_model", C.c_uint64),
                ("g_runtime", C.c_uint64), ("g_safety", C.c_uint64), ("t_fwd_ticks", C.c_uint64),
                ("s_in", C.c_uint32), ("s_out", C.c_uint32), ("gamma_num", C.c_uint32),
                ("gamma_den", C.c_uint32), ("beta_low", C.c_double), ("beta_high", C.c_double),
                ("defaults", InstanceParams)]


class Trace(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("req_off", "arr_tick", "l_pre", "seg_off", "n_seg",
                                          "gen_true", "gen_pred", "dur_true", "dur_pred", "ret_len")] + \
               [("n_traces", C.c_uint32), ("n_req", C.c_uint32), ("n_seg_total", C.c_uint32),
                ("reserved", C.c_uint32)]


class RecordSoA(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("kind", "id", "la", "lb", "lc", "ta", "flags", "last",
                                          "ctx", "kv", "cpu", "pend")]


class GenTables(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("gap", "prompt", "gen", "dur", "ret", "noise")] + \
               [("cls_th", C.c_uint32 * 3), ("calls_lo", C.c_uint32 * 4), ("calls_hi", C.c_uint32 * 4),
                ("edges", C.c_uint32 * 8), ("mids", C.c_uint32 * 8), ("acc_th", C.c_uint32),
                ("nocall_th", C.c_uint32), ("oracle_pred", C.c_uint32), ("reserved", C.c_uint32)]


class GenSpec(C.Structure):
    _fields_ = [("seed", C.c_uint32), ("n_traces", C.c_uint32), ("n_max", C.c_uint32),
                ("reserved", C.c_uint32), ("horizon_ticks", C.c_uint64), ("scale", C.c_void_p)]


class StepOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("budget", "n_active", "admitted", "order", "grant", "key",
                                          "tier_off")]


_lib = None


def lib():
    """Load libaugsched.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        # AUGSCHED_LIB: another build of this library (the AUGSCHED_DEBUG
        # variant, _build.build_debug); there is no fallback of any kind
        path = os.environ.get("AUGSCHED_LIB", LIB_PATH)
        if not os.path.exists(path):
            raise RuntimeError(f"libaugsched.so not built at {path}; run __graft_entry__.build()")
        L = C.CDLL(path)
        vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
        L.augsched_create.argtypes = [C.POINTER(Config), vp, u32, u32, C.c_int, vp, C.POINTER(vp)]
        L.augsched_enqueue.argtypes = [vp, u32, C.POINTER(RecordSoA), u32, C.c_int]
        L.augsched_step.argtypes = [vp, u64, C.POINTER(StepOut)]
        L.augsched_step_prefix.argtypes = [vp, u64, C.POINTER(StepOut)]
        L.augsched_simulate.argtypes = [vp, C.POINTER(Trace), vp, u64, vp, u32]
        L.augsched_generate.argtypes = [vp, C.POINTER(GenSpec), C.POINTER(GenTables), C.POINTER(Trace), u32, u32]
        L.augsched_generate.restype = C.c_int
        L.augsched_sync.argtypes = [vp]
        L.augsched_step_export.argtypes = [vp, u32, vp, vp]
        L.augsched_step_export.restype = C.c_int
        L.augsched_shard_offer_bytes.argtypes = [vp]
        L.augsched_shard_offer_bytes.restype = u64
        L.augsched_shard_begin.argtypes = [vp, u64, vp]
        L.augsched_shard_begin.restype = C.c_int
        L.augsched_shard_offer.argtypes = [vp, vp, vp]
        L.augsched_shard_offer.restype = C.c_int
        L.augsched_shard_commit.argtypes = [vp, vp, u32, u32, C.POINTER(StepOut)]
        L.augsched_shard_commit.restype = C.c_int
        L.augsched_launch_count.argtypes = [vp]
        L.augsched_launch_count.restype = u64
        L.augsched_destroy.argtypes = [vp]
        L.augsched_destroy.restype = None
        L.augsched_last_error.restype = C.c_char_p
        for f in (L.augsched_create, L.augsched_enqueue, L.augsched_step, L.augsched_step_prefix,
                  L.augsched_simulate,
                  L.augsched_sync):
            f.restype = C.c_int
        _lib = L
    return _lib


class AugschedError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"augsched error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != OK:
        raise AugschedError(rc, lib().augsched_last_error().decode())
    return rc


def make_config(cfg: dict, defaults: dict | None = None) -> Config:
    c = Config()
    for k, _ in Config._fields_:
        if k != "defaults":
            setattr(c, k, cfg[k])
    if defaults is not None:
        c.defaults = _params_struct(defaults)
    return c


def _params_struct(d: dict) -> InstanceParams:
    return InstanceParams(int(d["target_max"]), int(d["l_static"]), float(d["alpha"]),
                          int(d["slo_ttft_ticks"]), int(d["slo_norm_num"]), int(d["slo_norm_den"]),
                          int(d["ranking"]), int(d["budget_mode"]), int(d["policy_mode"]),
                          int(d.get("rank_seed", 0)))


def params_array(p: dict):
    """Per-instance parameter arrays (dict of length-n arrays) -> ctypes array."""
    n = len(p["target_max"])
    arr = (InstanceParams * n)()
    for i in range(n):
        arr[i] = _params_struct({k: v[i] for k, v in p.items()})
    return arr


def _torch():
    import torch
    return torch


class DeviceTraces:
    """A trace set resident in device memory (torch tensors)."""

    _names = ("req_off", "arr_tick", "l_pre", "seg_off", "n_seg", "gen_true", "gen_pred",
              "dur_true", "dur_pred", "ret_len")

    def __init__(self, traces, device="cuda"):
        torch = _torch()
        self.t = {}
        for k in self._names:
            a = np.ascontiguousarray(getattr(traces, k))
            if a.dtype == np.uint64:
                a = a.view(np.int64)
            elif a.dtype == np.uint32:
                a = a.view(np.int32)
            self.t[k] = torch.from_numpy(a.copy()).to(device)
        self.n_traces = int(traces.req_off.shape[0] - 1)
        self.n_req = int(traces.arr_tick.shape[0])
        self.n_seg_total = int(traces.gen_true.shape[0])

    def struct(self) -> Trace:
        s = Trace(**{k: self.t[k].data_ptr() for k in DeviceTraces._names})
        s.n_traces, s.n_req, s.n_seg_total = self.n_traces, self.n_req, self.n_seg_total
        return s


class GeneratedTraces(DeviceTraces):
    """A trace set drawn on the device by augsched_generate (the table-driven
    W1/W2/W3 generator; tracegen/tablegen.py is its host twin).  `tables` is
    the dict of tracegen.tablegen.build_tables (inputs only)."""

    def __init__(self, sched, tables: dict, seed: int, n_traces: int, n_max: int, rates,
                 horizon_ticks: int = 0, device="cuda"):
        torch = _torch()
        rates = list(rates) if hasattr(rates, "__len__") else [rates]
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
        self._tb = {k: dev(tables[k].view(np.int32) if tables[k].dtype == np.uint32 else tables[k])
                    for k in ("gap", "prompt", "gen", "dur", "ret", "noise")}
        self._scale = dev(np.array([1e6 / float(rates[k % len(rates)]) for k in range(n_traces)], np.float64))
        max_calls = int(np.max(tables["calls_hi"]))
        req_cap = n_traces * n_max
        seg_cap = req_cap * (max_calls + 1)
        i32 = dict(dtype=torch.int32, device=device)
        self.t = dict(req_off=torch.empty(n_traces + 1, **i32),
                      arr_tick=torch.empty(req_cap, dtype=torch.int64, device=device),
                      l_pre=torch.empty(req_cap, **i32), seg_off=torch.empty(req_cap, **i32),
                      n_seg=torch.empty(req_cap, **i32), gen_true=torch.empty(seg_cap, **i32),
                      gen_pred=torch.empty(seg_cap, **i32), dur_true=torch.empty(seg_cap, **i32),
                      dur_pred=torch.empty(seg_cap, dtype=torch.float32, device=device),
                      ret_len=torch.empty(seg_cap, **i32))
        tb = GenTables(**{k: v.data_ptr() for k, v in self._tb.items()})
        for k in ("cls_th", "calls_lo", "calls_hi", "edges", "mids"):
            getattr(tb, k)[:] = [int(x) for x in tables[k]]
        tb.acc_th, tb.nocall_th = int(tables["acc_th"]), int(tables["nocall_th"])
        tb.oracle_pred = int(tables["oracle_pred"])
        spec = GenSpec(int(seed), int(n_traces), int(n_max), 0, int(horizon_ticks), self._scale.data_ptr())
        out = Trace(**{k: self.t[k].data_ptr() for k in DeviceTraces._names})
        _check(sched.L.augsched_generate(sched.h, C.byref(spec), C.byref(tb), C.byref(out), req_cap, seg_cap))
        self.n_traces, self.n_req, self.n_seg_total = n_traces, int(out.n_req), int(out.n_seg_total)

    def to_numpy(self):
        """Copy the generated arrays to host numpy (same dtypes as tracegen.Traces)."""
        u = lambda x, n: x[:n].cpu().numpy()
        nr, ns = self.n_req, self.n_seg_total
        return dict(req_off=u(self.t["req_off"], self.n_traces + 1).view(np.uint32),
                    arr_tick=u(self.t["arr_tick"], nr).view(np.uint64),
                    l_pre=u(self.t["l_pre"], nr).view(np.uint32), seg_off=u(self.t["seg_off"], nr).view(np.uint32),
                    n_seg=u(self.t["n_seg"], nr).view(np.uint32), gen_true=u(self.t["gen_true"], ns).view(np.uint32),
                    gen_pred=u(self.t["gen_pred"], ns).view(np.uint32),
                    dur_true=u(self.t["dur_true"], ns).view(np.uint32), dur_pred=u(self.t["dur_pred"], ns),
                    ret_len=u(self.t["ret_len"], ns).view(np.uint32))


class PinnedTraces:
    """A trace set in page-locked host memory (for the end-to-end path)."""

    def __init__(self, traces):
        torch = _torch()
        self.t = {}
        for k in DeviceTraces._names:
            a = np.ascontiguousarray(getattr(traces, k))
            if a.dtype == np.uint64:
                a = a.view(np.int64)
            elif a.dtype == np.uint32:
                a = a.view(np.int32)
            self.t[k] = torch.from_numpy(a.copy()).pin_memory()
        self.n_traces = int(traces.req_off.shape[0] - 1)
        self.n_req = int(traces.arr_tick.shape[0])
        self.n_seg_total = int(traces.gen_true.shape[0])
        self.nbytes = int(sum(v.numel() * v.element_size() for v in self.t.values()))

    struct = DeviceTraces.struct


def host_trace_struct(traces):
    if isinstance(traces, PinnedTraces):
        return traces.struct(), None
    keep = {k: np.ascontiguousarray(getattr(traces, k)) for k in DeviceTraces._names}
    s = Trace(**{k: v.ctypes.data for k, v in keep.items()})
    s.n_traces = int(traces.req_off.shape[0] - 1)
    s.n_req = int(traces.arr_tick.shape[0])
    s.n_seg_total = int(traces.gen_true.shape[0])
    return s, keep


class Scheduler:
    """One libaugsched handle: n_instances independent serving instances."""

    def __init__(self, cfg: dict, inst: dict | None, n_instances: int, max_active: int,
                 device: int = 0, stream=None, defaults: dict | None = None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("augsched needs a CUDA device (no CPU fallback)")
        self.L = lib()
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self.n_instances = n_instances
        self.max_active = max_active
        self._cfg = make_config(cfg, defaults if defaults is not None else
                                (None if inst is None else {k: v[0] for k, v in inst.items()}))
        self._ip = params_array(inst) if inst is not None else None
        h = C.c_void_p()
        _check(self.L.augsched_create(C.byref(self._cfg), C.cast(self._ip, C.c_void_p) if self._ip else None,
                                      n_instances, max_active, device,
                                      C.c_void_p(stream.cuda_stream), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.augsched_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.L.augsched_launch_count(self.h))

    def sync(self):
        _check(self.L.augsched_sync(self.h))

    # ---- simulate ------------------------------------------------------------
    def simulate(self, traces, inst_trace_id, max_iters: int = 2**32, out=None, resume=False):
        """Device path: traces is a DeviceTraces, inst_trace_id a device int32
        tensor; returns (and fills) a device uint8 tensor of result records.
        Asynchronous on the handle's stream."""
        torch = _torch()
        if out is None:
            out = torch.empty(self.n_instances * RESULT_DTYPE.itemsize, dtype=torch.uint8,
                              device=f"cuda:{self.device}")
        ts = traces.struct()
        flags = RESUME if resume else 0
        _check(self.L.augsched_simulate(self.h, C.byref(ts), C.c_void_p(inst_trace_id.data_ptr()),
                                        int(max_iters), C.c_void_p(out.data_ptr()), flags))
        return out

    def simulate_host(self, traces, inst_trace_id, max_iters: int = 2**32, resume=False):
        """End-to-end path: host trace arrays in, host result records out (the
        library stages the copies; the call synchronizes)."""
        ts, keep = host_trace_struct(traces)
        tid = np.ascontiguousarray(inst_trace_id, np.uint32)
        res = np.zeros(self.n_instances, RESULT_DTYPE)
        flags = HOST_TRACES | HOST_RESULTS | (RESUME if resume else 0)
        _check(self.L.augsched_simulate(self.h, C.byref(ts), C.c_void_p(tid.ctypes.data),
                                        int(max_iters), C.c_void_p(res.ctypes.data), flags))
        del keep
        return res

    # ---- step mode -------------------------------------------------------------
    def enqueue(self, instance: int, rec: dict):
        """rec: dict of equal-length numpy arrays (host) with the record fields."""
        n = len(rec["kind"])
        keep = {}
        for f, _ in RecordSoA._fields_:
            dt = np.float32 if f == "ta" else np.uint32
            keep[f] = np.ascontiguousarray(np.broadcast_to(np.asarray(rec.get(f, 0), dt), (n,)).astype(dt))
        s = RecordSoA(**{k: v.ctypes.data for k, v in keep.items()})
        _check(self.L.augsched_enqueue(self.h, instance, C.byref(s), n, 0))

    def step(self, now: int, prefix: bool = False) -> StepOut:
        """One decision round (augsched_step); prefix=True calls
        augsched_step_prefix (order/key/grant only for the admitted prefix)."""
        out = StepOut()
        f = self.L.augsched_step_prefix if prefix else self.L.augsched_step
        _check(f(self.h, int(now), C.byref(out)))
        return out

    def slots(self, instance: int) -> np.ndarray:
        """[max_active, 6] int32 slot state (augsched_step_export): status,
        policy, ctx, kv, cpu, pend -- the layout of oracle.Step.slots()."""
        out = np.zeros((self.max_active, 6), np.int32)
        _check(self.L.augsched_step_export(self.h, instance, C.c_void_p(out.ctypes.data), None))
        return out

    def ledger(self, instance: int):
        """(A, P) of an instance (augsched_step_export)."""
        ap = np.zeros(2, np.int64)
        _check(self.L.augsched_step_export(self.h, instance, None, C.c_void_p(ap.ctypes.data)))
        return int(ap[0]), int(ap[1])

    # ---- sharded single queue (f4): the three calls of one step; the caller
    # runs the collectives (all-reduce of the ledger, all-gather of the offers)
    def shard_offer_bytes(self) -> int:
        return int(self.L.augsched_shard_offer_bytes(self.h))

    def shard_begin(self, now: int, ledger):
        """ledger: device int64 tensor [2] <- this shard's (A, P)."""
        _check(self.L.augsched_shard_begin(self.h, int(now), C.c_void_p(ledger.data_ptr())))

    def shard_offer(self, ledger_sum, offer):
        """ledger_sum: device int64 [2] (the all-reduced ledger); offer: device
        uint8 [shard_offer_bytes()] <- this shard's offer."""
        _check(self.L.augsched_shard_offer(self.h, C.c_void_p(ledger_sum.data_ptr()), C.c_void_p(offer.data_ptr())))

    def shard_commit(self, offers, n_ranks: int, rank: int) -> StepOut:
        """offers: device uint8, the rank-major all-gather of every shard's offer."""
        out = StepOut()
        _check(self.L.augsched_shard_commit(self.h, C.c_void_p(offers.data_ptr()), n_ranks, rank, C.byref(out)))
        return out

    def shard_result(self, out: StepOut) -> dict:
        """The global prefix of a committed step (synchronizes)."""
        self.sync()
        g = lambda ptr, cnt, dt: device_view(ptr, cnt, dt).cpu().numpy().copy()
        adm = int(g(out.admitted, 1, "<u4")[0])
        return dict(B=int(g(out.budget, 1, "<i8")[0]), n_active=int(g(out.n_active, 1, "<u4")[0]), admitted=adm,
                    order=g(out.order, adm, "<u4") if adm else np.zeros(0, np.uint32),
                    grant=g(out.grant, adm, "<u4") if adm else np.zeros(0, np.uint32),
                    keys=g(out.key, adm, "<u4") if adm else np.zeros(0, np.uint32))

    def step_result(self, out: StepOut) -> dict:
        """Copy one step's outputs to host numpy (synchronizes)."""
        n, m = self.n_instances, self.max_active
        self.sync()
        g = lambda ptr, cnt, dt: device_view(ptr, cnt, dt).cpu().numpy().copy()
        r = dict(B=g(out.budget, n, "<i8"), n_active=g(out.n_active, n, "<u4"),
                 admitted=g(out.admitted, n, "<u4"),
                 order=g(out.order, n * m, "<u4").reshape(n, m),
                 grant=g(out.grant, n * m, "<u4").reshape(n, m),
                 keys=g(out.key, n * m, "<u4").reshape(n, m))
        if out.tier_off:
            r["tier_off"] = g(out.tier_off, 3 * n, "<u4").reshape(n, 3)
        return r


class _CAI:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_view(ptr, n: int, typestr: str):
    """Zero-copy torch view of n elements at a device pointer owned by a handle."""
    torch = _torch()
    return torch.as_tensor(_CAI(ptr, n, typestr), device="cuda")


def results_to_numpy(dev_out) -> np.ndarray:
    """Device uint8 result tensor -> numpy RESULT_DTYPE array (synchronizes)."""
    return dev_out.cpu().numpy().view(RESULT_DTYPE).copy()


def as_dict(rec) -> dict:
    d = {name: int(rec["f"][i]) for i, name in enumerate(RESULT_FIELDS)}
    d["hist_ttft"] = rec["hist_ttft"].copy()
    d["hist_norm"] = rec["hist_norm"].copy()
    return d
