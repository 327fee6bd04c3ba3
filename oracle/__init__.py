"""ctypes wrapper of the CPU oracle (oracle/augsched_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2512_04013_b200) never imports this module and shares no code with it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "augsched_oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")

FIELDS = [
    "n_requests", "arrived", "completed", "slo_ok", "slo_ok_5x", "busy_steps", "decisions",
    "evictions", "demotions", "calls_preserve", "calls_swap", "calls_discard", "returns",
    "tokens_granted", "final_t", "makespan_iter", "sum_ttft_ticks", "sum_e2e_ticks",
    "sum_gen_tokens", "admitted", "err", "max_queue", "incomplete", "rsv23",
]
NBIN = 160
PRESERVE, SWAP, DISCARD = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (no FMA contraction, R3).  The environment
    variable AUGSCHED_ORACLE_LIB names a prebuilt library to load instead
    (tools/oracle_mutants.py uses it to run the pins against mutants)."""
    alt = os.environ.get("AUGSCHED_ORACLE_LIB")
    if alt:
        return alt
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call([
            "g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
            "-shared", "-pthread", "-o", LIB, SRC])
    return LIB


class OCfg(C.Structure):
    _fields_ = [("m_per_token", C.c_uint64), ("g_total", C.c_uint64), ("g_model", C.c_uint64),
                ("g_runtime", C.c_uint64), ("g_safety", C.c_uint64), ("t_fwd_ticks", C.c_uint64),
                ("s_in", C.c_uint32), ("s_out", C.c_uint32), ("gamma_num", C.c_uint32),
                ("gamma_den", C.c_uint32), ("beta_low", C.c_double), ("beta_high", C.c_double)]


class OInst(C.Structure):
    _fields_ = [("target_max", C.c_uint32), ("l_static", C.c_uint32), ("alpha", C.c_double),
                ("slo_ttft_ticks", C.c_uint64), ("slo_norm_num", C.c_uint32),
                ("slo_norm_den", C.c_uint32), ("ranking", C.c_uint32),
                ("budget_mode", C.c_uint32), ("policy_mode", C.c_uint32), ("rank_seed", C.c_uint32)]


class OTrace(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "req_off", "arr_tick", "l_pre", "seg_off", "n_seg", "gen_true", "gen_pred",
        "dur_true", "dur_pred", "ret_len")]


RESULT_DTYPE = np.dtype([("f", np.uint64, (len(FIELDS),)), ("hist_ttft", np.uint32, (NBIN,)),
                         ("hist_norm", np.uint32, (NBIN,))])

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.oracle_simulate.argtypes = [C.POINTER(OCfg), C.c_void_p, C.c_uint32, C.POINTER(OTrace),
                                      C.c_void_p, C.c_uint64, C.c_void_p, C.c_int]
        L.oracle_simulate.restype = C.c_int
        cfgp = C.POINTER(OCfg)
        L.oracle_waste.argtypes = [cfgp, C.c_uint32, C.c_int, C.c_uint64, C.c_double, C.c_uint64]
        L.oracle_waste.restype = C.c_double
        L.oracle_select_policy.argtypes = [cfgp, C.c_uint32, C.c_uint64, C.c_double, C.c_uint64,
                                           C.c_uint32]
        L.oracle_select_policy.restype = C.c_int
        L.oracle_stage1.argtypes = [cfgp, C.c_uint32, C.c_uint64, C.c_uint64, C.c_double, C.c_int]
        L.oracle_stage1.restype = C.c_double
        L.oracle_stage2.argtypes = [cfgp, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        L.oracle_stage2.restype = C.c_double
        L.oracle_final.argtypes = [cfgp, C.c_uint32, C.c_double, C.c_uint64, C.c_int, C.c_double]
        L.oracle_final.restype = C.c_double
        L.oracle_key.argtypes = [C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_uint64]
        L.oracle_key.restype = C.c_uint32
        L.oracle_budget.argtypes = [cfgp, C.c_uint32, C.c_int64, C.c_int64]
        L.oracle_budget.restype = C.c_int64
        L.oracle_cap.argtypes = [cfgp]
        L.oracle_cap.restype = C.c_int64
        L.oracle_hist_bin.argtypes = [C.c_uint64]
        L.oracle_hist_bin.restype = C.c_uint32
        L.oracle_result_size.restype = C.c_uint32
        L.oracle_splitmix64_mix.argtypes = [C.c_uint64]
        L.oracle_splitmix64_mix.restype = C.c_uint64
        L.oracle_random_key.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64]
        L.oracle_random_key.restype = C.c_uint32
        assert L.oracle_result_size() == RESULT_DTYPE.itemsize
    return _lib


def make_cfg(d: dict) -> OCfg:
    return OCfg(**{k: d[k] for k, _ in OCfg._fields_})


def make_inst(p: dict) -> np.ndarray:
    """Per-instance parameter arrays -> contiguous OInst array."""
    n = len(p["target_max"])
    arr = (OInst * n)()
    for i in range(n):
        arr[i] = OInst(int(p["target_max"][i]), int(p["l_static"][i]), float(p["alpha"][i]),
                       int(p["slo_ttft_ticks"][i]), int(p["slo_norm_num"][i]),
                       int(p["slo_norm_den"][i]), int(p["ranking"][i]),
                       int(p["budget_mode"][i]), int(p["policy_mode"][i]),
                       int(p["rank_seed"][i]) if "rank_seed" in p else 0)
    return arr


def _trace_struct(tr):
    a = tr.arrays()
    keep = {k: np.ascontiguousarray(v) for k, v in a.items()}
    s = OTrace(**{k: v.ctypes.data for k, v in keep.items()})
    return s, keep


def simulate(cfg: dict, inst: dict, traces, inst_trace_id, max_iters: int = 2**62,
             threads: int | None = None) -> np.ndarray:
    """Run Algorithm 1 for every instance; returns a RESULT_DTYPE array."""
    L = lib()
    c = make_cfg(cfg)
    ip = make_inst(inst)
    n = len(ip)
    tid = np.ascontiguousarray(inst_trace_id, np.uint32)
    assert tid.shape[0] == n
    ts, keep = _trace_struct(traces)
    out = np.zeros(n, RESULT_DTYPE)
    if threads is None:
        threads = os.cpu_count() or 1
    rc = L.oracle_simulate(C.byref(c), C.cast(ip, C.c_void_p), n, C.byref(ts), tid.ctypes.data,
                           int(max_iters), out.ctypes.data, int(threads))
    assert rc == 0
    del keep
    return out


def simulate_detail(cfg: dict, inst: dict, traces, trace_id: int = 0, max_iters: int = 2**62):
    """One instance (inst arrays of length 1); returns (record dict, ft, fin)
    with per-request first-token and finish iterations (-1 if none)."""
    L = lib()
    L.oracle_simulate_detail.argtypes = [C.POINTER(OCfg), C.c_void_p, C.POINTER(OTrace), C.c_uint32,
                                         C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
    c = make_cfg(cfg)
    ip = make_inst(inst)
    ts, keep = _trace_struct(traces)
    n = traces.trace_len(trace_id)
    ft = np.zeros(n, np.int64)
    fin = np.zeros(n, np.int64)
    out = np.zeros(1, RESULT_DTYPE)
    L.oracle_simulate_detail(C.byref(c), C.cast(ip, C.c_void_p), C.byref(ts), trace_id,
                             int(max_iters), out.ctypes.data, ft.ctypes.data, fin.ctypes.data)
    del keep
    return as_dict(out[0]), ft, fin


def as_dict(rec) -> dict:
    d = {name: int(rec["f"][i]) for i, name in enumerate(FIELDS)}
    d["hist_ttft"] = rec["hist_ttft"].copy()
    d["hist_norm"] = rec["hist_norm"].copy()
    return d


# ---- formula entry points ---------------------------------------------------
def waste(cfg, target_max, pol, C_, Ti, Co):
    return lib().oracle_waste(C.byref(make_cfg(cfg)), target_max, pol, C_, Ti, Co)


def select_policy(cfg, target_max, C_, Ti, Co, policy_mode=0):
    return lib().oracle_select_policy(C.byref(make_cfg(cfg)), target_max, C_, Ti, Co, policy_mode)


def stage1(cfg, target_max, L, O, A, pol):
    return lib().oracle_stage1(C.byref(make_cfg(cfg)), target_max, L, O, A, pol)


def stage2(cfg, target_max, Lt, R, O, pol):
    return lib().oracle_stage2(C.byref(make_cfg(cfg)), target_max, Lt, R, O, pol)


def final(cfg, target_max, V2, X, next_pol, An):
    return lib().oracle_final(C.byref(make_cfg(cfg)), target_max, V2, X, next_pol, An)


def key(V, alpha, Ts, now, last):
    return lib().oracle_key(V, alpha, Ts, now, last)


def splitmix64_mix(z):
    return lib().oracle_splitmix64_mix(z)


def random_key(seed, id_, t):
    return lib().oracle_random_key(seed, id_, t)


def budget(cfg, target_max, A, P):
    return lib().oracle_budget(C.byref(make_cfg(cfg)), target_max, A, P)


def cap(cfg):
    return lib().oracle_cap(C.byref(make_cfg(cfg)))


def hist_bin(v):
    return lib().oracle_hist_bin(v)


# ---- step mode ----------------------------------------------------------------
K_NEW, K_RETURN, K_CALL, K_FINISH, K_IMPORT = 1, 2, 3, 4, 5
REC_FIELDS = ("kind", "id", "la", "lb", "lc", "ta", "flags", "last", "ctx", "kv", "cpu", "pend")


def records(n: int, **cols) -> dict:
    """SoA record block of length n (missing columns are zero)."""
    out = {}
    for f in REC_FIELDS:
        dt = np.float32 if f == "ta" else np.uint32
        v = cols.get(f, 0)
        out[f] = np.ascontiguousarray(np.broadcast_to(np.asarray(v, dt), (n,)).astype(dt))
    return out


class Step:
    """Oracle of augsched_step: per-instance scheduler state + one step."""

    def __init__(self, cfg: dict, inst: dict, max_active: int):
        L = lib()
        L.oracle_step_create.restype = C.c_void_p
        L.oracle_step_create.argtypes = [C.POINTER(OCfg), C.c_void_p, C.c_uint32, C.c_uint32]
        L.oracle_step_destroy.argtypes = [C.c_void_p]
        L.oracle_step_enqueue.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32] + [C.c_void_p] * 12
        L.oracle_step.argtypes = [C.c_void_p, C.c_uint64] + [C.c_void_p] * 7
        L.oracle_step_ledger.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]
        self.L = L
        self.cfg = make_cfg(cfg)
        ip = make_inst(inst)
        self.n_inst = len(ip)
        self.max_active = max_active
        self.h = L.oracle_step_create(C.byref(self.cfg), C.cast(ip, C.c_void_p), self.n_inst,
                                      max_active)

    def close(self):
        if self.h:
            self.L.oracle_step_destroy(self.h)
            self.h = None

    __del__ = close

    def enqueue(self, inst: int, rec: dict) -> int:
        n = len(rec["kind"])
        cols = [rec[f] for f in ("kind", "id", "la", "lb", "lc", "ta", "flags", "last", "ctx",
                                 "kv", "cpu", "pend")]
        return self.L.oracle_step_enqueue(self.h, inst, n, *[c.ctypes.data for c in cols])

    def step(self, now: int):
        n, m = self.n_inst, self.max_active
        B = np.zeros(n, np.int64)
        na = np.zeros(n, np.uint32)
        adm = np.zeros(n, np.uint32)
        order = np.zeros(n * m, np.uint32)
        grant = np.zeros(n * m, np.uint32)
        keys = np.zeros(n * m, np.uint32)
        toff = np.zeros(3 * n, np.uint32)
        rc = self.L.oracle_step(self.h, now, B.ctypes.data, na.ctypes.data, adm.ctypes.data,
                                order.ctypes.data, grant.ctypes.data, keys.ctypes.data, toff.ctypes.data)
        return dict(rc=rc, B=B, n_active=na, admitted=adm, order=order.reshape(n, m),
                    grant=grant.reshape(n, m), keys=keys.reshape(n, m), tier_off=toff.reshape(n, 3))

    def slots(self, inst: int) -> np.ndarray:
        """[max_active, 6] int32: status, policy, ctx, kv, cpu, pend."""
        self.L.oracle_step_slots_all.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        out = np.zeros((self.max_active, 6), np.int32)
        self.L.oracle_step_slots_all(self.h, inst, out.ctypes.data)
        return out

    def ledger(self, inst: int):
        A = C.c_int64()
        P = C.c_int64()
        self.L.oracle_step_ledger(self.h, inst, C.byref(A), C.byref(P))
        return A.value, P.value
