"""Parity runs against the AUGSCHED_DEBUG build (run with AUGSCHED_LIB set to
its path; tests/test_gpu_debug.py): simulate (cfg1-3 shapes, all ranking /
budget / policy modes, tight memory) and step streams (full order single and
batched, prefix) must equal the oracle with no invariant check firing."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import oracle  # noqa: E402
import tracegen  # noqa: E402
import paper_2512_04013_b200 as aug  # noqa: E402
from test_gpu_step import random_events, compare, compare_slots  # noqa: E402

assert os.environ.get("AUGSCHED_LIB", "").endswith("libaugsched_debug.so")
torch.cuda.set_device(0)
# simulate
tr = tracegen.gen_traces(4, 400, [2.0, 4.0, 6.0, 8.0], seed=12, p_nocall=0.1)
n = 4 * 8
tid = np.repeat(np.arange(4), 8).astype(np.uint32)
ip = tracegen.inst_params(n, ranking=[0, 1, 2, 0, 0, 0, 0, 0] * 4, budget_mode=[0, 0, 0, 1, 0, 0, 0, 0] * 4,
                          policy_mode=[0, 0, 0, 0, 1, 2, 3, 0] * 4, rank_seed=7,
                          target_max=[500, 500, 500, 500, 500, 500, 500, 120] * 4)
for cfg in (tracegen.PRESET_7B, dict(tracegen.PRESET_7B, g_total=tracegen.PRESET_7B["g_total"] // 2 + 6 * 2**30)):
    s = aug.Scheduler(cfg, ip, n, 400)
    g = s.simulate_host(tr, tid)
    s.close()
    o = oracle.simulate(cfg, ip, tr, tid)
    assert g.tobytes() == o.tobytes(), "simulate differs from the oracle"
# step streams
for n_inst, MA, prefix in ((1, 300, False), (1, 300, True), (4, 128, False), (4, 128, True)):
    rng = np.random.default_rng(n_inst * 7 + MA)
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 700, g_model=1000)
    ipx = tracegen.inst_params(n_inst, base=tracegen.INST_G0, budget_mode=0, target_max=120, alpha=1.5)
    st = oracle.Step(cfg, ipx, MA)
    s = aug.Scheduler(cfg, ipx, n_inst, MA)
    for t in range(25):
        for i in range(n_inst):
            rec = random_events(rng, st.slots(i), t, p_new=0.5 if t == 0 else 0.15)
            if rec is not None:
                st.enqueue(i, rec)
                s.enqueue(i, rec)
        o = st.step(t)
        gq = s.step_result(s.step(t, prefix=prefix))
        compare(gq, o, n_inst, f"debug n_inst={n_inst} MA={MA} prefix={prefix} t={t}", prefix=prefix)
        compare_slots(s, st, n_inst, "debug")
    s.sync()      # raises E_STATE if an invariant check fired
    s.close()
# kept orders (session 4): batched with every ranking, and a single queue
# whose waiting requests are re-ordered by fp32 rounding (the checked merge
# falls back to the sort) -- the debug build also checks each merged order
for n_inst, MA, rk in ((3, 400, [0, 1, 3]), (1, 400, [0])):
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 10**6, g_model=1000)
    ipx = tracegen.inst_params(n_inst, base=tracegen.INST_G0, ranking=rk, budget_mode=1, l_static=30,
                               alpha=1e-5)
    st = oracle.Step(cfg, ipx, MA)
    s = aug.Scheduler(cfg, ipx, n_inst, MA)
    for t in range(120):
        for i in range(n_inst):
            rec = oracle.records(1, kind=oracle.K_NEW, id=[MA - 1 - t], la=[100], lb=[10], ta=[0.0], flags=[0])
            st.enqueue(i, rec)
            s.enqueue(i, rec)
        o = st.step(t)
        gq = s.step_result(s.step(t))
        compare(gq, o, n_inst, f"debug kept order n_inst={n_inst} t={t}")
    s.sync()
    s.close()
print("debug parity ok")
