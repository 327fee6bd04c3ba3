"""Small invocations of every kernel of libaugsched, for compute-sanitizer
(memcheck / racecheck / synccheck; tools/sanitize.sh): simulate on a few
instances (one-warp instances, work stealing, resumable windows), the device
trace generator, and augsched_step / augsched_step_prefix on single- and
multi-instance handles (cooperative full step, batched shared-memory step,
the device-wide LSD path for large slot counts, both prefix kernels), with
random NEW/CALL/RETURN/FINISH events and tight memory so the resolution
paths run.  Every result is also compared with the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import oracle  # noqa: E402
import tracegen  # noqa: E402
from tracegen import tablegen as tg  # noqa: E402
import paper_2512_04013_b200 as aug  # noqa: E402
from test_gpu_step import random_events, compare  # noqa: E402

torch.cuda.set_device(0)
# simulate: 2 windows, small traces, tight memory for one preset
tr = tracegen.gen_traces(2, 120, [3.0, 6.0], seed=3)
ip = tracegen.inst_params(6, ranking=[0, 1, 2, 0, 0, 0], budget_mode=[0, 0, 0, 1, 0, 0],
                          policy_mode=[0, 0, 0, 0, 1, 3], rank_seed=5)
tid = np.array([0, 0, 1, 1, 0, 1], np.uint32)
s = aug.Scheduler(tracegen.PRESET_7B, ip, 6, 120)
s.simulate_host(tr, tid, max_iters=400)
g = s.simulate_host(tr, tid, max_iters=2**32, resume=True)
s.close()
assert g.tobytes() == oracle.simulate(tracegen.PRESET_7B, ip, tr, tid).tobytes()
# generator
T = tg.build_tables(cv=2.0)
probe = aug.Scheduler(tracegen.PRESET_7B, tracegen.inst_params(1), 1, 8)
gt = aug.GeneratedTraces(probe, T, 11, 2, 300, [2.0, 3.0], horizon_ticks=60 * 10**6)
probe.close()
# step paths
cases = [(1, 200, False), (1, 200, True), (3, 64, False), (3, 64, True), (2, 9000, False)]
for n_inst, MA, prefix in cases:
    rng = np.random.default_rng(MA + n_inst)
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 500, g_model=1000)
    ipx = tracegen.inst_params(n_inst, base=tracegen.INST_G0, budget_mode=0, target_max=100, alpha=1.5,
                               ranking=[0, 1, 2][:n_inst] if n_inst > 1 else 0, rank_seed=3)
    st = oracle.Step(cfg, ipx, MA)
    sc = aug.Scheduler(cfg, ipx, n_inst, MA)
    for t in range(6):
        for i in range(n_inst):
            rec = random_events(rng, st.slots(i), t, p_new=0.6 if t == 0 else 0.2)
            if rec is not None:
                st.enqueue(i, rec)
                sc.enqueue(i, rec)
        o = st.step(t)
        compare(sc.step_result(sc.step(t, prefix=prefix)), o, n_inst, f"sanitize {n_inst}x{MA} prefix={prefix}",
                prefix=prefix)
    sc.sync()
    sc.close()
# time-invariant keys: incremental full order over several steps
rng = np.random.default_rng(5)
cfg = dict(tracegen.PRESET_G0, g_total=1000 + 500, g_model=1000)
ipt = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=3, budget_mode=0, target_max=100, alpha=1.5)
st = oracle.Step(cfg, ipt, 600)
sc = aug.Scheduler(cfg, ipt, 1, 600)
for t in range(6):
    rec = random_events(rng, st.slots(0), t, p_new=0.6 if t == 0 else 0.1)
    if rec is not None:
        st.enqueue(0, rec)
        sc.enqueue(0, rec)
    compare(sc.step_result(sc.step(t)), st.step(t), 1, "sanitize ti")
sc.sync()
sc.close()
# sharded queue: 2 shards
G, MA = 2, 300
ips = tracegen.inst_params(1, base=tracegen.INST_G0, budget_mode=0, target_max=100, alpha=1.5)
st = oracle.Step(cfg, ips, G * MA)
hs = [aug.Scheduler(cfg, ips, 1, MA) for _ in range(G)]
ob = hs[0].shard_offer_bytes()
led = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(G)]
off = [torch.zeros(ob, dtype=torch.uint8, device="cuda") for _ in range(G)]
for t in range(5):
    rec = random_events(rng, st.slots(0), t, p_new=0.5 if t == 0 else 0.1)
    if rec is not None:
        st.enqueue(0, rec)
        ids = rec["id"].astype(np.int64)
        for r in range(G):
            m = (ids // MA) == r
            if m.any():
                sub = {k: np.ascontiguousarray(v[m]) for k, v in rec.items()}
                sub["id"] = (ids[m] - r * MA).astype(np.uint32)
                hs[r].enqueue(0, sub)
    o = st.step(t)
    for r in range(G):
        hs[r].shard_begin(t, led[r])
    ls = torch.stack(led).sum(0)
    for r in range(G):
        hs[r].shard_offer(ls, off[r])
    allo = torch.cat(off)
    outs = [hs[r].shard_commit(allo, G, r) for r in range(G)]
    g = hs[0].shard_result(outs[0])
    a = int(o["admitted"][0])
    assert g["admitted"] == a and g["order"].tolist() == o["order"][0][:a].tolist()
    assert g["grant"].tolist() == o["grant"][0][:a].tolist()
for h in hs:
    h.sync()
    h.close()
print("sanitize driver ok")
