"""Robustness sweep at scale on the GPU (tab:cv; SURVEY f2 + f3):
W3 traces (Gamma arrivals, coefficient of variation CV, 30-minute horizon)
drawn on the device by augsched_generate, simulated under four systems side
by side in one augsched_simulate call per CV:
  vllm      FCFS + Discard-only + static limit 500
  infercept FCFS + adaptive policy + static 500
  maxbatch  FCFS + adaptive policy + dynamic limit   ("w/ MaxBatch")
  augserve  two-stage values + adaptive policy + dynamic limit
Every run stops at the 30-minute horizon (R28: max_iters = H / T^fwd);
requests unfinished then are excluded from attainment and counted as
incomplete.  Reports goodput (SLO-meeting completions per second
over the window, R25) and the incomplete share per (CV, rate, system).  Usage: python tools/cv_sweep.py [traces_per_rate]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import tracegen  # noqa: E402
from tracegen import tablegen as tg  # noqa: E402
import paper_2512_04013_b200 as aug  # noqa: E402
from paper_2512_04013_b200 import _build  # noqa: E402

H = 1800 * 10**6
SYSTEMS = {"vllm": dict(ranking=1, budget_mode=1, policy_mode=3), "infercept": dict(ranking=1, budget_mode=1),
           "maxbatch": dict(ranking=1, budget_mode=0), "augserve": dict(ranking=0, budget_mode=0)}
RATES = [1.0, 2.0, 3.0]


def main():
    per_rate = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    _build.build()
    torch.cuda.set_device(0)
    n_traces = per_rate * len(RATES)
    rates = [RATES[k // per_rate] for k in range(n_traces)]
    names = list(SYSTEMS)
    n_inst = n_traces * len(names)
    cols = {k: [] for k in ("ranking", "budget_mode", "policy_mode")}
    for k in range(n_traces):
        for nm in names:
            for c in cols:
                cols[c].append(SYSTEMS[nm].get(c, 0))
    ip = tracegen.inst_params(n_inst, l_static=500, **{c: np.array(v) for c, v in cols.items()})
    tid = np.repeat(np.arange(n_traces), len(names)).astype(np.int32)
    out = {"systems": names, "rates": RATES, "traces_per_rate": per_rate, "goodput_req_s": {}}
    for cv in (1.0, 1.5, 2.0, 3.0):
        T = tg.build_tables(cv=cv)
        probe = aug.Scheduler(tracegen.PRESET_7B, tracegen.inst_params(1), 1, 8)
        gt = aug.GeneratedTraces(probe, T, 1000 + int(cv * 10), n_traces, 20000, rates, horizon_ticks=H)
        ma = int(np.diff(gt.to_numpy()["req_off"].astype(np.int64)).max())
        probe.close()
        s = aug.Scheduler(tracegen.PRESET_7B, ip, n_inst, ma)
        t0 = time.time()
        max_iters = H // tracegen.PRESET_7B["t_fwd_ticks"]          # stop at the horizon (R28)
        res = aug.results_to_numpy(s.simulate(gt, torch.from_numpy(tid).cuda(), max_iters))
        s.sync()
        dt = time.time() - t0
        s.close()
        F = lambda k: res["f"][:, aug.RESULT_FIELDS.index(k)].astype(np.float64).reshape(n_traces, len(names))
        slo, inc, nreq = F("slo_ok"), F("incomplete"), F("n_requests")
        for ri, r in enumerate(RATES):
            rs = slice(ri * per_rate, (ri + 1) * per_rate)
            g = slo[rs].mean(axis=0) / 1800.0
            out["goodput_req_s"][f"cv{cv}_rate{r}"] = {nm: round(float(x), 4) for nm, x in zip(names, g)}
            out.setdefault("incomplete_share", {})[f"cv{cv}_rate{r}"] = {
                nm: round(float(x), 4) for nm, x in zip(names, inc[rs].sum(axis=0) / nreq[rs].sum(axis=0))}
        print(f"cv {cv}: {n_inst} instances simulated in {dt:.1f} s", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
