"""Probe one edge-case instance of tests/test_gpu_simulate.py::test_edge_cases_parity on the GPU."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import tracegen, oracle
import paper_2512_04013_b200 as aug


def R(arr, l_pre, segs):
    return {"arr": arr, "l_pre": l_pre,
            "segs": [(s[0], s[0], 0, 0.0, 0) if len(s) == 1 else (s[0], s[0], s[1], s[2], s[3]) for s in segs]}


which = int(sys.argv[1])
reqs = [[], [R(0, 5, [(1, 10_000, 0.01, 1)] * 254 + [(2,)])], [R(1000 * i, 1, [(3,)]) for i in range(400)],
        [R(0, 40, [(30,)]) for _ in range(160)]]
tr = tracegen.from_requests(reqs)
cfg = dict(tracegen.PRESET_G0, g_total=1000 + 3000, g_model=1000)
full = dict(budget_mode=[1, 1, 1, 0, 1, 0], l_static=[50, 0, 100, 0, 2000, 0], target_max=[50, 50, 50, 50, 50, 3000],
            alpha=[0.0, 0.0, 0.0, 2.0, 0.0, 1.0])
tid_all = [0, 1, 1, 2, 2, 3]
ip = tracegen.inst_params(1, base=tracegen.INST_G0, **{k: [v[which]] for k, v in full.items()})
tid = np.array([tid_all[which]], np.uint32)
s = aug.Scheduler(cfg, ip, 1, 400)
out = s.simulate(aug.DeviceTraces(tr), torch.from_numpy(tid.astype(np.int32)).cuda(), 5000)
g = aug.results_to_numpy(out)
s.sync(); s.close()
o = oracle.simulate(cfg, ip, tr, tid, max_iters=5000)
print(which, "equal", g.tobytes() == o.tobytes(), aug.as_dict(g[0])["busy_steps"], oracle.as_dict(o[0])["busy_steps"])
