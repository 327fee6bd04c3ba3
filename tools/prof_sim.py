"""Profiling driver (not a bench): cfg5-shaped augsched_simulate with
`--instances` instances, `--windows` windows of `--window` iterations."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import tracegen  # noqa: E402
import paper_2512_04013_b200 as aug  # noqa: E402
from paper_2512_04013_b200 import _build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--instances", type=int, default=8192)
ap.add_argument("--window", type=int, default=1500)
ap.add_argument("--windows", type=int, default=4)
a = ap.parse_args()
_build.build()
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
n_tr = max(1, a.instances // 16)
tr = tracegen.gen_traces(n_tr, 5000, [2.0, 3.0, 4.0, 5.0], seed=5000)
ip = tracegen.cfg5_params(a.instances)
tid = (np.arange(a.instances) // 16).astype(np.int32)
s = aug.Scheduler(tracegen.PRESET_7B, ip, a.instances, 5000, stream=st)
dtr = aug.DeviceTraces(tr)
tid_d = torch.from_numpy(tid).cuda()
out = torch.empty(a.instances * aug.RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
for w in range(a.windows):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.simulate(dtr, tid_d, (w + 1) * a.window, out=out, resume=w > 0)
    e1.record(st)
    torch.cuda.synchronize()
    r = aug.results_to_numpy(out)
    f = lambda k: int(r["f"][:, aug.RESULT_FIELDS.index(k)].sum())
    print("window", w, "ms %.2f" % e0.elapsed_time(e1), "decisions", f("decisions"), "busy", f("busy_steps"))
s.close()
