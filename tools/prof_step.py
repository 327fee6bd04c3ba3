"""Profiling driver (not a bench): cfg4 augsched_step over an n-slot queue,
`--steps` consecutive steps after `--warmup`.  Used under ncu on the GPU box."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import tracegen  # noqa: E402
import paper_2512_04013_b200 as aug  # noqa: E402
from paper_2512_04013_b200 import _build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--time", action="store_true")
ap.add_argument("--prefix", action="store_true")
a = ap.parse_args()
_build.build()
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
rec = tracegen.cfg4_records(a.n)
s = aug.Scheduler(tracegen.PRESET_CFG4, tracegen.inst_params(1), 1, a.n, stream=st)
s.enqueue(0, rec)
t = 65536
for _ in range(a.warmup):
    s.step(t, prefix=a.prefix); t += 1
torch.cuda.synchronize()
ms = []
for _ in range(a.steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.step(t, prefix=a.prefix); e1.record(st); t += 1
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
print("n", a.n, "step ms", ["%.4f" % x for x in ms], "median %.4f" % float(np.median(ms)))
s.close()
