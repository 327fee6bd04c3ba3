"""Timing driver (not a bench): augsched_step vs augsched_step_prefix on a
multi-instance handle (n_inst queues of MA slots, cfg4-shaped records per
instance), L2 flushed before each step."""
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
ap.add_argument("--inst", type=int, default=4096)
ap.add_argument("--ma", type=int, default=2048)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
_build.build()
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
rec = tracegen.cfg4_records(a.ma, n_running=16, n_swapped=16, n_paused=4)
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
for prefix in (False, True):
    s = aug.Scheduler(tracegen.PRESET_CFG4, tracegen.inst_params(a.inst), a.inst, a.ma, stream=st)
    for i in range(a.inst):
        s.enqueue(i, rec)
    t = 65536
    for _ in range(2):
        s.step(t, prefix=prefix); t += 1
    torch.cuda.synchronize()
    ms = []
    for _ in range(a.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); s.step(t, prefix=prefix); e1.record(st); t += 1
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    n = a.inst * a.ma
    med = float(np.median(ms))
    print(f"{'prefix' if prefix else 'full  '} {a.inst}x{a.ma}: {med*1e3:.1f} us/step, "
          f"{n/(med/1e3)/1e9:.1f} G decisions/s, frac {32*n/(med/1e3)/1e9/6539.2:.3f}", flush=True)
    s.close()
