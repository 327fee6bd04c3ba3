"""Timing driver (not a bench): bench.py's cfg5 workload through
augsched_simulate for `--windows` windows of 1,500 iterations; prints the
per-window time and counts and the rates over the driver's timed windows
(5 .. windows-1).  Used for same-box A/B of library builds."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import tracegen  # noqa: E402
import bench  # noqa: E402
import paper_2512_04013_b200 as aug  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--instances", type=int, default=65536)
ap.add_argument("--windows", type=int, default=25)
ap.add_argument("--warm", type=int, default=5)
ap.add_argument("--libs", default="", help="comma-separated .so files to A/B (copied over libaugsched.so)")
a = ap.parse_args()
args = argparse.Namespace(workload="cfg5", instances=a.instances, scaling="strong")
tr, ip, tid, ma, _, _ = bench.workload(args, 0, 1)
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
dtr = aug.DeviceTraces(tr)
tid_d = torch.from_numpy(tid.astype(np.int32)).cuda()
s = aug.Scheduler(tracegen.PRESET_7B, ip, len(tid), ma, stream=st)
out = torch.empty(len(tid) * aug.RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
ms, dec, bs = [], [], []
for w in range(a.windows):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.simulate(dtr, tid_d, (w + 1) * 1500, out=out, resume=w > 0)
    e1.record(st)
    torch.cuda.synchronize()
    r = aug.results_to_numpy(out)
    f = lambda k: int(r["f"][:, aug.RESULT_FIELDS.index(k)].sum())
    ms.append(e0.elapsed_time(e1)); dec.append(f("decisions")); bs.append(f("busy_steps"))
s.close()
T = sum(ms[a.warm:]) / 1e3
D = dec[-1] - dec[a.warm - 1]
S = bs[-1] - bs[a.warm - 1]
print("per-window ms", [round(x, 1) for x in ms])
print(f"windows {a.warm}..{a.windows - 1}: {T:.3f} s, {D / T / 1e9:.2f} G decisions/s, "
      f"{S / T / 1e6:.2f} M instance-steps/s, {D / S:.1f} decisions/instance-step; digest {int(r['f'].sum()) & 0xffffffff:08x}")
