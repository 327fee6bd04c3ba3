"""Path statistics of the simulator (not a bench): bench.py's cfg5 workload
through a -DAUGSCHED_SIM_STATS build of the library (AUGSCHED_LIB), run for
`--windows` windows of 1,500 iterations; prints per-window times and the
path counters of the windows after `--warm` (sim.cu SSTAT)."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import tracegen  # noqa: E402
import bench  # noqa: E402
import paper_2512_04013_b200 as aug  # noqa: E402

NAMES = {0: "steps reaching W (wall >= B)", 16: "  everything fits (WMODE_ALL)", 26: "  W pop rounds ended",
         20: "  W radix fallback", 27: "  W pop rounds", 28: "  W rescans", 17: "prefix ends in running tier",
         22: "prefix ends in swapped tier", 23: "select_cand (R)", 24: "select_arr (R)", 25: "tier-0 candidates",
         29: "memory resolution", 2: "  resolution with P == 0", 3: "  paused entries scanned", 4: "  eviction needed after demotion", 18: "busy steps", 30: "R entries", 31: "W entries"}

ap = argparse.ArgumentParser()
ap.add_argument("--instances", type=int, default=65536)
ap.add_argument("--windows", type=int, default=8)
ap.add_argument("--warm", type=int, default=5)
a = ap.parse_args()
args = argparse.Namespace(workload="cfg5", instances=a.instances, scaling="strong")
tr, ip, tid, ma, _, _ = bench.workload(args, 0, 1)
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
L = aug.lib()
fn = L.augsched_sim_stats
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 64)()
dtr = aug.DeviceTraces(tr)
tid_d = torch.from_numpy(tid.astype(np.int32)).cuda()
s = aug.Scheduler(tracegen.PRESET_7B, ip, len(tid), ma, stream=st)
out = torch.empty(len(tid) * aug.RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
for w in range(a.windows):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if w == a.warm:
        torch.cuda.synchronize()
        fn(buf, 1)
    e0.record(st)
    s.simulate(dtr, tid_d, (w + 1) * 1500, out=out, resume=w > 0)
    e1.record(st)
    torch.cuda.synchronize()
    print("window", w, "ms %.1f" % e0.elapsed_time(e1), flush=True)
fn(buf, 0)
v = list(buf)
for i, nm in sorted(NAMES.items()):
    print(f"{i:2d} {nm:36s} {v[i]:>16d}  per busy step {v[i] / max(v[18], 1):.4f}")
PH = ["intake", "R keys", "selection", "resolution", "grants+advance", "compaction+prep"]
nit, nf = max(v[47], 1), max(v[46], 1)
print(f"CTA iterations with full steps {v[47]}, full steps {v[46]} ({v[46] / nit:.2f} per iteration)")
print("phase               slowest-step cycles/iter   mean-step cycles/iter")
for i, nm in enumerate(PH):
    print(f"  {nm:18s} {v[32 + i] / nit:12.0f}            {v[40 + i] / nf:12.0f}")
print(f"  {'total':18s} {sum(v[32:38]) / nit:12.0f}            {sum(v[40:46]) / nf:12.0f}")
s.close()
