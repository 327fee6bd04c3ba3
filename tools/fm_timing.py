"""Per-phase clocks of the batched full step (full_multi_kernel) on bench.py's
step_multi workload, from a -DAUGSCHED_FM_TIMING build (AUGSCHED_LIB): the
average cycles per CTA (one instance) of each phase, and how many CTAs took
the incremental merge."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import tracegen  # noqa: E402
import paper_2512_04013_b200 as aug  # noqa: E402

n_inst, ma = 4096, 2048
torch.cuda.set_device(0)
rec = tracegen.cfg4_records(ma, n_running=16, n_swapped=16, n_paused=4)
s = aug.Scheduler(tracegen.PRESET_CFG4, tracegen.inst_params(n_inst), n_inst, ma)
for i in range(n_inst):
    s.enqueue(i, rec)
fn = aug.lib().augsched_fm_timing
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
t = 65536
for _ in range(5):
    s.step(t); t += 1
torch.cuda.synchronize()
fn(buf, 1)
K = 10
for _ in range(K):
    s.step(t); t += 1
torch.cuda.synchronize()
fn(buf, 0)
v = list(buf)
c = max(v[8], 1)
for i, nm in enumerate(["words + tier counts", "incremental merge / LSD sort", "kept-order write",
                        "pf_finish (prefix sort, admission, resolution, apply)", "order/key tail writes"]):
    print(f"{nm:55s} {v[i] / c:10.0f} cycles/CTA")
print(f"CTAs {v[8]}, incremental {v[9]} ({v[9] / c:.3f}), mean |D| {v[10] / max(v[9], 1):.1f}")
s.close()
