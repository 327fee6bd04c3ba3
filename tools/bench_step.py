"""Run only bench.py's cfg4 step measurements (same code path and timing:
L2 flushed before each step, CUDA events on the scheduler's stream)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--step-n", type=int, default=1_000_000)
ap.add_argument("--sizes", default="1000000,4194304,16000000")
ap.add_argument("--full", action="store_true", help="also the full-order step")
ap.add_argument("--multi", action="store_true", help="the batched step (4,096 instances x 2,048 slots) only")
ap.add_argument("--ti", action="store_true", help="also the full step with time-invariant keys (ranking 3)")
ap.add_argument("--only-ti", action="store_true", help="only the time-invariant full step")
a = ap.parse_args()
torch.cuda.set_device(0)
stream = torch.cuda.current_stream()
peak = bench.hbm_peak()[0]
out = {}
if a.multi:
    print(json.dumps(bench.step_multi_bench(a, 0, stream, peak), indent=1))
    sys.exit(0)
for n in [int(x) for x in a.sizes.split(",")]:
    if a.only_ti:
        r = bench.step_bench(a, 0, stream, peak, n_override=n, ranking=3)
        out[n] = {"ti_ms_cold": r["ms_per_step_cold_l2"], "ti_ms_warm": r["ms_per_step_warm_l2"]}
        continue
    r = bench.step_bench(a, 0, stream, peak, prefix=True, n_override=n)
    out[n] = {k: r[k] for k in ("value", "ms_per_step_cold_l2", "ms_per_step_warm_l2", "launches_per_step")}
    out[n]["frac"] = r["roofline"]["frac"]
    if a.full:
        r = bench.step_bench(a, 0, stream, peak, prefix=False, n_override=n)
        out[n]["full_ms_cold"] = r["ms_per_step_cold_l2"]
    if a.ti:
        r = bench.step_bench(a, 0, stream, peak, n_override=n, ranking=3)
        out[n]["ti_ms_cold"] = r["ms_per_step_cold_l2"]
print(json.dumps(out, indent=1))
