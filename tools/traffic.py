"""Summarise an ncu launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) into the traffic files bench.py reads:

  sim   python tools/traffic.py sim gpurun_out/traffic.csv [instances] [window]
        the first sim_kernel launches of a bench run (warm-up and timed
        windows in launch order) -> profiles/sim_kernel_traffic.json, one
        entry per window; bench.py averages the windows it times.
  step  python tools/traffic.py step gpurun_out/step.csv prefix|full
        steady launches of tools/bench_step.py per queue size ->
        profiles/step_{prefix,full}_traffic.json.
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def launches(path, pat):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[h]
    iname, imet, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    by, names = {}, {}
    for r in rows[h + 1:]:
        if len(r) <= ival or pat not in r[iname]:
            continue
        by.setdefault(int(r[0]), {})[r[imet]] = float(r[ival].replace(",", ""))
        names[int(r[0])] = r[iname]
    return [by[k] for k in sorted(by)], [names[k] for k in sorted(by)]


mode = sys.argv[1]
if mode == "sim":
    L, _ = launches(sys.argv[2], "sim_kernel")
    inst = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
    win = int(sys.argv[4]) if len(sys.argv) > 4 else 1500
    rd = [x["dram__bytes_read.sum"] for x in L]
    wr = [x["dram__bytes_write.sum"] for x in L]
    out = {
        "kernel": "sim_kernel",
        "workload": bench.workload_name(argparse.Namespace(workload="cfg5", instances=inst, scaling="strong"), 1),
        "window_iters": win,
        "source": os.path.basename(sys.argv[2]),
        "launches": len(L),
        "dram_bytes_read_per_launch": rd,
        "dram_bytes_write_per_launch": wr,
        "gpu_time_ns_per_launch": [x["gpu__time_duration.sum"] for x in L],
        "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                "--clock-control none -k regex:sim_kernel -c <warmup+steps> python bench.py ...: window k = "
                "launch k (warm-up windows first); the per-launch times are serialised, cold and under the "
                "profiler: only the bytes are used",
    }
    dst = os.path.join(ROOT, "profiles", "sim_kernel_traffic.json")
else:
    kind = sys.argv[3]
    pat = "pf_step_kernel" if kind == "prefix" else "full_coop_kernel"
    L, _ = launches(sys.argv[2], pat)
    # tools/bench_step.py runs sizes in order, warmup + 2*steps launches each
    per = int(os.environ.get("PER_SIZE", "0")) or len(L) // 3
    sizes = [int(x) for x in os.environ.get("SIZES", "1000000,4194304,16000000").split(",")]
    out = {"kernel": pat, "source": os.path.basename(sys.argv[2]), "sizes": {}}
    for i, n in enumerate(sizes):
        blk = L[i * per:(i + 1) * per][1:]      # the first launch of a size is the fallback / cold one
        if not blk:
            continue
        b = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in blk]
        out["sizes"][str(n)] = {"launches": len(blk), "dram_bytes_per_launch_mean": sum(b) / len(b),
                                "gpu_time_ns_mean": sum(x["gpu__time_duration.sum"] for x in blk) / len(blk)}
    dst = os.path.join(ROOT, "profiles", f"step_{kind}_traffic.json")
json.dump(out, open(dst, "w"), indent=1)
print(dst, json.dumps(out)[:300])
