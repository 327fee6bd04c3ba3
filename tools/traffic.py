"""Summarise an ncu launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) of the sim_kernel launches that bench.py times into
profiles/sim_kernel_traffic.json, which bench.py reads for roofline.traffic.
Usage: python tools/traffic.py gpurun_out/traffic.csv [instances] [window]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import argparse  # noqa: E402
import bench  # noqa: E402
rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
by = {}
for r in rows[h + 1:]:
    if "sim_kernel" not in r[4]:
        continue
    by.setdefault(r[0], {})[r[-3]] = float(r[-1].replace(",", ""))
launches = [by[k] for k in sorted(by, key=int)]
rd = [x["dram__bytes_read.sum"] for x in launches]
wr = [x["dram__bytes_write.sum"] for x in launches]
out = {
    "kernel": "sim_kernel",
    "workload": bench.workload_name(argparse.Namespace(
        workload="cfg5", instances=int(sys.argv[2]) if len(sys.argv) > 2 else 65536)),
    "window_iters": int(sys.argv[3]) if len(sys.argv) > 3 else 1500,
    "source": os.path.basename(sys.argv[1]),
    "launches": len(launches),
    "dram_bytes_read_per_launch": rd,
    "dram_bytes_write_per_launch": wr,
    "dram_bytes_per_launch_mean": (sum(rd) + sum(wr)) / len(launches),
    "gpu_time_ns_per_launch": [x["gpu__time_duration.sum"] for x in launches],
    "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
            "--clock-control none -k regex:sim_kernel -s <warmup> -c <steps> on bench.py's timed launches",
}
json.dump(out, open(os.path.join(ROOT, "profiles", "sim_kernel_traffic.json"), "w"), indent=1)
print(json.dumps(out)[:400])
