"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv): launches, total time,
share of the listed time, DRAM MB.  python tools/launch_summary.py CSV [header]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
iname, imet, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
by = {}
for r in rows[h + 1:]:
    if len(r) <= ival:
        continue
    k = by.setdefault(int(r[0]), {"name": r[iname]})
    k[r[imet]] = float(r[ival].replace(",", ""))
agg = {}
for k in by.values():
    nm = k["name"].split("(")[0][:60]
    a = agg.setdefault(nm, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += k.get("gpu__time_duration.sum", 0.0) / 1e3
    a[2] += (k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)) / 1e6
tot = sum(a[1] for a in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("# kernel | launches | total us | share | DRAM MB (serialised, cold: only the shares matter)")
for nm, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{nm:60s} | {a[0]:4d} | {a[1]:10.1f} | {100 * a[1] / tot:5.1f}% | {a[2]:10.1f}")
