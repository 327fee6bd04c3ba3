"""Per-source-line warp-stall and instruction shares of one kernel in an ncu
report (ncu -i REP --page source --csv --print-source cuda,sass)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
items, tot, toti, fname = [], 0.0, 0.0, ""
h = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        h = r
        si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        continue
    if h is None or r[0] in ("", "Function Name") or len(r) <= ii:
        continue
    try:
        v, n = float(r[si] or 0), float(r[ii] or 0)
    except ValueError:
        continue
    tot += v
    toti += n
    items.append((v, n, f"{fname}:{r[0]}", r[1].strip()[:100]))
items.sort(reverse=True)
for v, n, line, src in items[:top]:
    print(f"stall {100 * v / max(tot, 1):5.1f}%  instr {100 * n / max(toti, 1):5.1f}%  {line:>16} {src}")
