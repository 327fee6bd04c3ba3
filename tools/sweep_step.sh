#!/bin/bash
# Tuning sweep (GPU box) of the step path: for each set of -D overrides,
# rebuild, time tools/prof_step.py and list per-kernel device times (ncu).
# Usage: tools/sweep_step.sh N "SORT_ITEMS=16,LB_WIN=8" ...
set -u
n=$1; shift
for v in "$@"; do
  defs=""
  for kv in ${v//,/ }; do defs="$defs -DAUGSCHED_${kv}"; done
  AUGSCHED_NVCC_EXTRA="$defs" \
    python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
  echo "== $v"
  python tools/prof_step.py --n $n --steps 7 2>&1 | tail -1
  ncu --metrics gpu__time_duration.sum --clock-control none -s 14 -c 7 --csv \
      python tools/prof_step.py --n $n --steps 2 2>/dev/null | \
    python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10 and r[0].isdigit()]
print(' '.join('%s=%.1f' % (r[4].split('(')[0].split('::')[-1][:14], float(r[-1])/1e3) for r in rows))"
done
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
