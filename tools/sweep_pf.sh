#!/bin/bash
# prefix-step timing variants (GPU box): per-kernel device times for each -D set
set -u
for v in "$@"; do
  defs=""
  for kv in ${v//,/ }; do [ "$kv" != "-" ] && defs="$defs -DAUGSCHED_${kv}"; done
  AUGSCHED_NVCC_EXTRA="$defs" python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
  echo "== $v"
  python tools/prof_step.py --n 1000000 --steps 7 --prefix 2>&1 | tail -1
  ncu --metrics gpu__time_duration.sum --clock-control none -s 8 -c 3 --csv \
      python tools/prof_step.py --prefix --steps 2 2>/dev/null | \
    python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10 and r[0].isdigit()]
print(' '.join('%s=%.1f' % (r[4].split('(')[0].split('::')[-1][:14], float(r[-1])/1e3) for r in rows))"
done
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
