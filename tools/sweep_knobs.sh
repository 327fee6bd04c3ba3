#!/bin/bash
# Simulate-kernel knob sweep (GPU box): each argument is a set of -D flags;
# prints the per-window times of tools/prof_sim.py (cfg5-sized, 8 windows)
# and the sum of windows 4-8 (the ones bench.py times).
set -u
for v in "$@"; do
  AUGSCHED_NVCC_EXTRA="$v" python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
  python tools/prof_sim.py --instances 65536 --windows 8 | awk -v m="$v" '{n++; if (n>=4) t+=$4; s=s" "$4} END{print "[" m "] bench-windows", t, "|", s}'
done
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
