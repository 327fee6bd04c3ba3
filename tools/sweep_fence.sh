#!/bin/bash
# Simulate-kernel fence-set sweep (GPU box): AUGSCHED_SIM_PSYNC bitmask at
# SIM_WPC=16 / SIM_MINB=32; prints the per-window times of tools/prof_sim.py
# (cfg5-sized, 8 windows of 1,500 iterations) and their sum.
set -u
for m in "$@"; do
  AUGSCHED_NVCC_EXTRA="-DAUGSCHED_SIM_PSYNC=$m" \
    python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
  python tools/prof_sim.py --instances 65536 --windows 8 | awk -v m=$m '{t+=$4; s=s" "$4} END{print "mask", m, "sum", t, "|", s}'
done
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
