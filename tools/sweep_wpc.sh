#!/bin/bash
# Simulate-kernel sweep (GPU box): instances per CTA (SIM_WPC), register bound
# (SIM_MINB = warps per SM) and per-phase fences (SIM_PSYNC); times
# tools/prof_sim.py on cfg5-sized input.
# Usage: tools/sweep_wpc.sh INSTANCES "WPC MINB PSYNC" ...
set -u
inst=$1; shift
for v in "$@"; do
  set -- $v
  AUGSCHED_NVCC_EXTRA="-DAUGSCHED_SIM_WPC=$1 -DAUGSCHED_SIM_MINB=$2 -DAUGSCHED_SIM_PSYNC=${3:-0}" \
    python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
  echo "== WPC=$1 MINB=$2 PSYNC=${3:-0}"
  python tools/prof_sim.py --instances $inst --windows 3 | tail -1
done
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
