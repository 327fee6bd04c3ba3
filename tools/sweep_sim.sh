#!/bin/bash
# Tuning sweep (GPU box): rebuild libaugsched with each set of -D overrides
# and time tools/prof_sim.py.  Usage:
#   tools/sweep_sim.sh INSTANCES "NT=32,MINB=16,UNROLL=4,SCAP=384" ...
set -u
inst=$1; shift
for v in "$@"; do
  defs=""
  for kv in ${v//,/ }; do defs="$defs -DAUGSCHED_SIM_${kv}"; done
  AUGSCHED_NVCC_EXTRA="$defs" \
    python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
  echo "== $v"
  python tools/prof_sim.py --instances $inst --windows 4
done
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
