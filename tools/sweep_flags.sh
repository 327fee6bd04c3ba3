#!/bin/bash
# Build-flag sweep (GPU box): rebuild with each raw nvcc flag set and time tools/prof_sim.py.
# Usage: tools/sweep_flags.sh INSTANCES "-Xptxas -O2" "-Xptxas -O1" ...
set -u
inst=$1; shift
for v in "$@"; do
  AUGSCHED_NVCC_EXTRA="$v" python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
  echo "== $v"
  python tools/prof_sim.py --instances $inst --windows 4 | tail -1
done
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
