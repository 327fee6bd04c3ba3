#!/bin/bash
# A/B of sim.cu source variants on one box: tools/sweep_src.sh INSTANCES file1.cu file2.cu ...
set -u
inst=$1; shift
cp paper_2512_04013_b200/csrc/sim.cu /tmp/sim_orig.cu
for f in "$@"; do
  for rep in 1 2; do
    cp "$f" paper_2512_04013_b200/csrc/sim.cu
    python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
    echo "== $f (rep $rep)"
    python tools/prof_sim.py --instances $inst --windows 6 | tail -3
  done
done
cp /tmp/sim_orig.cu paper_2512_04013_b200/csrc/sim.cu
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
