#!/bin/bash
# A/B of (sim.cu, select.cuh) variant pairs on one box:
#   tools/sweep_src2.sh INSTANCES sim_a.cu:select_a.cuh sim_b.cu:select_b.cuh ...
set -u
inst=$1; shift
d=paper_2512_04013_b200/csrc
cp $d/sim.cu /tmp/sim_orig.cu; cp $d/select.cuh /tmp/select_orig.cuh
for pair in "$@"; do
  for rep in 1 2; do
    cp "${pair%%:*}" $d/sim.cu; cp "${pair##*:}" $d/select.cuh
    python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)" || exit 1
    echo "== $pair (rep $rep)"
    python tools/prof_sim.py --instances $inst --windows 6 | tail -2
  done
done
cp /tmp/sim_orig.cu $d/sim.cu; cp /tmp/select_orig.cuh $d/select.cuh
python -c "from paper_2512_04013_b200 import _build; _build.build(force=True)"
