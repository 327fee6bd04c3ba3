#!/bin/bash
# Same-box A/B of library builds: tools/ab_libs.sh OUT lib1.so lib2.so ...  (runs tools/sim_windows.py per build)
out=$1; shift
cp paper_2512_04013_b200/libaugsched.so /tmp/ab_keep.so
for f in "$@"; do
  cp "$f" paper_2512_04013_b200/libaugsched.so
  echo "== $f" >> "$out"
  python tools/sim_windows.py 2>&1 | tail -1 >> "$out"
done
cp /tmp/ab_keep.so paper_2512_04013_b200/libaugsched.so
