#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py: tools/sanitize.sh OUTDIR
out=${1:-gpurun_out}
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_driver.py > $out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $out/sanitize_summary.txt
  tail -3 $out/sanitize_$tool.log >> $out/sanitize_summary.txt
done
