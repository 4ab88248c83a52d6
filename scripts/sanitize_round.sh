#!/bin/bash
# compute-sanitizer passes over small solves of every entry point (scripts/sanitize_cases.py).
set -u
O=gpurun_out
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 --error-exitcode 9 python scripts/sanitize_cases.py \
      > $O/sanitize_$T.log 2>&1
  echo "$T rc=$?" >> $O/sanitize_summary.txt
  tail -5 $O/sanitize_$T.log >> $O/sanitize_summary.txt
done
cat $O/sanitize_summary.txt
