#!/bin/bash
# compute-sanitizer passes over tools/sanitize_run.py (one process per case so a hang or a crash in one
# kernel family does not hide the others).  Run from the repo root under gpurun; logs land in gpurun_out/.
set -u
mkdir -p gpurun_out
TOOLS=${TOOLS:-"memcheck"}
CASES=${CASES:-"cfg2 cfg2_ws cfg2_fh cfg2_x3 cfg1 cfg4 cfg3"}
for tool in $TOOLS; do
  for c in $CASES; do
    log=gpurun_out/sanitizer_${tool}_${c}.log
    timeout ${CASE_TIMEOUT:-600} compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_run.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)"
  done
done
