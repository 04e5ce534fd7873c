#!/bin/bash
# compute-sanitizer over the small runs of tools/sanitize_run.py; one summary
# line per (tool, case) into gpurun_out/sanitize/summary.txt, full logs beside it
mkdir -p gpurun_out/sanitize
out=gpurun_out/sanitize/summary.txt
: > $out
for tool in memcheck racecheck synccheck initcheck; do
  for c in ${CASES:-c1 thermal warp giant shock batch fused wb literal}; do
    log=gpurun_out/sanitize/${tool}_$c.log
    timeout ${SAN_TIMEOUT:-600} compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $c 2 > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok [0-9]' $log | tr '\n' ' ')" >> $out
  done
done
cat $out
