#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_step.py
# with graphs + PDL on (the default path) and off.  Logs -> gpurun_out/sanitize/.
out=gpurun_out/sanitize; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for mode in "1 1" "0 0"; do
  set -- $mode
  for tool in memcheck racecheck synccheck; do
    log=$out/${tool}_graphs$1_pdl$2.txt
    IRKG_GRAPHS=$1 IRKG_PDL=$2 timeout 1200 $CS --tool $tool --error-exitcode 99 \
      --target-processes all python tools/sanitize_step.py > $log 2>&1
    echo "$tool graphs=$1 pdl=$2 rc=$?" | tee -a $out/summary.txt
    tail -3 $log >> $out/summary.txt
  done
done
