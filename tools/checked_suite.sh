#!/bin/bash
# The compute-sanitizer stand-in (the pool does not allow compute-sanitizer):
# run the whole GPU test suite, the smoke test and one bench-sized step against
# the CHECKED build (-DIRKG_CHECKED: device bounds / invariant checks that trap
# with file:line), with graphs + PDL on (default) and off.
# Logs -> gpurun_out/checked/.
set -u
out=gpurun_out/checked; mkdir -p $out
lib=paper_2101_01776_b200/libirkg_checked.so
[ -f $lib ] || python -m paper_2101_01776_b200._build --checked > $out/build.log 2>&1
export IRKG_LIB=$PWD/$lib
python -c "from paper_2101_01776_b200 import _lib; print(\"library:\", _lib.LIB_PATH)" | tee -a $out/summary.txt
for mode in "1 1" "0 0"; do
  set -- $mode
  tag=graphs$1_pdl$2
  IRKG_GRAPHS=$1 IRKG_PDL=$2 timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider \
    > $out/tests_$tag.txt 2>&1
  echo "checked gpu suite $tag rc=$? $(tail -1 $out/tests_$tag.txt)" | tee -a $out/summary.txt
  IRKG_GRAPHS=$1 IRKG_PDL=$2 timeout 600 python tools/one_step.py > $out/step_$tag.txt 2>&1
  echo "checked configs[1] step $tag rc=$? $(tail -1 $out/step_$tag.txt)" | tee -a $out/summary.txt
done
grep -h "IRKG_DCHECK failed" $out/*.txt | sort | uniq -c | head -20 | tee -a $out/summary.txt
