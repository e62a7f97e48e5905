#!/bin/bash
# compute-sanitizer over every kernel of libfcfs.so at small sizes (tools/sanitize_driver.py).
# Usage (under gpurun): bash tools/sanitize.sh <tag>   -> gpurun_out/<tag>_sanitize_<tool>_<case>.log
set -u
T=${1:-r02}
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-memcheck synccheck racecheck initcheck}; do
  for c in extract c1 c3 c4 haar; do
    timeout ${TMO:-600} $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_driver.py $c \
      > $O/${T}_sanitize_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" | tee -a $O/${T}_sanitize_summary.txt
  done
done
