#!/bin/bash
# The bounds-checked build (libfcfs_checked.so: -DFCFS_CHECKED, device-side FCFS_DCHECK invariants on
# SMEM / TMEM / global indices and pipeline slots) over every kernel (tools/sanitize_driver.py) and the
# whole GPU parity suite.  compute-sanitizer is closed on this GPU pool; this is the substitute.
# Usage (under gpurun): bash tools/checked_run.sh <tag>  -> gpurun_out/<tag>_checked_*.log
set -u
T=${1:-r02}
O=gpurun_out
LIB=$(pwd)/paper_1010_5562_b200/libfcfs_checked.so
test -f $LIB || python -m paper_1010_5562_b200.build --checked
FCFS_LIBRARY=$LIB timeout 600 python tools/sanitize_driver.py > $O/${T}_checked_driver.log 2>&1
echo "driver rc=$?" | tee $O/${T}_checked_summary.txt
FCFS_LIBRARY=$LIB timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/${T}_checked_pytest.log 2>&1
echo "pytest -m gpu (checked build) rc=$?" | tee -a $O/${T}_checked_summary.txt
tail -3 $O/${T}_checked_pytest.log | tee -a $O/${T}_checked_summary.txt
grep -h "FCFS_DCHECK failed" $O/${T}_checked_*.log | sort | uniq -c | tee -a $O/${T}_checked_summary.txt
