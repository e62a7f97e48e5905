# ncu --set full (source page) of one kernel of a bench command (usage under gpurun:
#   bash tools/ncu_kernel_src.sh <tag> <kernel regex> <bench args...>)
T=$1; K=$2; shift 2
O=gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extra $@"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o $O/${T} $B > $O/${T}_ncu.log 2>&1
tail -1 $O/${T}_ncu.log
