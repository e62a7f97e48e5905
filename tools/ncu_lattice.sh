# ncu --set full of k_lattice on c3 with the source page (usage under gpurun: bash tools/ncu_lattice.sh <tag> [lib])
T=${1:-lat}
LIB=${2:-paper_1010_5562_b200/libfcfs.so}
O=gpurun_out
B3="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extra"
FCFS_LIBRARY=$LIB $B3 > /dev/null 2>&1 && FCFS_LIBRARY=$LIB ncu --set full --clock-control none --import-source on -k regex:k_lattice -s 1 -c 1 -o $O/${T} $B3 > $O/${T}_ncu.log 2>&1
tail -2 $O/${T}_ncu.log
