#!/bin/bash
# Final-state profile of one round (usage under gpurun: bash tools/final_profile.sh <tag>): ncu launch lists of
# c3 / c4 / c5 and --set full captures of the c3 step's two kernels and the c4 FFT-route kernels (each command
# first exits 0 without ncu).  Bench lines of every config come from tools/final_bench.sh.
set -u
T=${1:-r02v}
O=gpurun_out
NB="--no-cpu-baseline --no-e2e --no-extra"
B3="python bench.py --steps 2 --warmup 1 $NB"
B4="python bench.py --config c4 --steps 1 --warmup 1 $NB"
B5="python bench.py --config c5 --steps 1 --warmup 1 $NB"
$B4 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${T}_launches_c4_fp64.csv $B4 > /dev/null 2>&1
$B5 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${T}_launches_c5_fp64.csv $B5 > /dev/null 2>&1
F="ncu --set full --clock-control none --import-source on"
$B3 > /dev/null 2>&1 && $F -k regex:k_lattice -s 1 -c 1 -o $O/${T}_prof_c3_lattice $B3 > $O/${T}_ncu_f1.log 2>&1
$B3 > /dev/null 2>&1 && $F -k regex:k_clip_corners -s 1 -c 1 -o $O/${T}_prof_c3_extract $B3 > $O/${T}_ncu_f2.log 2>&1
$B4 > /dev/null 2>&1 && $F -k regex:"k_fr_rows|k_fr_fft2" -s 0 -c 2 -o $O/${T}_prof_c4_fp64_fft $B4 > $O/${T}_ncu_f3.log 2>&1
ls -la $O | grep $T
