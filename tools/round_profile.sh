#!/bin/bash
# One GPU session of measurements for profiles/: bench lines (no profiler), launch lists and
# ncu --set full captures of the dominant kernels.  Usage (under gpurun): bash tools/round_profile.sh <tag>
set -u
T=${1:-r01}
O=gpurun_out
NB="--no-cpu-baseline --no-e2e --no-extra"
# ---- bench lines (each command exits before any profiler run of the same command)
timeout 900 python bench.py --steps 10 --warmup 3 > $O/${T}_bench_c3.json 2> $O/${T}_bench_c3.err
timeout 300 python bench.py --form edge --steps 10 --warmup 3 $NB > $O/${T}_bench_c3_edges.json 2>/dev/null
timeout 300 python bench.py --config c1 --no-small --steps 10 --warmup 3 --no-cpu-baseline > $O/${T}_bench_c1_general.json 2>/dev/null
timeout 300 python bench.py --prec f16x3 --steps 10 --warmup 3 $NB > $O/${T}_bench_c3_f16x3.json 2>/dev/null
timeout 300 python bench.py --form corner --steps 10 --warmup 3 $NB > $O/${T}_bench_c3_corners.json 2>/dev/null
for c in c1 c2 c4 c5; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/${T}_bench_${c}_fp64.json 2>/dev/null
done
for c in c4 c5; do for p in tf32x3 f16x3; do
  timeout 300 python bench.py --config $c --prec $p --steps 5 --warmup 3 $NB > $O/${T}_bench_${c}_${p}.json 2>/dev/null
done; done
timeout 300 python bench.py --route gemm --config c4 --steps 5 --warmup 3 $NB > $O/${T}_bench_c4_fp64_gemm.json 2>/dev/null
timeout 300 python bench.py --route gemm --config c4 --prec tf32x3 --steps 5 --warmup 3 $NB > $O/${T}_bench_c4_tf32x3_gemm.json 2>/dev/null
timeout 300 python bench.py --config layout --steps 5 --warmup 3 --no-cpu-baseline > $O/${T}_bench_layout.json 2>/dev/null
timeout 300 python bench.py --config haar --steps 5 --warmup 3 > $O/${T}_bench_haar.json 2>/dev/null
timeout 300 python bench.py --input polygons --steps 5 --warmup 3 $NB > $O/${T}_bench_c3_polygons.json 2>/dev/null
# ---- launch lists (serialised, cold; shares not absolutes)
B3="python bench.py --steps 2 --warmup 1 $NB"
B4="python bench.py --config c4 --steps 1 --warmup 1 $NB"
B5="python bench.py --config c5 --steps 1 --warmup 1 $NB"
$B3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/${T}_launches_c3.csv $B3 > $O/ncu_l3.log 2>&1
$B4 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${T}_launches_c4_fp64.csv $B4 > $O/ncu_l4.log 2>&1
$B5 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${T}_launches_c5_fp64.csv $B5 > $O/ncu_l5.log 2>&1
# ---- ncu --set full of the dominant kernels
F="ncu --set full --clock-control none --import-source on"
$B3 > /dev/null 2>&1 && $F -k regex:k_lattice -s 1 -c 1 -o $O/${T}_prof_c3_lattice $B3 > $O/ncu_f1.log 2>&1
$B3 --form edge > /dev/null 2>&1 && $F -k regex:k_gemm_tf32 -s 1 -c 1 -o $O/${T}_prof_c3_tf32 $B3 --form edge > $O/ncu_f1e.log 2>&1
B1="python bench.py --config c1 --steps 2 --warmup 1 $NB"
$B1 > /dev/null 2>&1 && $F -k regex:k_small_clip -s 1 -c 1 -o $O/${T}_prof_c1_small $B1 > $O/ncu_f1s.log 2>&1
$B3 > /dev/null 2>&1 && $F -k regex:k_clip_corners -s 1 -c 1 -o $O/${T}_prof_c3_extract $B3 > $O/ncu_f2.log 2>&1
$B3 --form edge > /dev/null 2>&1 && $F -k regex:k_edges -s 1 -c 1 -o $O/${T}_prof_c3_edges $B3 --form edge > $O/ncu_f2e.log 2>&1
$B4 > /dev/null 2>&1 && $F -k regex:"k_fr_rows|k_fr_fft2|k_fr_row0" -s 0 -c 4 -o $O/${T}_prof_c4_fp64_fft $B4 > $O/ncu_f3.log 2>&1
$B4 --route gemm > /dev/null 2>&1 && $F -k regex:"k_gemm_fp64|k_gsum_fp64|k_hsum_fp64" -s 0 -c 3 -o $O/${T}_prof_c4_fp64_gemm $B4 --route gemm > $O/ncu_f4.log 2>&1
B4t="python bench.py --config c4 --prec tf32x3 --steps 1 --warmup 1 $NB"
$B4t --route gemm > /dev/null 2>&1 && $F -k regex:"k_gemm_tf32|k_gsum_tc|k_hsum_tc" -s 0 -c 3 -o $O/${T}_prof_c4_tf32_gemm $B4t --route gemm > $O/ncu_f5.log 2>&1
B4t2="python bench.py --config c4 --prec tf32x3 --steps 1 --warmup 1 $NB"
$B4t2 > /dev/null 2>&1 && $F -k regex:"k_fr_rows|k_fr_fft2" -s 0 -c 2 -o $O/${T}_prof_c4_f32_fft $B4t2 > $O/ncu_f6.log 2>&1
BL="python bench.py --config layout --steps 1 --warmup 1 $NB"
$BL > /dev/null 2>&1 && $F -k regex:"k_chop" -s 0 -c 4 -o $O/${T}_prof_layout_chop $BL > $O/ncu_f7.log 2>&1
BH="python bench.py --config haar --steps 1 --warmup 1 --no-cpu-baseline"
$BH > /dev/null 2>&1 && $F -k regex:"k_haar" -s 0 -c 3 -o $O/${T}_prof_haar $BH > $O/ncu_f8.log 2>&1
BP="python bench.py --input polygons --steps 1 --warmup 1 $NB"
$BP > /dev/null 2>&1 && $F -k regex:"k_clip_polygons" -s 0 -c 1 -o $O/${T}_prof_c3_polygons $BP > $O/ncu_f9.log 2>&1
ls -la $O | grep $T
