#!/bin/bash
# One GPU session of measurements for profiles/: bench lines (no profiler), the launch list of the
# default c3 step, and ncu --set full captures of the dominant kernels.  Usage (under gpurun):
#   bash tools/round_profile.sh <tag>
set -u
T=${1:-r01}
O=gpurun_out
B3="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
B4="python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 python bench.py --steps 10 --warmup 3 > $O/${T}_bench_c3.json 2> $O/${T}_bench_c3.err
for c in c1 c2 c4 c5; do
  timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > $O/${T}_bench_${c}_fp64.json 2>/dev/null
done
timeout 300 python bench.py --config c4 --prec tf32x3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/${T}_bench_c4_tf32x3.json 2>/dev/null
timeout 300 python bench.py --prec f16x3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${T}_bench_c3_f16x3.json 2>/dev/null
$B3 > $O/plain3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/${T}_launches_c3.csv $B3 > $O/ncu_a.log 2>&1
$B3 > $O/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gemm_tf32 -s 1 -c 1 -o $O/${T}_prof_c3_tf32 $B3 > $O/ncu_b.log 2>&1
$B3 > $O/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_clip_corners -s 1 -c 1 -o $O/${T}_prof_c3_extract $B3 > $O/ncu_c.log 2>&1
$B4 > $O/plain4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/${T}_launches_c4.csv $B4 > $O/ncu_d.log 2>&1
$B4 > $O/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_gemm_fp64|k_gsum_fp64" -s 4 -c 2 -o $O/${T}_prof_c4_fp64 $B4 > $O/ncu_e.log 2>&1
ls -la $O | tail -30
