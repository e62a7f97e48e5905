O=gpurun_out
NB="--no-cpu-baseline --no-e2e --no-extra"
timeout 300 python bench.py --form edge --steps 10 --warmup 3 $NB > $O/r02z_bench_c3_edges.json 2>/dev/null
timeout 300 python bench.py --form corner --steps 10 --warmup 3 $NB > $O/r02z_bench_c3_corners.json 2>/dev/null
timeout 300 python bench.py --prec f16x3 --steps 10 --warmup 3 $NB > $O/r02z_bench_c3_f16x3.json 2>/dev/null
timeout 300 python bench.py --input polygons --steps 10 --warmup 3 $NB > $O/r02z_bench_c3_polygons.json 2>/dev/null
for c in c1 c2 c4 c5; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-extra > $O/r02z_bench_${c}_fp64.json 2>/dev/null; done
timeout 300 python bench.py --config c1 --no-small --steps 10 --warmup 3 $NB > $O/r02z_bench_c1_general.json 2>/dev/null
timeout 300 python bench.py --config c2 --no-graph --steps 10 --warmup 3 $NB > $O/r02z_bench_c2_nograph.json 2>/dev/null
for c in c2 c4 c5; do timeout 300 python bench.py --config $c --prec tf32x3 --steps 5 --warmup 3 $NB > $O/r02z_bench_${c}_tf32x3.json 2>/dev/null; done
timeout 300 python bench.py --config c4 --route gemm --steps 5 --warmup 3 $NB > $O/r02z_bench_c4_fp64_gemm.json 2>/dev/null
timeout 300 python bench.py --config layout --steps 5 --warmup 3 --no-cpu-baseline --no-extra > $O/r02z_bench_layout.json 2>/dev/null
timeout 300 python bench.py --config haar --steps 5 --warmup 3 > $O/r02z_bench_haar.json 2>/dev/null
echo done
