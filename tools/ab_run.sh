# A/B of library builds (usage under gpurun: bash tools/ab_run.sh "<pytest -k expr>" "<bench args>" <variant tag> ...)
O=gpurun_out
V=paper_1010_5562_b200/variants
K="$1"; BA="$2"; shift 2
for t in default "$@"; do
  L=paper_1010_5562_b200/libfcfs.so; [ $t != default ] && L=$V/libfcfs_$t.so
  FCFS_LIBRARY=$L python -m pytest tests -m gpu -q -x -k "$K" > $O/ab_test_$t.log 2>&1; echo "$t: $(tail -1 $O/ab_test_$t.log)"
done
for i in 1 2; do for t in default "$@"; do
  L=paper_1010_5562_b200/libfcfs.so; [ $t != default ] && L=$V/libfcfs_$t.so
  FCFS_LIBRARY=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-extra $BA > $O/ab_$t_$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/ab_$t_$i.json').read().strip().splitlines()[-1]);print('$t',d['value'],d['ms_per_step'],d['roofline']['stage_ms_per_step'])"
done; done
