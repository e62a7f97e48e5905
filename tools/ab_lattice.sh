# A/B of lattice-kernel builds on c3 (usage under gpurun: bash tools/ab_lattice.sh <variant tag> ...)
O=gpurun_out
V=paper_1010_5562_b200/variants
python -m pytest tests -m gpu -q -x -k "lattice" > $O/ab_test_default.log 2>&1; tail -1 $O/ab_test_default.log
for t in "$@"; do FCFS_LIBRARY=$V/libfcfs_$t.so python -m pytest tests -m gpu -q -x -k "lattice" > $O/ab_test_$t.log 2>&1; echo "$t: $(tail -1 $O/ab_test_$t.log)"; done
NB="--no-cpu-baseline --no-e2e --no-extra --steps 20 --warmup 5"
for i in 1 2; do
for lib in paper_1010_5562_b200/libfcfs.so $(for t in "$@"; do echo $V/libfcfs_$t.so; done); do
  FCFS_LIBRARY=$lib timeout 300 python bench.py $NB > $O/ab_$(basename $lib .so)_$i.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('$O/ab_$(basename $lib .so)_$i.json').read().strip().splitlines()[-1]);print('$(basename $lib)',d['value'],d['ms_per_step'],d['roofline']['stage_ms_per_step'])"
done; done
