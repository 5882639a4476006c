#!/bin/bash
# per-variant k_allocate durations (ncu launch list) with and without the wave table, C4 at 10^5 sets
cd $GRAFT_REPO_ROOT
BENCH_ARGS=${BENCH_ARGS:---config c4 --reps 2000}
mkdir -p gpurun_out
for kb in 100 0; do
  GP_ALLOC_TAB_KB=$kb timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_allocate -c 10 --csv --log-file gpurun_out/tab_$kb.csv python bench.py $BENCH_ARGS --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python - gpurun_out/tab_$kb.csv $kb <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hd = rows[h]; ki = hd.index('Kernel Name'); vi = hd.index('Metric Value')
v = [(r[ki].split('(')[0][-12:], round(float(r[vi]) / 1e3)) for r in rows[h + 1:] if len(r) > vi]
print("tab_kb", sys.argv[2], v[5:10], "sum", sum(x[1] for x in v[5:10]))
PY
done
