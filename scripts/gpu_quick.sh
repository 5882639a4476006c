#!/bin/bash
# usage: bash scripts/gpu_quick.sh TAG "pytest -k expr" [bench args...]
cd $GRAFT_REPO_ROOT
TAG=${1:-quick}; K=${2:-exhaustive}; shift 2
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > /dev/null
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - gpurun_out/bench_$TAG.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read()); r = d["roofline"]
print("value %.4e ms/step %.3f dom_ms %.3f frac %.3f e2e %.4e launches %s" % (d["value"], d["ms_per_step"], r["dominant_ms_per_step"], r["frac"], d["e2e"]["value"], d["gpu_launches"]))
PY
if [ -n "$GP_LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > /dev/null 2>&1; echo "ncu launches rc=$?"
python scripts/ncu_summary.py --launches gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt; head -8 gpurun_out/launches_$TAG.txt
fi
