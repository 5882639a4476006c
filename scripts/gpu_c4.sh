#!/bin/bash
# C4 heuristics check: allocate parity tests + C4/C3 bench lines (+ optional launch list)
cd $GRAFT_REPO_ROOT
TAG=${1:-c4}
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "allocate" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-direct > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err; echo "c3 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_allocate -c 10 --csv --log-file gpurun_out/launches_${TAG}_c4.csv python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
python - gpurun_out/bench_${TAG}_c4.json gpurun_out/bench_${TAG}_c3.json <<'PY'
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read()); r = d["roofline"]
        print(f, "value %.4e ms/step %.2f dom_ms %.2f frac %.4f" % (d["value"], d["ms_per_step"], r["dominant_ms_per_step"], r["frac"]),
              {k: r[k] for k in r if k.endswith("per_step") and isinstance(r[k], (int, float))})
    except Exception as e:
        print(f, "failed", e)
PY
python scripts/ncu_summary.py --launches gpurun_out/launches_${TAG}_c4.csv 2>/dev/null | head -12
