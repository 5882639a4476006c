#!/bin/bash
# Round measurement: full gpu tests, smoke, benches (c3 default + A/B, c2, c4, c5, reference),
# ncu launch list of the c3 bench and ncu --set full of the c3 dominant kernels.
cd $GRAFT_REPO_ROOT
TAG=${1:-round}
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --per-candidate --no-cpu-baseline > gpurun_out/bench_${TAG}_c3_percand.json 2> gpurun_out/bench_${TAG}_c3_percand.err; echo "c3 per-candidate rc=$?"
for cfg in c2 c4 c5; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_$cfg.json 2> gpurun_out/bench_${TAG}_$cfg.err; echo "$cfg rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_${TAG}_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_exh_(memo|bp)" -c 2 -o gpurun_out/prof_${TAG}_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu full rc=$?"
for f in gpurun_out/bench_${TAG}_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read())
except Exception as e:
    print(sys.argv[1], "unreadable", e); sys.exit()
r = d.get("roofline") or {}
print(sys.argv[1].split("/")[-1], "%.3e" % d["value"], "ms/step %.2f" % d["ms_per_step"],
      "frac", r.get("frac"), "exec", (r.get("executed") or {}).get("frac"), "clk", d.get("clocks"))
PY
done
