#!/bin/bash
# Full round check: gpu tests, smoke, default bench, per-config benches, reference arm.
cd $GRAFT_REPO_ROOT
TAG=${1:-full}
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err; echo "default rc=$?"
cat gpurun_out/bench_${TAG}_default.json
for cfg in c2 c4 c5; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_$cfg.json 2> gpurun_out/bench_${TAG}_$cfg.err
  echo "$cfg rc=$?"; head -c 400 gpurun_out/bench_${TAG}_$cfg.json; echo
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err; echo "ref rc=$?"
cat gpurun_out/bench_${TAG}_reference.json
