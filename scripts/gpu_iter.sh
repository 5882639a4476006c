#!/bin/bash
# usage: bash scripts/gpu_iter.sh TAG [ncu]
cd $GRAFT_REPO_ROOT
TAG=${1:-iter}
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
if [ "$2" == "ncu" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exhaustive -s 1 -c 1 -o gpurun_out/prof_exh_$TAG python bench.py --steps 1 --warmup 1 --reps 100 --no-e2e --no-cpu-baseline > gpurun_out/ncu_exh_$TAG.log 2>&1
fi
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['events_per_candidate'], d['roofline']['ops_per_unit'], d.get('clocks'))"; tail -3 gpurun_out/bench_$TAG.err
