#!/bin/bash
# Full measurement session for profiles/: bench lines, launch lists, ncu --set full captures.
cd $GRAFT_REPO_ROOT
TAG=${1:-r01}
mkdir -p gpurun_out/$TAG
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/$TAG/smoke.log
timeout 900 python bench.py > gpurun_out/$TAG/bench_c3.json 2> gpurun_out/$TAG/bench_c3.err
timeout 900 python bench.py --config c4 > gpurun_out/$TAG/bench_c4.json 2> gpurun_out/$TAG/bench_c4.err
timeout 900 python bench.py --config c2 --no-cpu-baseline > gpurun_out/$TAG/bench_c2.json 2> gpurun_out/$TAG/bench_c2.err
timeout 900 python bench.py --config c5 --no-cpu-baseline > gpurun_out/$TAG/bench_c5.json 2> gpurun_out/$TAG/bench_c5.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$TAG/bench_reference_c3.json 2> gpurun_out/$TAG/bench_reference_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/$TAG/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/$TAG/ncu_launch_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/$TAG/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/$TAG/ncu_launch_c4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_exhaustive -s 1 -c 1 -o gpurun_out/$TAG/full_exh_c3 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/$TAG/ncu_full_exh.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_allocate -s 5 -c 5 -o gpurun_out/$TAG/full_alloc_c4 python bench.py --config c4 --reps 200 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/$TAG/ncu_full_alloc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_generate -s 1 -c 1 -o gpurun_out/$TAG/full_gen_c4 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/$TAG/ncu_full_gen.log 2>&1
ls -la gpurun_out/$TAG
