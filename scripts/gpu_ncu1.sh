#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exhaustive -s 1 -c 1 -o gpurun_out/prof_exh python bench.py --steps 1 --warmup 1 --reps 100 --no-e2e --no-cpu-baseline > gpurun_out/ncu_exh.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allocate -s 5 -c 2 -o gpurun_out/prof_alloc python bench.py --steps 1 --warmup 1 --reps 100 --no-e2e --no-cpu-baseline > gpurun_out/ncu_alloc.log 2>&1
ls -la gpurun_out
