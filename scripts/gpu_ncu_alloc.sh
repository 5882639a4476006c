#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allocate -s 10 -c 5 -o gpurun_out/prof_alloc_c4 python bench.py --config c4 --reps 200 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_alloc_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1
ls -la gpurun_out | tail -5
