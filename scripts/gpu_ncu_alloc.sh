#!/bin/bash
# ncu --set full of k_allocate (c3: 5 variants; c4: 5 variants at 10^5 sets) and k_generate (c4)
cd $GRAFT_REPO_ROOT
TAG=${1:-al}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allocate -c 5 -o gpurun_out/prof_${TAG}_alloc_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_a3.log 2>&1; echo "ncu alloc c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allocate -c 5 -o gpurun_out/prof_${TAG}_alloc_c4 python bench.py --config c4 --reps 2000 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_a4.log 2>&1; echo "ncu alloc c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_generate -c 1 -o gpurun_out/prof_${TAG}_gen_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_g4.log 2>&1; echo "ncu gen c4 rc=$?"
