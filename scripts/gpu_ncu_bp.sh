#!/bin/bash
# usage: bash scripts/gpu_ncu_bp.sh TAG [bench args]  -- ncu --set full of the c3 exhaustive kernels
cd $GRAFT_REPO_ROOT
TAG=${1:-bp}; shift
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_exh_(memo|bp)" -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu full rc=$?"
