#!/bin/bash
# Per-kernel A/B: ncu launch lists (gpu__time_duration) of the default library and variants
# usage: bash scripts/gpu_ab_kernels.sh TAG "bench args" "kernel regex" variants/lib_a.so ...
cd $GRAFT_REPO_ROOT
TAG=$1; BA=$2; KR=$3; shift 3
mkdir -p gpurun_out
for lib in "" "$@"; do
  name=$(basename "${lib:-default}" .so)
  GP_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$KR" -c 40 --csv --log-file gpurun_out/abk_${TAG}_$name.csv python bench.py --no-cpu-baseline --no-e2e --no-direct --steps 1 --warmup 1 $BA > /dev/null 2>&1
  echo "== $name"; python scripts/ncu_summary.py --launches gpurun_out/abk_${TAG}_$name.csv | head -12
done
