#!/bin/bash
# compute-sanitizer over small parity tests (memcheck, racecheck, synccheck):
#   bash scripts/gpu_sanitize.sh TAG   -> gpurun_out/TAG/compute_sanitizer_*.log
cd $GRAFT_REPO_ROOT
T=${1:-san}; O=gpurun_out/$T; mkdir -p $O
python -c "import oracle; oracle.build()" > /dev/null
K="c1 or exhaustive_random_sets or allocate_random_sets or f4_masks_random or threshold_random or pipeline_step or contract_violation or large_n"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests -m gpu -q -x -k "$K" -p no:cacheprovider > $O/compute_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $O/compute_sanitizer_$tool.log
  tail -3 $O/compute_sanitizer_$tool.log
done
