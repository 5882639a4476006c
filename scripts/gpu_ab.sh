#!/bin/bash
# A/B of library variants: bash scripts/gpu_ab.sh TAG "bench args" variants/libgpart_a.so ...
cd $GRAFT_REPO_ROOT
TAG=$1; BA=$2; shift 2
mkdir -p gpurun_out
for lib in "" "$@"; do
  name=$(basename "${lib:-default}" .so)
  GP_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e $BA > gpurun_out/ab_${TAG}_$name.json 2> gpurun_out/ab_${TAG}_$name.err
  python - gpurun_out/ab_${TAG}_$name.json $name <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read()); r = d["roofline"]
    print("%-22s value %.4e ms/step %.3f dom_ms %.3f" % (sys.argv[2], d["value"], d["ms_per_step"], r["dominant_ms_per_step"]))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
