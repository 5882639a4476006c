#!/bin/bash
# A/B of library variants: bash scripts/gpu_ab.sh TAG "bench args" variants/libgpart_a.so ...
# Each variant is copied over the in-tree libgpart.so (this is the GPU box's scratch copy of
# the repo), so every arm loads its library exactly the way the default does.
cd $GRAFT_REPO_ROOT
TAG=$1; BA=$2; shift 2
mkdir -p gpurun_out
LIB=paper_2105_10312_b200/libgpart.so
cp $LIB /tmp/libgpart_default.so
for lib in "" "$@"; do
  name=$(basename "${lib:-default}" .so)
  cp "${lib:-/tmp/libgpart_default.so}" $LIB
  timeout 600 python bench.py --no-cpu-baseline --no-e2e $BA > gpurun_out/ab_${TAG}_$name.json 2> gpurun_out/ab_${TAG}_$name.err
  python - gpurun_out/ab_${TAG}_$name.json $name <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read()); r = d["roofline"]
    print("%-22s value %.4e ms/step %.3f dom_ms %.3f" % (sys.argv[2], d["value"], d["ms_per_step"], r["dominant_ms_per_step"]))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
cp /tmp/libgpart_default.so $LIB
