#!/bin/bash
# usage: bash scripts/gpu_bench_all.sh TAG
cd $GRAFT_REPO_ROOT
TAG=${1:-all}
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
for cfg in c3 c2 c4 c5; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 2 ${EXTRA} > gpurun_out/bench_${TAG}_$cfg.json 2> gpurun_out/bench_${TAG}_$cfg.err
  echo "$cfg rc=$?"; python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_${TAG}_$cfg.json').read())
r=d['roofline']; print('$cfg', '%.3e'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'frac %.4f'%r['frac'], 'dom_ms %.2f'%r['dominant_ms_per_step'], 'cpu', d.get('cpu_baseline',{}).get('value'), 'e2e', d.get('e2e',{}).get('value'))
" ; tail -2 gpurun_out/bench_${TAG}_$cfg.err
done
