#!/bin/bash
# exhaustive evaluators: parity tests + C3/C2 bench (bit-sliced default, per-candidate A/B)
cd $GRAFT_REPO_ROOT
TAG=${1:-exh}
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -k "exhaustive or smoke or threshold or pipeline" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -4 gpurun_out/pytest_$TAG.log
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_$cfg.json 2> gpurun_out/bench_${TAG}_$cfg.err
  echo "$cfg rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/bench_${TAG}_$cfg.json').read())
r=d['roofline']; print('$cfg', '%.3e'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'frac %.4f'%r['frac'], 'dom', r.get('kernel'), 'dom_ms %.2f'%r['dominant_ms_per_step'], 'e2e %.3e'%d['e2e']['value'])
"; tail -2 gpurun_out/bench_${TAG}_$cfg.err
done
GP_EXH_PERCAND=1 timeout 600 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c3_percand.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/bench_${TAG}_c3_percand.json').read()); print('c3 per-candidate', '%.3e'%d['value'], 'ms/step %.2f'%d['ms_per_step'])
"
