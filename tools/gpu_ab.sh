#!/bin/bash
# Fast GPU tests + A/B bench of kernel variants (2 runs each, interleaved).
# Usage: bash tools/gpu_ab.sh "ENV=.. ENV2=.." "ENV=.." ...   (e.g. GT_LIB=tools/variants/x/libgt.so)
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
[ -z "$SKIP_TESTS" ] && { timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log; }
: > gpurun_out/ab.log
for rep in 1 2; do
for v in "$@"; do
  echo "=== $v" >> gpurun_out/ab.log
  env $v timeout 600 python bench.py --steps ${AB_STEPS:-30} --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab.log 2>&1
done
done
python - <<'PY' >> gpurun_out/ab.log
import json
cur=None
for l in open('gpurun_out/ab.log'):
    if l.startswith('=== '): cur=l[4:].strip()
    elif l.startswith('{'):
        d=json.loads(l); print('SUMMARY', cur or 'default', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items() if v}, 'sm_mhz', (d.get('clocks') or {}).get('sm_mhz'))
PY
echo done
