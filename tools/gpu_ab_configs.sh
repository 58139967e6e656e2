#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pytest.log
: > gpurun_out/ab.log
for rep in 1 2; do
for v in "X=0" "GT_LIB=tools/variants/old/libgt.so"; do
  for c in C3 C2; do
    echo "=== $v $c" >> gpurun_out/ab.log
    env $v timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab.log 2>&1
  done
done
done
python - <<'PY' >> gpurun_out/ab.log
import json
cur=None
for l in open('gpurun_out/ab.log'):
    if l.startswith('=== '): cur=l[4:].strip()
    elif l.startswith('{'):
        d=json.loads(l); print('SUMMARY', cur, round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items() if v}, 'sm_mhz', (d.get('clocks') or {}).get('sm_mhz'))
PY
