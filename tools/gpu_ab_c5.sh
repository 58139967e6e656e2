#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
: > gpurun_out/ab.log
for rep in 1 2; do
for v in "X=0" "GT_LIB=tools/variants/g2/libgt.so" "GT_LIB=tools/variants/g4/libgt.so"; do
  for c in ${CONFIGS:-C5 C3}; do
    echo "=== $v $c" >> gpurun_out/ab.log
    env $v timeout 900 python bench.py --config $c --steps ${AB_STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/ab.log 2>&1
  done
done
done
python - <<'PY' >> gpurun_out/ab.log
import json
cur=None
for l in open('gpurun_out/ab.log'):
    if l.startswith('=== '): cur=l[4:].strip()
    elif l.startswith('{'):
        d=json.loads(l); print('SUMMARY', cur, round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items() if v}, 'sm_mhz', (d.get('clocks') or {}).get('sm_mhz'))
PY
