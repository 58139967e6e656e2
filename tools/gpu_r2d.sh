#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab_r2d.log
for v in "C5 1" "C5 0"; do set -- $v
  echo "=== $1 fp8=$2" >> gpurun_out/ab_r2d.log
  timeout 900 python bench.py --config $1 --kv-fp8 $2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/ab_r2d.log 2>&1
done
echo done
