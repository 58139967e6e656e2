#!/bin/bash
# Tests + A/B bench of kernel variants.  Usage: bash tools/gpu_ab.sh "ENV=.. ENV2=.." "ENV=.." ...
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab.log
for v in "$@"; do
  echo "=== $v" >> gpurun_out/ab.log
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/ab.log 2>&1
done
echo done
