#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_hot.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_hot.log
: > gpurun_out/ab_hot.log
for v in "C5 0" "C5 65536" "C5 131072" "C3 0" "C3 65536"; do set -- $v
  echo "=== $1 hot=$2" >> gpurun_out/ab_hot.log
  timeout 900 python bench.py --config $1 --hot-cols $2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/ab_hot.log 2>&1
done
echo done
