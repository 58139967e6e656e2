#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab5.log
for rep in 1 2 3; do for v in win0 win1; do
  echo "=== $v" >> gpurun_out/ab5.log
  GT_LIB=tools/variants/$v/libgt.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab5.log 2>&1
done; done
for v in win0 win1; do
  echo "=== C5 $v" >> gpurun_out/ab5.log
  GT_LIB=tools/variants/$v/libgt.so timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/ab5.log 2>&1
done
echo done
