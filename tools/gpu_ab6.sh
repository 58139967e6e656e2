#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab6.log
for rep in 1 2 3; do for v in c2 c1; do
  echo "=== $v" >> gpurun_out/ab6.log
  GT_LIB=tools/variants/$v/libgt.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab6.log 2>&1
done; done
echo done
