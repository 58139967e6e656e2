#!/bin/bash
mkdir -p gpurun_out
V="base c6 w3 r6"
: > gpurun_out/ab4.log
for rep in 1 2 3; do for v in $V; do
  echo "=== $v" >> gpurun_out/ab4.log
  GT_LIB=tools/variants/$v/libgt.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab4.log 2>&1
done; done
echo done
