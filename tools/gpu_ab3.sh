#!/bin/bash
mkdir -p gpurun_out
V="old new s4"
: > gpurun_out/ab3.log
for rep in 1 2 3; do for v in $V; do
  echo "=== $v" >> gpurun_out/ab3.log
  GT_LIB=tools/variants/$v/libgt.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab3.log 2>&1
done; done
for v in old new; do
  echo "=== C4 $v" >> gpurun_out/ab3.log
  GT_LIB=tools/variants/$v/libgt.so timeout 600 python bench.py --config C4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab3.log 2>&1
done
echo done
