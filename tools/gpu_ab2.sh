#!/bin/bash
# A/B of pipeline parameters (one-shape builds), 2 interleaved rounds, 20 steps each.
mkdir -p gpurun_out
V="base g1 g4 w2 w8 s3 carve"
: > gpurun_out/ab2.log
for rep in 1 2; do for v in $V; do
  echo "=== $v" >> gpurun_out/ab2.log
  GT_LIB=tools/variants/$v/libgt.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab2.log 2>&1
done; done
echo done
