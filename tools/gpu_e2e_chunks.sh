#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/e2e_chunks.log
for c in 4 8 16 32; do
  echo "=== chunks=$c" >> gpurun_out/e2e_chunks.log
  GT_E2E_CHUNKS=$c timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline >> gpurun_out/e2e_chunks.log 2>&1
done
echo done
