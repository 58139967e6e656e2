#!/bin/bash
# fp8 K/V option: GPU tests, then A/B bench lines (bf16 vs kv_fp8) on C3 and C5, and the fast suite.
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fp8.py -m gpu -q -x -s > gpurun_out/pytest_fp8.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fp8.log
: > gpurun_out/ab_fp8.log
for cfg in C3 C5; do for fp8 in 0 1; do
  echo "=== $cfg fp8=$fp8" >> gpurun_out/ab_fp8.log
  timeout 900 python bench.py --config $cfg --kv-fp8 $fp8 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/ab_fp8.log 2>&1
done; done
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fullsize and not fp8" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
echo done
