#!/bin/bash
# Full GPU tests + kernel-only bench lines of the other full-size configs (C4 Reddit, C5 R-MAT).
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "exit $?" >> gpurun_out/bench_$c.log
done
echo done
