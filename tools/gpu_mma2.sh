#!/bin/bash
# Per-pass A/B of the tensor-core consumer (GT_PIPE_MMA bit p = pass p): 7 (main lib), 6, 4, 2, 0.
mkdir -p gpurun_out/mma2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/mma2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/mma2/pytest.log
: > gpurun_out/mma2/ab.log
for rep in 1 2; do for v in m7 fma m6 m4 m2; do
  echo "=== $v" >> gpurun_out/mma2/ab.log
  if [ $v = m7 ]; then L=paper_2604_16715_b200/libgt.so; else L=tools/variants/$v/libgt.so; fi
  GT_LIB=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/mma2/ab.log 2>&1
done; done
echo done
