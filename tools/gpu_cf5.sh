#!/bin/bash
# Stage-wide (LSE2, D) gather in the column pass: parity + bitwise column-first test, A/B vs the previous build.
O=gpurun_out/cf5
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
: > $O/ab.log
for rep in 1 2 3; do for v in main head; do
  echo "=== $v" >> $O/ab.log
  if [ $v = main ]; then L=paper_2604_16715_b200/libgt.so; else L=tools/variants/$v/libgt.so; fi
  GT_LIB=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> $O/ab.log 2>&1
done; done
echo done
