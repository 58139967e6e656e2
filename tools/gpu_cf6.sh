#!/bin/bash
# Column-first row pass occupancy: uncapped (63 registers, 8 CTAs/SM) vs 10 CTAs/SM (48 registers).
O=gpurun_out/cf6
mkdir -p $O
: > $O/ab.log
for rep in 1 2 3; do for v in main cfr10; do
  echo "=== $v" >> $O/ab.log
  if [ $v = main ]; then L=paper_2604_16715_b200/libgt.so; else L=tools/variants/$v/libgt.so; fi
  GT_LIB=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> $O/ab.log 2>&1
done; done
GT_LIB=tools/variants/cfr10/libgt.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "column_first or power_law or star" > $O/pytest_cfr10.log 2>&1; echo "exit $?" >> $O/pytest_cfr10.log
echo done
