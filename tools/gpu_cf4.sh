#!/bin/bash
# Column-first column pass register budget: 5 CTAs/SM cap (default, 87 registers) vs 4 (96 registers).
O=gpurun_out/cf4
mkdir -p $O
: > $O/ab.log
for rep in 1 2 3; do for v in main cfm4; do
  echo "=== $v" >> $O/ab.log
  if [ $v = main ]; then L=paper_2604_16715_b200/libgt.so; else L=tools/variants/$v/libgt.so; fi
  GT_LIB=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> $O/ab.log 2>&1
done; done
echo done
