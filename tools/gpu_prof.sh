#!/bin/bash
# ncu --set full of the three hot kernels (light-row launches) on the C3 bench workload.
mkdir -p gpurun_out
python __graft_entry__.py build
for k in fwd_kernel rowb_kernel colb_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "${k}" -s 0 -c 1 \
     -o gpurun_out/prof_${k} -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_${k}.log 2>&1
done
echo done
