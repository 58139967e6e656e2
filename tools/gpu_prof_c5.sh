#!/bin/bash
# ncu --set full of the three passes on C5 (R-MAT 2^24 / 2^28): DRAM traffic and utilisation.
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
for i in 0 1 2; do
  timeout 900 ncu --set full --clock-control none -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o /tmp/c5_pass$i -f python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c5_prof$i.log 2>&1
  python tools/ncu_summary.py /tmp/c5_pass$i.ncu-rep > gpurun_out/c5_ncu_pass$i.txt 2>&1
done
echo done
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5_bench.log 2>&1
