#!/bin/bash
# ncu --set full of the three pipelined passes (launches 0,1,2 of pipe_kernel after warmup skip)
mkdir -p gpurun_out
python __graft_entry__.py build > /dev/null 2>&1
for i in ${PASSES:-0 1 2}; do
  env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o gpurun_out/prof_pipe$i -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_pipe$i.log 2>&1
done
echo done
