#!/bin/bash
# GPU suite, then ncu --set full of the three passes (default build) and of the row pass of the TMA
# gather4 variant (tools/variants/tma), for the A/B explanation in DESIGN.md section 6.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for i in 0 1 2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o gpurun_out/prof_pipe$i -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_pipe$i.log 2>&1
done
GT_LIB=tools/variants/tma/libgt.so timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s 4 -c 1 \
     -o gpurun_out/prof_tma_pipe1 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_tma_pipe1.log 2>&1
echo done
