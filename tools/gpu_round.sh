#!/bin/bash
# GPU tests (incl. full-size sampled parity) + ncu full of the three passes (one report each).
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for i in ${PASSES:-0 1 2}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o gpurun_out/prof_pass$i -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_pass$i.log 2>&1
done
echo done
