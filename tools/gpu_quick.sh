#!/bin/bash
# Quick iteration: build, fast GPU tests (no full-size), bench line (kernel-only), optional ncu passes.
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
for i in ${PASSES}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o /tmp/prof_pass$i -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_pass$i.log 2>&1
  python tools/ncu_summary.py /tmp/prof_pass$i.ncu-rep > gpurun_out/ncu_pass$i.txt 2>&1
  python tools/sass_mix.py 123718280 /tmp/prof_pass$i.ncu-rep > gpurun_out/sass_pass$i.txt 2>&1
  ncu -i /tmp/prof_pass$i.ncu-rep --page source --csv --print-source sass > gpurun_out/src_pass$i.csv 2>&1
done
echo done
