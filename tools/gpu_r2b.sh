#!/bin/bash
# New-feature GPU checks: graph-transformer model tests, multi-process host-IPC tests, L2 microbenchmark,
# bench line.
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
./tools/l2bw 32 40 > gpurun_out/l2bw.json 2>&1; ./tools/l2bw 96 16 >> gpurun_out/l2bw.json 2>&1
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_multiproc.py -m gpu -q -x > gpurun_out/pytest_new.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_new.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
