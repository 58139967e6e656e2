#!/bin/bash
# Round-2 evidence pass: full-size parity (C3, C3f, C4, C5 with the stratified samples), the fast GPU
# suite, the default bench line (with e2e and cpu_baseline), then ncu of the three passes.
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s > gpurun_out/pytest_fullsize.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fullsize.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_full.log
PASSES="0 1 2" SKIP_TESTS= bash tools/gpu_quick.sh
