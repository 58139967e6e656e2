#!/bin/bash
# Re-entry check of HEAD: GPU suite, smoke, default bench line.
mkdir -p gpurun_out/verify
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/verify/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/verify/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/verify/smoke.log
timeout 900 python bench.py > gpurun_out/verify/bench_default.log 2>&1; echo "exit $?" >> gpurun_out/verify/bench_default.log
echo done
