#!/bin/bash
# Final round-2 evidence for the committed kernels: whole GPU suite (incl. full-size), smoke, default
# bench line, ncu launch list of the same command, ncu --set full of the three passes.
mkdir -p gpurun_out/final
python __graft_entry__.py build > gpurun_out/final/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/final/pytest_gpu_all.log 2>&1; echo "pytest exit $?" >> gpurun_out/final/pytest_gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench_default.log 2>&1; echo "exit $?" >> gpurun_out/final/bench_default.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/launches_bench.log 2>&1
PASSES="0 1 2" SKIP_TESTS=1 bash tools/gpu_quick.sh
echo done
