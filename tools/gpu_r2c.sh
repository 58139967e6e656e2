#!/bin/bash
# fp8 U=8 + streamed e2e: GPU tests; A/B of fp8 on C3/C5; e2e streamed vs unchunked on C3; racecheck re-run.
mkdir -p gpurun_out/sanitizer
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab_r2c.log
for v in "C5 1" "C3 1"; do set -- $v
  echo "=== $1 fp8=$2" >> gpurun_out/ab_r2c.log
  timeout 900 python bench.py --config $1 --kv-fp8 $2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/ab_r2c.log 2>&1
done
for sm in 0 1; do
  echo "=== e2e stream=$sm" >> gpurun_out/ab_r2c.log
  GT_E2E_STREAM=$sm timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 3 --no-cpu-baseline >> gpurun_out/ab_r2c.log 2>&1
done
CS="compute-sanitizer --error-exitcode 1 --print-limit 20"
for es in 1 -1; do
  timeout 1200 $CS --tool racecheck python tools/sanitize_case.py $es > gpurun_out/sanitizer/racecheck_single_es${es}.log 2>&1
  echo "exit $?" >> gpurun_out/sanitizer/racecheck_single_es${es}.log
done
timeout 1500 $CS --tool racecheck python tools/sanitize_multi.py > gpurun_out/sanitizer/racecheck_multirank.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer/racecheck_multirank.log
echo done
