#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the hot kernels (small single-rank cases with
# and without entry state) and memcheck of the multi-rank loopback cases; logs under gpurun_out/sanitizer/.
mkdir -p gpurun_out/sanitizer
python __graft_entry__.py build > gpurun_out/build.log 2>&1
CS="compute-sanitizer --error-exitcode 1 --print-limit 20"
for es in 1 -1; do
  for tool in memcheck racecheck synccheck; do
    timeout 1200 $CS --tool $tool python tools/sanitize_case.py $es > gpurun_out/sanitizer/${tool}_single_es${es}.log 2>&1
    echo "exit $?" >> gpurun_out/sanitizer/${tool}_single_es${es}.log
  done
done
timeout 1500 $CS --tool memcheck python tools/sanitize_multi.py > gpurun_out/sanitizer/memcheck_multirank.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer/memcheck_multirank.log
timeout 1500 $CS --tool racecheck python tools/sanitize_multi.py > gpurun_out/sanitizer/racecheck_multirank.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer/racecheck_multirank.log
timeout 900 python -m paper_2604_16715_b200.agp --fig5 --config C2 --worlds 2,4 --out gpurun_out/fig5_C2.json > gpurun_out/fig5.log 2>&1
echo "fig5 exit $?" >> gpurun_out/fig5.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
echo done
