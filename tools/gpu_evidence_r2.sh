#!/bin/bash
# Round-2 evidence: default bench line, ncu launch list of the same command, ncu --set full of the three
# passes (refreshing profiles/ncu_traffic.json), C4 / C5 full bench lines, sanitizers, L2 microbench, Fig. 5.
mkdir -p gpurun_out/sanitizer gpurun_out/configs
python __graft_entry__.py build > gpurun_out/build.log 2>&1
./tools/l2bw 32 400 > gpurun_out/l2bw.json 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "exit $?" >> gpurun_out/bench_default.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
PASSES="0 1 2" SKIP_TESTS=1 bash tools/gpu_quick.sh
for cfg in C4 C5; do
  timeout 1500 python bench.py --config $cfg > gpurun_out/configs/bench_$cfg.log 2>&1; echo "exit $?" >> gpurun_out/configs/bench_$cfg.log
done
CS="compute-sanitizer --error-exitcode 1 --print-limit 20"
for tool in memcheck racecheck synccheck; do
  for es in 1 -1; do
    timeout 1200 $CS --tool $tool python tools/sanitize_case.py $es > gpurun_out/sanitizer/${tool}_single_es${es}.log 2>&1
    echo "exit $?" >> gpurun_out/sanitizer/${tool}_single_es${es}.log
  done
  timeout 1200 $CS --tool $tool python tools/sanitize_case.py 1 fp8 > gpurun_out/sanitizer/${tool}_single_fp8.log 2>&1
  echo "exit $?" >> gpurun_out/sanitizer/${tool}_single_fp8.log
done
timeout 1500 $CS --tool memcheck python tools/sanitize_multi.py > gpurun_out/sanitizer/memcheck_multirank.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer/memcheck_multirank.log
timeout 900 python -m paper_2604_16715_b200.agp --fig5 --config C2 --worlds 2,4 --out gpurun_out/fig5_C2.json > gpurun_out/fig5.log 2>&1
echo done
