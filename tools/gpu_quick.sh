#!/bin/bash
# Quick iteration: build, fast GPU tests (no full-size), bench line (kernel-only), optional ncu passes
# (PASSES="0 1 2"): summary, SASS mix, source page, and the per-pass counters bench.py reads
# (gpurun_out/ncu_traffic.json, merged into profiles/ncu_traffic.json by the caller).
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
[ -z "$SKIP_TESTS" ] && { timeout 600 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log; }
timeout 600 python bench.py --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
# pipe_kernel launches per step: fwd, then the backward passes in the plan's order (world 1: column pass
# first unless GT_COLFIRST=0)
if [ "${GT_COLFIRST:-1}" = "0" ]; then NAMES=(fwd bwd_rows bwd_cols); else NAMES=(fwd bwd_cols bwd_rows); fi
WL=${WL:-C3-products}
for i in ${PASSES}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o /tmp/prof_pass$i -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/prof_pass$i.log 2>&1
  python tools/ncu_summary.py /tmp/prof_pass$i.ncu-rep > gpurun_out/ncu_pass$i.txt 2>&1
  python tools/sass_mix.py ${UNITS:-123718280} /tmp/prof_pass$i.ncu-rep > gpurun_out/sass_pass$i.txt 2>&1
  ncu -i /tmp/prof_pass$i.ncu-rep --page source --csv --print-source sass > gpurun_out/src_pass$i.csv 2>&1
  ncu -i /tmp/prof_pass$i.ncu-rep --page raw --csv > gpurun_out/raw_pass$i.csv 2>&1
  python tools/make_traffic.py --out gpurun_out/ncu_traffic.json $WL ${NAMES[$i]}=gpurun_out/raw_pass$i.csv >> gpurun_out/ncu_pass$i.txt 2>&1
done
echo done
