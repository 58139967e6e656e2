#!/bin/bash
# Round evidence: tests, smoke, bench line, reference arm, ncu launch list of the bench command,
# ncu --set full of the three passes (reports kept in /tmp on the box; text summaries to gpurun_out/).
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; nvidia-smi >> gpurun_out/host.txt 2>&1
python __graft_entry__.py build > gpurun_out/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
fi
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
[ -z "$SKIP_REF" ] && { timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
for i in ${PASSES:-0 1 2}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o /tmp/prof_pass$i -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_pass$i.log 2>&1
  python tools/ncu_summary.py /tmp/prof_pass$i.ncu-rep > gpurun_out/ncu_pass$i.txt 2>&1
  python tools/sass_mix.py 123718280 /tmp/prof_pass$i.ncu-rep > gpurun_out/sass_pass$i.txt 2>&1
  ncu -i /tmp/prof_pass$i.ncu-rep --page details > gpurun_out/details_pass$i.txt 2>&1
  ncu -i /tmp/prof_pass$i.ncu-rep --page raw --csv > gpurun_out/raw_pass$i.csv 2>&1
  ncu -i /tmp/prof_pass$i.ncu-rep --page source --csv --print-source sass > gpurun_out/src_pass$i.csv 2>&1
done
python tools/make_traffic.py C3-products fwd=/tmp/prof_pass0.ncu-rep bwd_rows=/tmp/prof_pass1.ncu-rep bwd_cols=/tmp/prof_pass2.ncu-rep > gpurun_out/traffic.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
du -sh gpurun_out
echo done
