#!/bin/bash
# Final round-2 evidence for the committed kernels (second session): whole GPU suite, smoke, default bench
# line, C4 / C5 bench lines with e2e and CPU baselines, ncu launch list of the default bench command,
# ncu --set full of the three passes (refreshes the per-pass counters bench.py reads).
O=gpurun_out/${FINAL_DIR:-final2}
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s > $O/pytest_gpu_all.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "exit $?" >> $O/bench_default.log
for c in C4 C5; do
  timeout 1200 python bench.py --config $c > $O/bench_$c.log 2>&1; echo "exit $?" >> $O/bench_$c.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_c3.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches_bench.log 2>&1
PASSES="0 1 2" SKIP_TESTS=1 bash tools/gpu_quick.sh
for f in ncu_pass0.txt ncu_pass1.txt ncu_pass2.txt sass_pass0.txt sass_pass1.txt sass_pass2.txt ncu_traffic.json bench.log; do mv gpurun_out/$f $O/ 2>/dev/null; done
gzip -f gpurun_out/raw_pass*.csv 2>/dev/null; mv gpurun_out/raw_pass*.csv.gz $O/ 2>/dev/null; rm -f gpurun_out/src_pass*.csv
echo done
