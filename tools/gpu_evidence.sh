#!/bin/bash
# Round evidence: bench line, ncu launch list of the same bench command, ncu --set full of the
# dominant (column-pass) kernel.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s 5 -c 1 \
   -o gpurun_out/prof_colb -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_colb.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s 4 -c 1 \
   -o gpurun_out/prof_rowb -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_rowb.log 2>&1
echo done
