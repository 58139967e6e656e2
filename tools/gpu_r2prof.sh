#!/bin/bash
# GPU suite, then ncu --set full of the three passes (default build) and of the row pass of the TMA
# gather4 variant (tools/variants/tma).  Reports are reduced to CSV pages on the box (size limit).
mkdir -p gpurun_out
[ -z "$SKIP_TESTS" ] && { timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log; }
prof() {  # name skip [env]
  env $3 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $2 -c 1 \
     -o /tmp/$1 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_src.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
}
for i in ${PASSES:-0 1 2}; do prof prof_pipe$i $((3+i)); done
[ -n "$TMA" ] && prof prof_tma_pipe1 4 GT_LIB=tools/variants/tma/libgt.so
du -sh gpurun_out
echo done
