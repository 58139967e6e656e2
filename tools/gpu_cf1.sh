#!/bin/bash
# Column-first backward: parity (world 1 incl. full size, random sweep, state binding, model, multi-rank
# row-first paths), A/B against GT_COLFIRST=0, ncu --set full of its two backward passes.
O=gpurun_out/cf1
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state_binding.py tests/test_gpu_random_sweep.py tests/test_gpu_model.py tests/test_gpu_fp8.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -s > $O/pytest_full.log 2>&1; echo "exit $?" >> $O/pytest_full.log
: > $O/ab.log
for rep in 1 2 3; do for v in 1 0; do
  echo "=== colfirst=$v" >> $O/ab.log
  GT_COLFIRST=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> $O/ab.log 2>&1
done; done
# ncu of the column-first backward passes (launch order per step: fwd, column pass, row pass)
for i in 1 2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o /tmp/prof_cf$i -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/prof_cf$i.log 2>&1
  python tools/ncu_summary.py /tmp/prof_cf$i.ncu-rep > $O/ncu_cf$i.txt 2>&1
  python tools/sass_mix.py 123718280 /tmp/prof_cf$i.ncu-rep > $O/sass_cf$i.txt 2>&1
  ncu -i /tmp/prof_cf$i.ncu-rep --page raw --csv > $O/raw_cf$i.csv 2>&1
done
gzip -f $O/raw_cf*.csv
echo done
