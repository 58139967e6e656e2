#!/bin/bash
# Column-first backward (third cut: hoisted lane constants): bitwise test vs row-first, parity, A/B,
# ncu of the column pass.
O=gpurun_out/cf3
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state_binding.py tests/test_gpu_random_sweep.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
: > $O/ab.log
for rep in 1 2 3; do for v in 1 0; do
  echo "=== colfirst=$v" >> $O/ab.log
  GT_COLFIRST=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> $O/ab.log 2>&1
done; done
NAMES=(fwd bwd_cols bwd_rows)
ARGS=""
for i in 0 1 2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pipe_kernel" -s $((3+i)) -c 1 \
     -o /tmp/prof_cf$i -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/prof_cf$i.log 2>&1
  python tools/ncu_summary.py /tmp/prof_cf$i.ncu-rep > $O/ncu_${NAMES[$i]}.txt 2>&1
  python tools/sass_mix.py 123718280 /tmp/prof_cf$i.ncu-rep > $O/sass_${NAMES[$i]}.txt 2>&1
  ncu -i /tmp/prof_cf$i.ncu-rep --page raw --csv > $O/raw_${NAMES[$i]}.csv 2>&1
  ARGS="$ARGS ${NAMES[$i]}=$O/raw_${NAMES[$i]}.csv"
done
ncu -i /tmp/prof_cf1.ncu-rep --page source --csv --print-source sass > $O/src_bwd_cols.csv 2>&1
python tools/make_traffic.py --out $O/ncu_traffic.json C3-products $ARGS >> $O/ncu_fwd.txt 2>&1
gzip -f $O/raw_*.csv $O/src_*.csv
echo done
