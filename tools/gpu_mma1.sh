#!/bin/bash
# Tensor-core consumer: parity (incl. full size), A/B against the CUDA-core FMA consumer, ncu of the passes.
mkdir -p gpurun_out/mma1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state_binding.py tests/test_gpu_random_sweep.py tests/test_gpu_multirank.py -x -q > gpurun_out/mma1/pytest.log 2>&1; echo "exit $?" >> gpurun_out/mma1/pytest.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/mma1/pytest_full.log 2>&1; echo "exit $?" >> gpurun_out/mma1/pytest_full.log
: > gpurun_out/mma1/ab.log
for rep in 1 2; do for v in mma fma; do
  echo "=== $v" >> gpurun_out/mma1/ab.log
  if [ $v = mma ]; then L=paper_2604_16715_b200/libgt.so; else L=tools/variants/fma/libgt.so; fi
  GT_LIB=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/mma1/ab.log 2>&1
done; done
PASSES="0 1 2" SKIP_TESTS=1 bash tools/gpu_quick.sh
for f in ncu_pass0.txt ncu_pass1.txt ncu_pass2.txt sass_pass0.txt sass_pass1.txt sass_pass2.txt ncu_traffic.json bench.log; do mv gpurun_out/$f gpurun_out/mma1/ 2>/dev/null; done
gzip -f gpurun_out/raw_pass*.csv gpurun_out/src_pass*.csv 2>/dev/null; mv gpurun_out/raw_pass*.csv.gz gpurun_out/src_pass*.csv.gz gpurun_out/mma1/ 2>/dev/null
echo done
