#!/bin/bash
# Repeated bench runs (variance check).  Usage: tools/gpu_rep.sh N [bench args]
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
N=$1; shift
: > gpurun_out/rep.log
for i in $(seq $N); do timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" >> gpurun_out/rep.log 2>&1; done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv >> gpurun_out/rep.log
echo done
