#!/bin/bash
# ncu --set full of one kernel: tools/gpu_prof1.sh <kernel-name-regex> <out-name> [launch-skip] [env...]
mkdir -p gpurun_out
python __graft_entry__.py build > /dev/null 2>&1
K=$1; O=$2; S=${3:-0}; shift 3
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s $S -c 1 \
   -o gpurun_out/$O -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/$O.log 2>&1
echo done
