#!/bin/bash
# Power of the gathers alone: the L2 -> SM microbenchmark (tools/l2bw.cu) run back to back for 4 s next
# to a 20-ms nvidia-smi trace - does moving the bytes by itself reach the board's 1000 W limit?
mkdir -p gpurun_out/power_l2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2bw tools/l2bw.cu
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.sw_power_cap --format=csv,nounits -i 0 -lms 20 > gpurun_out/power_l2/smi_trace.csv 2>&1 &
SMI=$!
sleep 1
/tmp/l2bw 32 40 4 > gpurun_out/power_l2/l2bw_32mib.log 2>&1
sleep 2
/tmp/l2bw 2048 4 4 > gpurun_out/power_l2/l2bw_2gib.log 2>&1
sleep 1
kill $SMI
echo done
