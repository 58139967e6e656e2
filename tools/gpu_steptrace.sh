#!/bin/bash
# Per-step times of a long timed region next to a 20-ms nvidia-smi trace (SM / memory clocks, power,
# temperatures, clock-event reasons): what slows the sustained steps down.
mkdir -p gpurun_out/steptrace
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE > gpurun_out/steptrace/smi_q.txt 2>&1
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown --format=csv,nounits -i 0 -lms 20 > gpurun_out/steptrace/smi_trace.csv 2>&1 &
SMI=$!
timeout 900 python bench.py --steps 60 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/steptrace/bench60.log 2>&1
sleep 2
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/steptrace/bench10.log 2>&1
kill $SMI
echo done
