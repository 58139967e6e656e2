#!/bin/bash
# The bench's multi-rank path (barriers, max over ranks, report fields) with N processes sharing one GPU
# over CUDA IPC (--comm hostipc; NCCL refuses two ranks on one device).  Functional check, not scaling.
mkdir -p gpurun_out
python __graft_entry__.py build > /dev/null 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 \
     bench.py --gpus $n --comm hostipc --config C2 --steps 5 --warmup 3 > gpurun_out/bench_mp_C2_$n.log 2>&1; echo "exit $?" >> gpurun_out/bench_mp_C2_$n.log
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
   bench.py --gpus 2 --comm hostipc --steps 5 --warmup 3 > gpurun_out/bench_mp_C3_2.log 2>&1; echo "exit $?" >> gpurun_out/bench_mp_C3_2.log
echo done
