"""Two NCCL ranks on ONE GPU (torchrun --nproc-per-node 2): exercises the real NCCL transport of
libgt (grouped send/recv, all-gather, stream barrier, plan-time probes) where only one GPU exists.
Prints per-rank normwise errors against the fp64 oracle.  NCCL may refuse duplicate GPUs."""
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import gtgen  # noqa: E402
import oracle  # noqa: E402
import paper_2604_16715_b200 as gt  # noqa: E402
from tests._util import inputs, normwise, to_f64, to_torch  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
strategy = sys.argv[1] if len(sys.argv) > 1 else "halo"
kw = dict(a.split("=") for a in sys.argv[2:])
kw = {k: int(v) for k, v in kw.items()}
rp, ci = gtgen.random_graph(3000, 40000, seed=21, directed=True, power=2.1)
n, h, d = len(rp) - 1, 4, 64
q, k, v, dy = inputs(n, h, d, "bf16", 77)
scale = 1 / math.sqrt(h * d)
comm = gt.NcclComm()          # bootstrap over the gloo group; NCCL communicator of libgt
plan = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, world=world, rank=rank, comm=comm, strategy=strategy, **kw)
lo, hi = plan.row_lo, plan.row_hi
t = [to_torch(x)[lo:hi].contiguous() for x in (q, k, v, dy)]
for _ in range(2):
    y, lse = plan.fwd(t[0], t[1], t[2])
    dq, dk, dv = plan.bwd(t[0], t[1], t[2], y, lse, t[3])
torch.cuda.synchronize()
Y, _ = oracle.forward(rp, ci, q, k, v, scale)
DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, scale)
errs = {nm: normwise(to_f64(a), r[lo:hi]) for nm, a, r in (("y", y, Y), ("dq", dq, DQ), ("dk", dk, DK), ("dv", dv, DV))}
print(f"rank {rank} strategy {plan.info()['strategy_name']} {kw} errors {errs}", flush=True)
assert all(e <= 2e-2 for e in errs.values()), errs
plan.close()
comm.close()
dist.destroy_process_group()
