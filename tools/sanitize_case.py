"""Small fwd+bwd cases for compute-sanitizer runs (no checks; the sanitizer reports faults)."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import gtgen  # noqa: E402
import paper_2604_16715_b200 as gt  # noqa: E402
from tests._util import inputs, to_torch  # noqa: E402

es = int(sys.argv[1]) if len(sys.argv) > 1 else 1
fp8 = len(sys.argv) > 2 and sys.argv[2] == "fp8"   # the fp8 K||V kernels (gt_opts.kv_fp8)
rp, ci = gtgen.random_graph(3000, 45000, seed=11, directed=True, power=2.05)
h, d = 4, 64
q, k, v, dy = (to_torch(x) for x in inputs(3000, h, d, "bf16", 5))
plan = gt.Plan(rp, ci, h, d, dtype="bf16", heavy_threshold=48, edge_state=es, kv_fp8=fp8)
y, lse = plan.fwd(q, k, v)
torch.cuda.synchronize()
print("fwd ok", flush=True)
dq, dk, dv = plan.bwd(q, k, v, y, lse, dy)
torch.cuda.synchronize()
print("bwd ok", flush=True)
# host-buffer step (streamed chunks)
pin = [t.cpu().pin_memory() for t in (q, k, v, dy)]
outs = [torch.empty_like(pin[0]).pin_memory() for _ in range(4)]
lh = torch.empty((3000, h), dtype=torch.float32).pin_memory()
plan.fwd_bwd_host(pin[0], pin[1], pin[2], pin[3], outs[0], lh, outs[1], outs[2], outs[3])
print("host ok", flush=True)
