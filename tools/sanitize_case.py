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
rp, ci = gtgen.random_graph(3000, 45000, seed=11, directed=True, power=2.05)
h, d = 4, 64
q, k, v, dy = (to_torch(x) for x in inputs(3000, h, d, "bf16", 5))
plan = gt.Plan(rp, ci, h, d, dtype="bf16", heavy_threshold=48, edge_state=es)
y, lse = plan.fwd(q, k, v)
torch.cuda.synchronize()
print("fwd ok", flush=True)
dq, dk, dv = plan.bwd(q, k, v, y, lse, dy)
torch.cuda.synchronize()
print("bwd ok", flush=True)
