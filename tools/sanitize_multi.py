"""Small multi-rank loopback cases for compute-sanitizer (reduce-scatter backward, peer gather,
GP-A2A, heads*d = 64); the sanitizer reports faults, the script checks nothing."""
import math
import sys
import threading

import torch

sys.path.insert(0, ".")
import gtgen  # noqa: E402
import paper_2604_16715_b200 as gt  # noqa: E402
from tests._util import inputs, to_torch  # noqa: E402


def run(world, strategy, h, d, dtype, **kw):
    rp, ci = gtgen.random_graph(1200, 14000, seed=3, directed=True, power=2.1)
    n = len(rp) - 1
    full = [to_torch(x) for x in inputs(n, h, d, dtype, 7)]
    grp = gt.LoopbackGroup(world)
    errs = []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            plan = gt.Plan(rp, ci, h, d, dtype=dtype, scale=1 / math.sqrt(h * d), world=world, rank=r, comm=grp,
                           strategy=strategy, heavy_threshold=40, **kw)
            lo, hi = plan.row_lo, plan.row_hi
            with torch.cuda.stream(s):
                t = [x[lo:hi].contiguous() for x in full]
            s.synchronize()
            for _ in range(2):
                y, lse = plan.fwd(t[0], t[1], t[2], stream=s)
                plan.bwd(t[0], t[1], t[2], y, lse, t[3], stream=s)
            s.synchronize()
            plan.close()
        except Exception as e:
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    grp.close()
    print(world, strategy, h, d, dtype, kw, "errors:", errs, flush=True)


run(3, "halo", 4, 64, "bf16", bwd_mode=1)
run(3, "allgather", 4, 64, "bf16", bwd_mode=1, edge_state=-1)
run(3, "halo", 4, 64, "bf16", transport=1)
run(2, "a2a", 4, 64, "bf16")
run(4, "a2a", 4, 64, "bf16")
run(2, "halo", 4, 16, "bf16")
