"""Per-step time of small configs with and without CUDA-graph replay (gt_opts.cuda_graphs)."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import gtgen  # noqa: E402
import paper_2604_16715_b200 as gt  # noqa: E402

for cname in sys.argv[1:] or ["C1", "C2"]:
    cfg = gtgen.CONFIGS[cname]
    rp, ci = gtgen.make_graph(cfg.graph)
    n, h, d = len(rp) - 1, cfg.heads, cfg.d
    feats = [gtgen.features(3, nm, n, h, d, cfg.dtype) for nm in ("q", "k", "v", "dy")]
    conv = (lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()) if cfg.dtype == "bf16" else \
        (lambda x: torch.from_numpy(x).cuda())
    q, k, v, dy = (conv(x) for x in feats)
    for graphs in (False, True):
        plan = gt.Plan(rp, ci, h, d, dtype=cfg.dtype, scale=1 / math.sqrt(h * d), cuda_graphs=graphs)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            y, lse = torch.empty_like(q), torch.empty((n, h), dtype=torch.float32, device="cuda")
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)

        def step():
            plan.fwd(q, k, v, y, lse, stream=s)
            plan.bwd(q, k, v, y, lse, dy, dq, dk, dv, stream=s)
        for _ in range(5):
            step()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(200):
            step()
        e1.record(s)
        s.synchronize()
        print(f"{cname} graphs={graphs}: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us per fwd+bwd step", flush=True)
        plan.close()
