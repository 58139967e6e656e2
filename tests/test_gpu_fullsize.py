"""Full-size parity: BASELINE.json configs C3 (products-shaped), C4 (Reddit-shaped) and C5 (R-MAT) at
their full sizes, in the launch configuration bench.py times (default plan options, one GPU), compared
with the fp64 oracle on sampled outputs the oracle computes one by one (oracle.sample): rows for Y, LSE,
dQ and columns for dK, dV.  Samples always include the heaviest rows/columns (chunked + merged), empty
rows, and uniformly random ones.  Tolerance: normwise over the sample, bf16 <= 2e-2 (Z8)."""
import math

import numpy as np
import pytest

import gtgen
import oracle
from tests._util import TOL, check_lse, normwise

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def sample_ids(deg, rng, k_heavy=4, k_rand=300):
    n = len(deg)
    heavy = np.argsort(deg)[-k_heavy:]
    empty = np.nonzero(deg == 0)[0][:4]
    rand = rng.choice(n, size=min(k_rand, n), replace=False)
    return np.unique(np.concatenate([heavy, empty, rand])).astype(np.int64)


@pytest.mark.parametrize("cfg_name", ["C3", "C4", "C5"])
def test_fullsize_sampled(cfg_name):
    import torch
    import paper_2604_16715_b200 as gt
    cfg = gtgen.CONFIGS[cfg_name]
    rp, ci = gtgen.make_graph(cfg.graph)
    n = len(rp) - 1
    h, d = cfg.heads, cfg.d
    scale = 1.0 / math.sqrt(h * d)
    feats = {nm: gtgen.features(77, nm, n, h, d, cfg.dtype) for nm in ("q", "k", "v", "dy")}
    plan = gt.Plan(rp, ci, h, d, dtype=cfg.dtype, scale=scale)   # bench.py's launch configuration
    dev = {nm: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda() for nm, x in feats.items()}
    y, lse = plan.fwd(dev["q"], dev["k"], dev["v"])
    dq, dk, dv = plan.bwd(dev["q"], dev["k"], dev["v"], y, lse, dev["dy"])
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    rows = sample_ids(np.diff(rp), rng)
    cols = sample_ids(np.bincount(ci, minlength=n), rng, k_rand=120)
    ref = oracle.sample(rp, ci, feats["q"], feats["k"], feats["v"], feats["dy"], scale, rows, cols)
    ti = lambda idx: torch.from_numpy(idx).cuda()  # noqa: E731
    got = {
        "y": y[ti(rows)].double().cpu().numpy(),
        "dq": dq[ti(rows)].double().cpu().numpy(),
        "dk": dk[ti(cols)].double().cpu().numpy(),
        "dv": dv[ti(cols)].double().cpu().numpy(),
    }
    for name in ("y", "dq", "dk", "dv"):
        e = normwise(got[name], ref[name])
        assert e <= TOL[cfg.dtype], f"{cfg_name} {name}: normwise {e:.3e}"
    check_lse(lse[ti(rows)].double().cpu().numpy(), ref["lse"], cfg.dtype)
    info = plan.info()
    if cfg_name in ("C3", "C5"):
        assert info["heavy_rows"] > 0 and info["heavy_cols"] > 0  # chunked path exercised
    plan.close()
