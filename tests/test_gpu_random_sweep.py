"""Randomized parity sweep (GPU): many small seeded graphs, shapes and plan options against the fp64
oracle, single-rank.  Graph recipe per case: random node count, density, power-law exponent, directed
or symmetrized, optional isolated tail; every option combination of edge_state / heavy threshold.
Tolerances as in test_gpu_parity (reading Z8)."""
import math

import numpy as np
import pytest

import gtgen
import oracle
from tests._util import TOL, check_lse, inputs, normwise, to_f64, to_torch

pytestmark = pytest.mark.gpu

SHAPES = [(1, 64, "bf16"), (2, 32, "f32"), (4, 64, "bf16"), (8, 16, "f32"), (8, 64, "bf16"), (2, 256, "f32"),
          (4, 128, "bf16"), (1, 512, "bf16")]


@pytest.mark.parametrize("case", range(24))
def test_random_sweep(case):
    import torch
    import paper_2604_16715_b200 as gt
    rng = np.random.default_rng(1000 + case)
    n = int(rng.integers(1, 2500))
    m = int(rng.integers(0, 12 * n + 1))
    m = min(m, n * (n - 1) // 4)  # leave the generator room to find m unique non-loop pairs
    h, d, dtype = SHAPES[case % len(SHAPES)]
    directed = bool(case % 3)
    rp, ci = gtgen.random_graph(n, m, seed=2000 + case, directed=directed, power=float(rng.uniform(1.9, 3.0)))
    n = len(rp) - 1
    q, k, v, dy = inputs(n, h, d, dtype, 3000 + case, qk_scale=float(rng.choice([1.0, 4.0])))
    scale = float(rng.choice([1.0 / math.sqrt(h * d), 1.0 / math.sqrt(d)]))
    es = int(rng.choice([1, -1]))
    heavy = int(rng.choice([0, 16, 100]))
    plan = gt.Plan(rp, ci, h, d, dtype=dtype, scale=scale, heavy_threshold=heavy, edge_state=es)
    tq, tk, tv, tdy = (to_torch(x) for x in (q, k, v, dy))
    y, lse = plan.fwd(tq, tk, tv)
    dq, dk, dv = plan.bwd(tq, tk, tv, y, lse, tdy)
    torch.cuda.synchronize()
    Y, LSE = oracle.forward(rp, ci, q, k, v, scale)
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, scale)
    for name, got, ref in (("y", y, Y), ("dq", dq, DQ), ("dk", dk, DK), ("dv", dv, DV)):
        e = normwise(to_f64(got), ref)
        assert e <= TOL[dtype], f"case {case} (n={n}, m={m}, {h}x{d} {dtype}, es={es}, T={heavy}): {name} {e:.3e}"
    check_lse(to_f64(lse), LSE, dtype)
    plan.close()
