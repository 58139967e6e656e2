"""The SGA block and the 3-layer graph transformer on the GPU (Eq. 3-5,
P:80-93, backward P:98, the 3-layer GT of P:356) against the fp64 oracle (oracle/sga.py):

* one block, forward X' and backward (dX, dW_Q, dW_K, dW_V, dW_o) - normwise (reading Z8), fp32 <= 1e-4,
  bf16 <= 2e-2;
* five plain-SGD steps of the 3-layer model sharing one plan (fp32): the loss trajectory against the
  oracle's, and the final weights;
* the same five steps at world 2 over the in-process loopback transport (halo and all-gather; the
  ranks hold row ranges of X and the labels, weight gradients and losses are summed over ranks) equal
  to the world-1 trajectory ("single vs distributed trajectory equivalence").
"""
import math
import threading

import numpy as np
import pytest

import gtgen
import oracle.sga as osga
from tests._util import TOL, normwise

pytestmark = pytest.mark.gpu


def problem(n=1500, m=24000, dim=128, heads=4, classes=8, layers=3, seed=11):
    rp, ci = gtgen.random_graph(n, m, seed=seed, directed=True, power=2.1)
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, dim))
    mk = lambda: rng.standard_normal((dim, dim)) / math.sqrt(dim)  # noqa: E731
    params = {"layers": [{"wq": mk(), "wk": mk(), "wv": mk(), "wo": mk()} for _ in range(layers)],
              "wc": rng.standard_normal((dim, classes)) / math.sqrt(dim)}
    labels = rng.integers(0, classes, n)
    return rp, ci, X, params, labels, heads, 1.0 / math.sqrt(dim)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_block_forward_backward(dtype):
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci, X, params, labels, heads, scale = problem(layers=1)
    dim = X.shape[1]
    cd = torch.float32 if dtype == "f32" else torch.bfloat16
    # the oracle sees the inputs the GPU sees (rounded to the compute dtype)
    Xr = torch.tensor(X).to(cd).double().numpy()
    Wr = {k: torch.tensor(w).to(cd).double().numpy() for k, w in params["layers"][0].items()}
    G = np.random.default_rng(2).standard_normal(X.shape)
    Gr = torch.tensor(G).to(cd).double().numpy()
    Xp_ref, cache = osga.block_forward(rp, ci, Xr, Wr, heads, scale)
    dX_ref, g_ref = osga.block_backward(rp, ci, Wr, cache, Gr, heads, scale)

    plan = gt.Plan(rp, ci, heads, dim // heads, dtype=dtype, scale=scale, heavy_threshold=64)
    model = gt.GraphTransformer({"layers": [Wr], "wc": np.zeros((dim, 2))}, heads)
    tX = torch.tensor(Xr, dtype=torch.float32).cuda()
    Xp, c = model._block_fwd(plan, model.layers[0], tX)
    dX, g = model._block_bwd(plan, model.layers[0], c, torch.tensor(Gr, dtype=torch.float32).cuda())
    torch.cuda.synchronize()
    f64 = lambda t: t.double().cpu().numpy()  # noqa: E731
    for name, a, r in [("x'", Xp, Xp_ref), ("dx", dX, dX_ref)] + [(k, g[k], g_ref[k]) for k in ("wq", "wk", "wv", "wo")]:
        e = normwise(f64(a), r)
        assert e <= TOL[dtype], f"{dtype} {name}: normwise {e:.3e}"
    plan.close()


def _labels_t(labels, lo, hi):
    import torch
    return torch.tensor(labels[lo:hi], dtype=torch.int64).cuda()


def test_three_layer_sgd_world1_vs_oracle():
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci, X, params, labels, heads, scale = problem()
    dim, lr, steps = X.shape[1], 0.5, 5
    ref_losses, ref_final = osga.sgd_trajectory(rp, ci, X, params, labels, heads, scale, lr, steps)
    plan = gt.Plan(rp, ci, heads, dim // heads, dtype="f32", scale=scale, heavy_threshold=64)
    model = gt.GraphTransformer(params, heads)
    tX = torch.tensor(X, dtype=torch.float32).cuda()
    lab = _labels_t(labels, 0, len(labels))
    losses = [model.sgd_step(plan, tX, lab, len(labels), lr) for _ in range(steps)]
    rel = max(abs(a - b) / abs(b) for a, b in zip(losses, ref_losses))
    assert rel <= 1e-4, (losses, ref_losses)
    assert ref_losses[-1] < ref_losses[0]
    e = normwise(model.wc.double().cpu().numpy(), ref_final["wc"])
    assert e <= 1e-4, e
    for W, R in zip(model.layers, ref_final["layers"]):
        for k in W:
            assert normwise(W[k].double().cpu().numpy(), R[k]) <= 1e-4, k
    assert plan.info()["stale_bwds"] >= 1   # layers 1..L-1 ran their backward after a later forward
    plan.close()


class ThreadAllReduce:
    """Sum over in-process loopback ranks (threads): every rank contributes its tensors, all receive the
    sum, added in rank order (deterministic)."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.buf = [None] * world

    def __call__(self, rank, tensors):
        import torch
        torch.cuda.current_stream().synchronize()
        self.buf[rank] = [t.clone() for t in tensors]
        self.bar.wait()
        for i, t in enumerate(tensors):
            acc = self.buf[0][i].clone()
            for r in range(1, self.world):
                acc += self.buf[r][i]
            t.copy_(acc)
        torch.cuda.current_stream().synchronize()
        self.bar.wait()


@pytest.mark.parametrize("strategy", ["halo", "allgather"])
def test_three_layer_sgd_world2_equals_world1(strategy):
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci, X, params, labels, heads, scale = problem()
    dim, lr, steps, world = X.shape[1], 0.5, 5, 2
    plan1 = gt.Plan(rp, ci, heads, dim // heads, dtype="f32", scale=scale, heavy_threshold=64)
    m1 = gt.GraphTransformer(params, heads)
    tX = torch.tensor(X, dtype=torch.float32).cuda()
    l1 = [m1.sgd_step(plan1, tX, _labels_t(labels, 0, len(labels)), len(labels), lr) for _ in range(steps)]
    plan1.close()

    grp = gt.LoopbackGroup(world)
    ar = ThreadAllReduce(world)
    res, errors = [None] * world, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                plan = gt.Plan(rp, ci, heads, dim // heads, dtype="f32", scale=scale, world=world, rank=r,
                               comm=grp, strategy=strategy, heavy_threshold=64)
                lo, hi = plan.row_lo, plan.row_hi
                m = gt.GraphTransformer(params, heads)
                x = torch.tensor(X[lo:hi], dtype=torch.float32).cuda()
                lab = _labels_t(labels, lo, hi)
                res[r] = [m.sgd_step(plan, x, lab, len(labels), lr, allreduce=lambda ts: ar(r, ts))
                          for _ in range(steps)]
                s.synchronize()
                res[r] = (res[r], m.wc.double().cpu().numpy(), plan.info()["strategy_name"])
                plan.close()
        except Exception as e:  # surfaced below
            errors.append((r, repr(e)))
            ar.bar.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    grp.close()
    assert not errors, errors
    for r in range(world):
        losses, wc, strat = res[r]
        assert strat == strategy
        rel = max(abs(a - b) / abs(b) for a, b in zip(losses, l1))
        assert rel <= 1e-4, (r, losses, l1)
        assert normwise(wc, m1.wc.double().cpu().numpy()) <= 1e-4
