"""A backward is bound to the forward it differentiates (ADVICE high).

The plan retains state of its last gt_attn_fwd (per-entry logits, received or published K||V rows,
GP-A2A head slices).  gt_attn_bwd may use it only for that forward's (q, k, v, lse); any other call
order - several layers sharing one plan, fwd(A) fwd(B) bwd(A) bwd(B), a backward with no forward -
must still return the gradients of PAPER.md Section 2.2 for the tensors it is given.  Every
case is checked against the fp64 oracle (normwise, reading Z8).
"""
import math
import threading

import numpy as np
import pytest

import gtgen
import oracle
from tests._util import TOL, check_lse, inputs, normwise, to_f64, to_torch

pytestmark = pytest.mark.gpu


def _ref(rp, ci, ins, scale):
    q, k, v, dy = ins
    Y, LSE = oracle.forward(rp, ci, q, k, v, scale)
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, scale)
    return Y, LSE, DQ, DK, DV


def _check(got, ref, dtype, what):
    y, lse, dq, dk, dv = got
    Y, LSE, DQ, DK, DV = ref
    for name, a, r in (("y", y, Y), ("dq", dq, DQ), ("dk", dk, DK), ("dv", dv, DV)):
        if a is None:
            continue
        e = normwise(a, r)
        assert e <= TOL[dtype], f"{what} {name}: normwise error {e:.3e}"
    if lse is not None:
        check_lse(lse, LSE, dtype)


@pytest.mark.parametrize("dtype,h,d", [("bf16", 4, 64), ("f32", 8, 16)])
@pytest.mark.parametrize("cuda_graphs", [False, True])
def test_interleaved_forwards_world1(dtype, h, d, cuda_graphs):
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(3000, 42000, seed=301, directed=True, power=2.1)
    n = len(rp) - 1
    scale = 1.0 / math.sqrt(h * d)
    A = inputs(n, h, d, dtype, 3011)
    B = inputs(n, h, d, dtype, 3012, qk_scale=4.0)  # peaked logits: B's logits differ a lot from A's
    plan = gt.Plan(rp, ci, h, d, dtype=dtype, scale=scale, heavy_threshold=64, edge_state=1,
                   cuda_graphs=cuda_graphs)
    assert plan.info()["edge_state"] == 1
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ta = [to_torch(x) for x in A]
        tb = [to_torch(x) for x in B]
        outs = {}
        for rep in range(3 if cuda_graphs else 1):  # graph mode: eager, capture, replay
            ya, la = plan.fwd(*ta[:3], stream=s)
            yb, lb = plan.fwd(*tb[:3], stream=s)
            ga = plan.bwd(*ta[:3], ya, la, ta[3], stream=s)   # stale: B's logits are in the plan
            gb = plan.bwd(*tb[:3], yb, lb, tb[3], stream=s)   # fresh
            gb2 = plan.bwd(*tb[:3], yb, lb, tb[3], stream=s)  # fresh again (state not consumed)
            outs[rep] = (ya, la, ga, yb, lb, gb, gb2)
    s.synchronize()
    info = plan.info()
    assert info["stale_bwds"] >= 1 and info["fwd_gen"] >= 2
    ra, rb = _ref(rp, ci, A, scale), _ref(rp, ci, B, scale)
    for rep, (ya, la, ga, yb, lb, gb, gb2) in outs.items():
        _check((to_f64(ya), to_f64(la), *(to_f64(t) for t in ga)), ra, dtype, f"A rep{rep}")
        _check((to_f64(yb), to_f64(lb), *(to_f64(t) for t in gb)), rb, dtype, f"B rep{rep}")
        for t1, t2 in zip(gb, gb2):
            assert torch.equal(t1, t2)
    plan.close()


def test_backward_without_forward_world1():
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(1500, 20000, seed=302, directed=True, power=2.1)
    n, h, d = len(rp) - 1, 4, 64
    scale = 1.0 / math.sqrt(h * d)
    A = inputs(n, h, d, "bf16", 3021)
    ref = _ref(rp, ci, A, scale)
    ta = [to_torch(x) for x in A]
    # the forward ran elsewhere (here: the oracle's Y and LSE, rounded to the plan's types)
    lse = to_torch(np.ascontiguousarray(ref[1], np.float32))
    y = to_torch(gtgen.f32_to_bf16_bits(np.ascontiguousarray(ref[0], np.float32)))
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, edge_state=1)
    g = plan.bwd(*ta[:3], y, lse, ta[3])
    torch.cuda.synchronize()
    _check((None, None, *(to_f64(t) for t in g)), ref, "bf16", "bwd-only")
    assert plan.info()["stale_bwds"] == 1
    plan.close()


def test_three_layers_share_one_plan_autograd():
    """The paper's GT stacks layers over one graph: one Plan, three forwards, then autograd
    runs the three backwards in reverse order - only the last one can use the retained state."""
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(2500, 36000, seed=303, directed=False, power=2.2, comm_size=256, f_in=0.8)
    n, h, d = len(rp) - 1, 4, 64
    scale = 1.0 / math.sqrt(h * d)
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, heavy_threshold=64, edge_state=1)
    layers = [inputs(n, h, d, "bf16", 3030 + i) for i in range(3)]
    leaves, ys = [], []
    for q, k, v, _ in layers:
        tq, tk, tv = (to_torch(x).requires_grad_(True) for x in (q, k, v))
        leaves.append((tq, tk, tv))
        ys.append(gt.sparse_graph_attention(plan, tq, tk, tv))
    loss = sum((y.float() * to_torch(L[3]).float()).sum() for y, L in zip(ys, layers))
    loss.backward()
    torch.cuda.synchronize()
    for i, (L, (tq, tk, tv), y) in enumerate(zip(layers, leaves, ys)):
        ref = _ref(rp, ci, L, scale)
        _check((to_f64(y), None, to_f64(tq.grad), to_f64(tk.grad), to_f64(tv.grad)), ref, "bf16", f"layer {i}")
    assert plan.info()["stale_bwds"] >= 2  # every layer but the last forward
    plan.close()


def _loopback_interleaved(rp, ci, h, d, dtype, world, strategy, transport=0, bwd_mode=0, edge_state=1):
    import torch
    import paper_2604_16715_b200 as gt
    n = len(rp) - 1
    scale = 1.0 / math.sqrt(h * d)
    A = inputs(n, h, d, dtype, 3101)
    B = inputs(n, h, d, dtype, 3102, qk_scale=3.0)
    fa, fb = [to_torch(x) for x in A], [to_torch(x) for x in B]
    grp = gt.LoopbackGroup(world)
    res, errors = [None] * world, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            plan = gt.Plan(rp, ci, h, d, dtype=dtype, scale=scale, world=world, rank=r, comm=grp,
                           strategy=strategy, heavy_threshold=64, edge_state=edge_state, transport=transport,
                           bwd_mode=bwd_mode)
            lo, hi = plan.row_lo, plan.row_hi
            with torch.cuda.stream(s):
                a = [t[lo:hi].contiguous() for t in fa]
                b = [t[lo:hi].contiguous() for t in fb]
                ya, la = plan.fwd(*a[:3], stream=s)
                yb, lb = plan.fwd(*b[:3], stream=s)
                ga = plan.bwd(*a[:3], ya, la, a[3], stream=s)  # stale on every rank
                gb = plan.bwd(*b[:3], yb, lb, b[3], stream=s)  # fresh
            s.synchronize()
            res[r] = ([to_f64(t) for t in (ya, la, *ga)], [to_f64(t) for t in (yb, lb, *gb)], plan.info())
            plan.close()
        except Exception as e:
            errors.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    grp.close()
    assert not errors, errors
    for which, ins in ((0, A), (1, B)):
        got = [np.concatenate([r[which][i] for r in res]) for i in range(5)]
        _check(got, _ref(rp, ci, ins, scale), dtype, f"{strategy} t{transport} b{bwd_mode} {'AB'[which]}")
    for r in res:
        assert r[2]["strategy_name"] == strategy
        assert r[2]["stale_bwds"] >= 1  # bwd(A) re-fetched; bwd(B) then re-fetches B's rows


@pytest.mark.parametrize("strategy,transport,bwd_mode", [("halo", 0, 0), ("allgather", 0, 0), ("halo", 0, 1),
                                                         ("halo", 1, 0), ("allgather", 1, 0)])
def test_interleaved_forwards_loopback(strategy, transport, bwd_mode):
    rp, ci = gtgen.random_graph(2400, 30000, seed=311, directed=True, power=2.1)
    _loopback_interleaved(rp, ci, 4, 64, "bf16", 2, strategy, transport=transport, bwd_mode=bwd_mode)


@pytest.mark.parametrize("world", [2, 4])
def test_interleaved_forwards_loopback_a2a(world):
    rp, ci = gtgen.random_graph(2000, 26000, seed=312, directed=True, power=2.1)
    _loopback_interleaved(rp, ci, 8, 32, "f32", world, "a2a")
