"""Multi-rank path on one GPU: `world` host threads, each a rank with its own plan, exchanging rows
through the in-process loopback transport (device-to-device copies on each rank's stream).

Checks: outputs of all ranks, concatenated in row order, match the fp64 oracle within the
single-GPU tolerances; bounds, halo sets and send lists match the oracle bit-exactly; both
strategies (all-gather, halo) and the cost-model choice (auto).
"""
import math
import threading

import numpy as np
import pytest

import gtgen
import oracle
from tests._util import TOL, check_lse, inputs, normwise, to_f64, to_torch

pytestmark = pytest.mark.gpu


def run_loopback(rp, ci, h, d, dtype, world, strategy, seed, heavy=0, partition=0, edge_state=0, bwd_mode=0,
                 transport=0, steps=1, beta_profile=None, reserve_sms=0):
    import torch
    import paper_2604_16715_b200 as gt
    n = len(rp) - 1
    q, k, v, dy = inputs(n, h, d, dtype, seed)
    scale = 1.0 / math.sqrt(h * d)
    grp = gt.LoopbackGroup(world)
    res = [None] * world
    errors = []
    full = [to_torch(x) for x in (q, k, v, dy)]

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            plan = gt.Plan(rp, ci, h, d, dtype=dtype, scale=scale, world=world, rank=r, comm=grp,
                           strategy=strategy, heavy_threshold=heavy, partition=partition, edge_state=edge_state,
                           bwd_mode=bwd_mode, transport=transport, beta_profile=beta_profile,
                           reserve_sms=reserve_sms)
            lo, hi = plan.row_lo, plan.row_hi
            with torch.cuda.stream(s):
                tq, tk, tv, tdy = (t[lo:hi].contiguous() for t in full)
            s.synchronize()
            for _ in range(steps):  # repeated steps exercise the reuse of exchange / publish buffers
                y, lse = plan.fwd(tq, tk, tv, stream=s)
                dq, dk, dv = plan.bwd(tq, tk, tv, y, lse, tdy, stream=s)
            s.synchronize()
            ex = {w: plan.export(w) for w in ("bounds", "halo_out", "halo_in")}
            ex["send_out"] = [plan.export("send_out", p) for p in range(world)]
            ex["send_in"] = [plan.export("send_in", p) for p in range(world)]
            ex["csc_ptr"], ex["csc_idx"] = plan.export("csc_ptr"), plan.export("csc_idx")
            res[r] = (lo, hi, [to_f64(t) for t in (y, lse, dq, dk, dv)], ex, plan.info())
            plan.close()
        except Exception as e:  # surfaced below
            errors.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    grp.close()
    assert not errors, errors
    return (q, k, v, dy, scale), res


def check(rp, ci, dtype, ins, res, world, partition=0):
    q, k, v, dy, scale = ins
    Y, LSE = oracle.forward(rp, ci, q, k, v, scale)
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, scale)
    outs = [np.concatenate([r[2][i] for r in res]) for i in range(5)]
    for name, got, ref in (("y", outs[0], Y), ("dq", outs[2], DQ), ("dk", outs[3], DK), ("dv", outs[4], DV)):
        e = normwise(got, ref)
        assert e <= TOL[dtype], f"{name}: {e}"
    check_lse(outs[1], LSE, dtype)
    bounds = oracle.partition(rp, world, partition)
    cp, ri = oracle.transpose(rp, ci)
    for r, (lo, hi, _, ex, info) in enumerate(res):
        np.testing.assert_array_equal(ex["bounds"], bounds)
        assert (lo, hi) == (bounds[r], bounds[r + 1])
        np.testing.assert_array_equal(ex["halo_out"], oracle.halo(rp, ci, lo, hi))
        np.testing.assert_array_equal(ex["halo_in"], oracle.halo(rp, ci, lo, hi, inward=True))
        for p in range(world):
            if p == r:
                continue
            hp = oracle.halo(rp, ci, bounds[p], bounds[p + 1])
            hpi = oracle.halo(rp, ci, bounds[p], bounds[p + 1], inward=True)
            np.testing.assert_array_equal(ex["send_out"][p], oracle.send_list(hp, bounds, r))
            np.testing.assert_array_equal(ex["send_in"][p], oracle.send_list(hpi, bounds, r))
        # owned-column slice of A^T, global row ids
        np.testing.assert_array_equal(ex["csc_ptr"], cp[lo:hi + 1] - cp[lo])
        np.testing.assert_array_equal(ex["csc_idx"], ri[cp[lo]:cp[hi]])


# bwd_mode 0: transposed owner (default); 1: reduce-scatter of fp32 partials (paper-faithful, Z11)
@pytest.mark.parametrize("bwd_mode", [0, 1])
@pytest.mark.parametrize("edge_state", [1, -1])
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("strategy", ["halo", "allgather"])
def test_loopback_directed_power_law(world, strategy, edge_state, bwd_mode):
    rp, ci = gtgen.random_graph(2500, 30000, seed=70 + world, directed=True, power=2.1)
    ins, res = run_loopback(rp, ci, 4, 64, "bf16", world, strategy, seed=700 + world, heavy=64,
                            edge_state=edge_state, bwd_mode=bwd_mode)
    check(rp, ci, "bf16", ins, res, world)
    for r in res:
        assert r[4]["strategy_name"] == strategy
        assert r[4]["edge_state"] == (0 if edge_state < 0 else 1)
        assert r[4]["bwd_mode"] == bwd_mode


@pytest.mark.parametrize("bwd_mode", [0, 1])
def test_loopback_communities_f32_auto(bwd_mode):
    rp, ci = gtgen.random_graph(4096, 50000, seed=81, directed=False, power=2.2, comm_size=512, f_in=0.9)
    ins, res = run_loopback(rp, ci, 8, 16, "f32", 4, "auto", seed=801, bwd_mode=bwd_mode)
    check(rp, ci, "f32", ins, res, 4)
    chosen = {r[4]["strategy_name"] for r in res}
    assert len(chosen) == 1 and chosen <= {"halo", "allgather"}  # every rank applies rank 0's decision


@pytest.mark.parametrize("bwd_mode,transport", [(0, 0), (1, 0), (0, 1)])
def test_loopback_more_ranks_than_rows_and_node_partition(bwd_mode, transport):
    rp, ci = gtgen.csr_from_pairs(3, [(0, 1), (1, 2), (2, 0), (2, 1)])
    ins, res = run_loopback(rp, ci, 2, 64, "f32", 5, "halo", seed=901, bwd_mode=bwd_mode, transport=transport)
    check(rp, ci, "f32", ins, res, 5)
    rp, ci = gtgen.random_graph(700, 6000, seed=91, power=2.3)
    ins, res = run_loopback(rp, ci, 4, 32, "bf16", 3, "allgather", seed=902, partition=1, bwd_mode=bwd_mode,
                            transport=transport)
    check(rp, ci, "bf16", ins, res, 3, partition=1)


def test_reduce_scatter_hub_columns_chunked_and_deterministic():
    """Hub columns with more in-edges than the chunk threshold on several ranks: partial pieces, a
    summed send row per slot and a multi-source merge; two runs are bitwise identical."""
    n = 900
    pairs = [(i, 0) for i in range(1, n)] + [(i, n - 1) for i in range(0, n - 1)] + [(0, j) for j in range(1, n)]
    rp, ci = gtgen.csr_from_pairs(n, pairs)
    outs = []
    for _ in range(2):
        ins, res = run_loopback(rp, ci, 4, 64, "f32", 3, "halo", seed=911, heavy=50, bwd_mode=1)
        check(rp, ci, "f32", ins, res, 3)
        outs.append(np.concatenate([np.concatenate([r[2][i] for r in res]).ravel() for i in (0, 2, 3, 4)]))
    assert np.array_equal(outs[0], outs[1])


# GP-A2A head parallelism (Alg. 2): heads / world heads of all rows per rank
@pytest.mark.parametrize("world,h,d,dtype", [(2, 4, 64, "bf16"), (2, 8, 32, "f32"), (4, 8, 64, "f32"),
                                             (4, 8, 64, "bf16"), (4, 4, 64, "bf16")])
@pytest.mark.parametrize("edge_state", [1, -1])
def test_loopback_a2a_head_parallel(world, h, d, dtype, edge_state):
    rp, ci = gtgen.random_graph(2200, 28000, seed=120 + world + h, directed=True, power=2.1)
    ins, res = run_loopback(rp, ci, h, d, dtype, world, "a2a", seed=1200 + world, heavy=64, edge_state=edge_state)
    check(rp, ci, dtype, ins, res, world)
    for r in res:
        assert r[4]["strategy_name"] == "a2a"


def test_a2a_infeasible_shapes_are_config_errors():
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(300, 2000, seed=5, power=2.3)
    grp = gt.LoopbackGroup(2)
    try:
        with pytest.raises(gt.GTError) as e:  # heads % world != 0 (checked before any collective)
            gt.Plan(rp, ci, 1, 128, dtype="f32", world=2, rank=0, comm=grp, strategy="a2a")
        assert e.value.status == 3
    finally:
        grp.close()


def test_loopback_auto_considers_a2a():
    rp, ci = gtgen.random_graph(3000, 40000, seed=131, directed=False, power=2.2)
    ins, res = run_loopback(rp, ci, 8, 32, "bf16", 2, "auto", seed=1310)
    check(rp, ci, "bf16", ins, res, 2)
    for r in res:
        assert np.isfinite(r[4]["predicted_ms"][4])  # GP-A2A probed and costed
    assert len({r[4]["strategy_name"] for r in res}) == 1


# fused peer gather (transport 1): kernels read remote K || V rows from the owners'
# published buffers (loopback ranks share one device, so peer pointers are plain device pointers)
@pytest.mark.parametrize("edge_state", [1, -1])
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("strategy", ["halo", "allgather"])
def test_loopback_peer_gather(world, strategy, edge_state):
    rp, ci = gtgen.random_graph(2600, 32000, seed=140 + world, directed=True, power=2.1)
    ins, res = run_loopback(rp, ci, 4, 64, "bf16", world, strategy, seed=1400 + world, heavy=64,
                            edge_state=edge_state, transport=1, steps=3)
    check(rp, ci, "bf16", ins, res, world)
    for r in res:
        assert r[4]["transport"] == 1


def test_peer_gather_config_errors():
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(300, 2000, seed=6, power=2.3)
    grp = gt.LoopbackGroup(2)
    try:
        with pytest.raises(gt.GTError) as e:  # rejected before any collective
            gt.Plan(rp, ci, 4, 64, dtype="f32", world=2, rank=0, comm=grp, strategy="halo", transport=1, bwd_mode=1)
        assert e.value.status == 3
    finally:
        grp.close()


def test_auto_follows_a_beta_profile(tmp_path):
    """gt_opts.beta_profile (Fig. 2 / Alg. 3 profiled beta, reading Z14) replaces the plan-time probe:
    the planner's choice follows the profile, per GPU count or as plain numbers."""
    import json
    rp, ci = gtgen.random_graph(2000, 24000, seed=151, directed=True, power=2.1)
    for fast, slow in (("allgather", "halo"), ("halo", "allgather")):
        path = tmp_path / f"beta_{fast}.json"
        path.write_text(json.dumps({fast: {"2": 1e-12, "3": 1e-12}, slow: 1.0, "a2a": 1.0}))
        _, res = run_loopback(rp, ci, 4, 64, "f32", 2, "auto", seed=1510, beta_profile=str(path))
        assert {r[4]["strategy_name"] for r in res} == {fast}
        for r in res:
            assert r[4]["beta_s_per_row"][{"allgather": 2, "halo": 3}[fast]] == pytest.approx(1e-12)


@pytest.mark.parametrize("reserve_sms", [-1, 40])
def test_loopback_reserve_sms(reserve_sms):
    """gt_opts.reserve_sms only changes how many SMs the overlapped phase leaves free, not the results."""
    rp, ci = gtgen.random_graph(2500, 30000, seed=171, directed=True, power=2.1)
    ins, res = run_loopback(rp, ci, 4, 64, "bf16", 2, "halo", seed=1710, heavy=64, reserve_sms=reserve_sms)
    check(rp, ci, "bf16", ins, res, 2)
