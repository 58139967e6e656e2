"""The real cross-process data plane on one GPU: `world` PROCESSES, one rank each,
bootstrapped over a gloo process group (127.0.0.1), exchanging rows through CUDA IPC
(GT_COMM_HOSTIPC: IPC memory handles + interprocess events, gt_hostipc_create) - the path a one-process-
per-GPU deployment uses for its buffers (Alg. 1; the fused peer gather maps the owners'
published rows), run here by several processes sharing one B200 (NCCL refuses two ranks on one
device).  Each case checks the concatenated outputs against the fp64 oracle within the single-GPU
tolerances and the partition, halos, send lists and CSC slices bit for bit (tests/test_gpu_multirank.check).
"""
import math
import multiprocessing as mp
import os
import socket
import traceback

import numpy as np
import pytest

import gtgen
from tests._util import inputs

pytestmark = pytest.mark.gpu

CASES = {
    # name: graph, (h, d, dtype), world, strategy, transport, bwd_mode, edge_state
    "halo_copy": (("power", 2600, 32000, 71), (4, 64, "bf16"), 2, "halo", 0, 0, 1),
    "allgather_copy_w3": (("power", 2600, 32000, 72), (4, 64, "bf16"), 3, "allgather", 0, 0, -1),
    "halo_reduce_scatter": (("power", 2400, 30000, 73), (8, 16, "f32"), 2, "halo", 0, 1, 1),
    "peer_gather_halo": (("power", 2600, 32000, 74), (4, 64, "bf16"), 2, "halo", 1, 0, 1),
    "peer_gather_allgather_w3": (("power", 2600, 32000, 75), (4, 64, "bf16"), 3, "allgather", 1, 0, -1),
    "a2a": (("power", 2200, 28000, 76), (4, 64, "bf16"), 2, "a2a", 0, 0, 1),
    "auto_communities": (("comm", 4096, 50000, 77), (8, 16, "f32"), 2, "auto", 0, 0, 1),
    "halo_w4": (("power", 3000, 36000, 78), (4, 64, "bf16"), 4, "halo", 0, 0, 1),
    "peer_gather_halo_w4": (("power", 3000, 36000, 79), (4, 64, "bf16"), 4, "halo", 1, 0, -1),
}


def _graph(spec):
    kind, n, m, seed = spec
    if kind == "comm":
        return gtgen.random_graph(n, m, seed=seed, directed=False, power=2.2, comm_size=512, f_in=0.9)
    return gtgen.random_graph(n, m, seed=seed, directed=True, power=2.1)


def _worker(rank, world, port, case, out_q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        import paper_2604_16715_b200 as gt
        from tests._util import to_f64, to_torch
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        gspec, (h, d, dtype), _, strategy, transport, bwd_mode, edge_state = CASES[case]
        rp, ci = _graph(gspec)
        n = len(rp) - 1
        q, k, v, dy = inputs(n, h, d, dtype, seed=gspec[3] * 10)
        grp = gt.HostIpcGroup()
        plan = gt.Plan(rp, ci, h, d, dtype=dtype, scale=1.0 / math.sqrt(h * d), world=world, rank=rank, comm=grp,
                       strategy=strategy, heavy_threshold=64, edge_state=edge_state, bwd_mode=bwd_mode,
                       transport=transport)
        lo, hi = plan.row_lo, plan.row_hi
        tq, tk, tv, tdy = (to_torch(x[lo:hi]) for x in (q, k, v, dy))
        for _ in range(3):  # repeated steps reuse the published / mapped buffers
            y, lse = plan.fwd(tq, tk, tv)
            dq, dk, dv = plan.bwd(tq, tk, tv, y, lse, tdy)
        torch.cuda.synchronize()
        ex = {w: plan.export(w) for w in ("bounds", "halo_out", "halo_in")}
        ex["send_out"] = [plan.export("send_out", p) for p in range(world)]
        ex["send_in"] = [plan.export("send_in", p) for p in range(world)]
        ex["csc_ptr"], ex["csc_idx"] = plan.export("csc_ptr"), plan.export("csc_idx")
        info = plan.info()
        res = (lo, hi, [to_f64(t) for t in (y, lse, dq, dk, dv)], ex,
               {k_: info[k_] for k_ in ("strategy_name", "transport", "bwd_mode", "edge_state")})
        plan.close()
        grp.close()
        dist.barrier()
        dist.destroy_process_group()
        out_q.put((rank, res, None))
    except Exception:
        out_q.put((rank, None, traceback.format_exc()))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_processes(case, timeout=420):
    world = CASES[case][2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res, errs = [None] * world, []
    try:
        for _ in range(world):
            r, out, err = q.get(timeout=timeout)
            if err:
                errs.append((r, err))
            res[r] = out
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()      # this test's own child, by handle
                p.join()
    assert not errs, errs
    return res


@pytest.mark.parametrize("case", sorted(CASES))
def test_multiprocess_hostipc(case):
    from tests.test_gpu_multirank import check
    gspec, (h, d, dtype), world, strategy, transport, bwd_mode, edge_state = CASES[case]
    rp, ci = _graph(gspec)
    n = len(rp) - 1
    q, k, v, dy = inputs(n, h, d, dtype, seed=gspec[3] * 10)
    res = run_processes(case)
    check(rp, ci, dtype, (q, k, v, dy, 1.0 / math.sqrt(h * d)), res, world)
    names = {r[4]["strategy_name"] for r in res}
    assert len(names) == 1 and (strategy == "auto" or names == {strategy})
    for r in res:
        assert r[4]["transport"] == transport and r[4]["bwd_mode"] == bwd_mode


# ---- distributed training across processes: the 3-layer graph transformer (Eq. 3-5) ----
def _train_worker(rank, world, port, strategy, out_q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        import paper_2604_16715_b200 as gt
        from tests.test_gpu_model import problem
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        rp, ci, X, params, labels, heads, scale = problem()
        dim = X.shape[1]
        grp = gt.HostIpcGroup()
        plan = gt.Plan(rp, ci, heads, dim // heads, dtype="f32", scale=scale, world=world, rank=rank, comm=grp,
                       strategy=strategy, heavy_threshold=64)
        lo, hi = plan.row_lo, plan.row_hi
        m = gt.GraphTransformer(params, heads)
        x = torch.tensor(X[lo:hi], dtype=torch.float32).cuda()
        lab = torch.tensor(labels[lo:hi], dtype=torch.int64).cuda()

        def allreduce(ts):  # gradient and loss sums over ranks (gloo, host staging)
            for t in ts:
                c = t.detach().cpu()
                dist.all_reduce(c)
                t.copy_(c.to(t.device))

        losses = [m.sgd_step(plan, x, lab, len(labels), 0.5, allreduce=allreduce) for _ in range(5)]
        wc = m.wc.double().cpu().numpy()
        plan.close()
        grp.close()
        dist.barrier()
        dist.destroy_process_group()
        out_q.put((rank, (losses, wc), None))
    except Exception:
        out_q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("strategy", ["halo", "allgather"])
def test_multiprocess_training_trajectory(strategy):
    """Two processes (one rank each; attention exchange over CUDA IPC, gradient sums over gloo) train the
    3-layer graph transformer for 5 SGD steps: the loss trajectory and final weights equal world 1's."""
    import torch
    import paper_2604_16715_b200 as gt
    from tests._util import normwise
    from tests.test_gpu_model import problem
    rp, ci, X, params, labels, heads, scale = problem()
    dim = X.shape[1]
    plan1 = gt.Plan(rp, ci, heads, dim // heads, dtype="f32", scale=scale, heavy_threshold=64)
    m1 = gt.GraphTransformer(params, heads)
    tX = torch.tensor(X, dtype=torch.float32).cuda()
    lab = torch.tensor(labels, dtype=torch.int64).cuda()
    l1 = [m1.sgd_step(plan1, tX, lab, len(labels), 0.5) for _ in range(5)]
    plan1.close()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, world, port, strategy, q)) for r in range(world)]
    for p in procs:
        p.start()
    res, errs = [None] * world, []
    try:
        for _ in range(world):
            r, out, err = q.get(timeout=420)
            if err:
                errs.append((r, err))
            res[r] = out
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
                p.join()
    assert not errs, errs
    for losses, wc in res:
        assert max(abs(a - b) / abs(b) for a, b in zip(losses, l1)) <= 1e-4, (losses, l1)
        assert normwise(wc, m1.wc.double().cpu().numpy()) <= 1e-4
