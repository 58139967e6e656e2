"""world_size-2 (and 3) multi-process tests of the multi-rank host path on CPU (gloo backend).

Each process is a rank.  Through libgt's host entry points (the same code gt_plan uses) every rank
computes the row partition, its halo sets and the lists of rows it sends to each peer; the ranks
then check, across process boundaries, that
  * every rank derived the same partition (collective agreement);
  * what rank s sends to rank r is exactly what r expects from s, in both exchanges (forward
    K||V rows of the out-halo, backward Q||dY rows of the in-halo);
  * an all-to-all-v of synthetic feature rows driven by those lists over torch.distributed delivers
    to every rank exactly the global rows of its halo, in the order the kernels index them;
  * the NCCL bootstrap id created by rank 0 reaches every rank bit-identically;
  * the strategy decision (Alg. 3 on rank 0) is broadcast and agreed.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gtgen


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, seed, result_q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2604_16715_b200 as gt

        rp, ci = gtgen.random_graph(900, 7000, seed=seed, directed=True, power=2.2)
        n = len(rp) - 1
        bounds = gt.partition(rp, world)
        allb = [None] * world
        dist.all_gather_object(allb, bounds.tolist())
        assert all(b == bounds.tolist() for b in allb)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])

        for inward in (False, True):
            halo = gt.halo(rp, ci, lo, hi, inward=inward)
            sends = [gt.send_list(rp, ci, lo, hi, int(bounds[s]), int(bounds[s + 1]), inward=inward).tolist()
                     if s != rank else [] for s in range(world)]
            all_sends = [None] * world
            dist.all_gather_object(all_sends, sends)
            for s in range(world):
                if s == rank:
                    continue
                expect = halo[(halo >= bounds[s]) & (halo < bounds[s + 1])].tolist()
                assert all_sends[s][rank] == expect, (rank, s, inward)

            # all-to-all-v of feature rows following the send lists (row payload = the global rows)
            D = 16
            feat = gtgen.normal_f32(seed, 9, (n, D))
            send_bufs = [torch.from_numpy(feat[np.array(sends[s], dtype=np.int64)]) if sends[s]
                         else torch.zeros((0, D)) for s in range(world)]
            recv_counts = [len(all_sends[s][rank]) if s != rank else 0 for s in range(world)]
            recv_bufs = [torch.zeros((c, D)) for c in recv_counts]
            ops = []
            for s in range(world):
                if s == rank:
                    continue
                if send_bufs[s].shape[0]:
                    ops.append(dist.P2POp(dist.isend, send_bufs[s].contiguous(), s))
                if recv_counts[s]:
                    ops.append(dist.P2POp(dist.irecv, recv_bufs[s], s))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            received = torch.cat([recv_bufs[s] for s in range(world)]) if halo.size else torch.zeros((0, D))
            # the receive table is ordered by owner, then ascending id == the sorted halo order
            np.testing.assert_array_equal(received.numpy(), feat[halo.astype(np.int64)])

        # NCCL bootstrap id: created on rank 0, broadcast through the group
        import ctypes
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            assert gt.lib().gt_nccl_unique_id(ctypes.addressof(uid)) == 0
        t = torch.tensor(list(uid.raw), dtype=torch.uint8)
        dist.broadcast(t, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, bytes(t.tolist()))
        assert all(x == ids[0] for x in ids) and any(ids[0])

        # strategy decision: Alg. 3 evaluated on rank 0, broadcast, identical everywhere
        beta = np.abs(np.random.default_rng(rank).normal(size=(2, world + 1))) * 1e-7
        dec = [gt.agp_select(float(n), 1.0, beta)[:2] if rank == 0 else None]
        dist.broadcast_object_list(dec, src=0)
        decs = [None] * world
        dist.all_gather_object(decs, dec[0])
        assert all(d == decs[0] for d in decs)
        dist.barrier()
        dist.destroy_process_group()
        result_q.put((rank, "ok"))
    except Exception as e:  # reported to the parent
        import traceback
        result_q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world,seed", [(2, 11), (2, 12), (3, 13)])
def test_gloo_multirank_protocol(world, seed):
    from paper_2604_16715_b200 import _build
    _build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert results.get(r) == "ok", results.get(r)


def _agp_worker(rank, world, port, result_q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2604_16715_b200 import agp
        import paper_2604_16715_b200 as gt

        import gtgen
        rp, ci = gtgen.random_graph(3000, 40000, seed=17, directed=False, power=2.2, comm_size=512, f_in=0.9)
        n = len(rp) - 1
        beta, raw, per_row = agp.profile_beta(world, [2048, 8192, 32768], 256, torch.device("cpu"), reps=2,
                                              graph=(rp, ci), N=n)
        if rank == 0:
            for ci_, c in enumerate(agp.COLLECTIVES):
                for p in range(2, world + 1):
                    assert beta[ci_, p] > 0 and np.isfinite(beta[ci_, p]), (c, p)
                    assert per_row[c][p] > 0
                    if c != "halo":
                        assert [r for r, _ in raw[c][p]] == [2048, 8192, 32768]
            # the halo candidate moves exactly the rows of libgt's send lists (forward + backward)
            for p in range(2, world + 1):
                b = gt.partition(rp, p)
                want = sum(len(gt.send_list(rp, ci, b[s], b[s + 1], b[0], b[1], inward))
                           for s in range(1, p) for inward in (False, True))
                assert raw["halo"][p][0][0] == want
            # Alg. 3 on the profiled table: a huge t_iter(1) makes every candidate feasible (the argmin
            # is then the smallest score), a tiny one none (single GPU, reading Z12)
            big = agp.decide(1e6, 1e8, 1e6, beta)
            scores = {(c, p): v["score"] for c, d in big["estimates"].items() for p, v in d.items()}
            best = min(scores.values())
            assert big["score"] == best and big["strategy"] in agp.COLLECTIVES and big["gpus"] >= 2
            assert set(big["estimates"]) == set(agp.COLLECTIVES)
            assert all(v["feasible"] for d in big["estimates"].values() for v in d.values())
            small = agp.decide(1e6, 1e8, 1e-12, beta)
            assert small["strategy"] == "single" and small["gpus"] == 1
            # Eq. 7 / 8 estimate = t1 / p + beta N
            est = big["estimates"]["allgather"][2]["t_iter_est_s"]
            assert abs(est - (1e6 / 2 + beta[0, 2] * 1e6)) <= 1e-9 * est
            # halo wins Alg. 3 when its beta is the smallest
            b2 = beta.copy()
            b2[agp.COLLECTIVES.index("halo"), 2:] = 1e-15
            assert agp.decide(1e6, 1e8, 1e6, b2)["strategy"] == "halo"
        dist.barrier()
        dist.destroy_process_group()
        result_q.put((rank, "ok"))
    except Exception:
        import traceback
        result_q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_agp_beta_profile_and_selection(world):
    """NEXT-2 driver (paper_2604_16715_b200.agp): Fig. 2-style beta sweeps over p = 2..world on a
    gloo group, the log-log fit, and Alg. 3 / Eq. 7-8 on the profiled table."""
    from paper_2604_16715_b200 import _build
    _build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert results.get(r) == "ok", results.get(r)
