"""Automatic graph parallelism over the GPU count.

PAPER.md Section 4:
  * Eq. 7: t_iter(p) = alpha(p) E + beta_c(p) N, with Eq. 8 alpha(s p) = alpha(p) / s;
  * Fig. 2: beta_c(p) is profiled per collective c and GPU count p from message-size sweeps,
    whose time-vs-size relation is linear on log-log axes, so one coefficient per (c, p) (fit: gt_fit_beta);
  * Alg. 3: with k = t_iter(1) / N, keep the candidates i b / (i - 1) <= k over i = 2..P and
    c in the open set of strategies; return the argmin (c, s) (gt_agp_select; reading Z12 for ties / none);
  * Fig. 5: the model's estimate next to the measured iteration time.

Candidates c (COLLECTIVES): GP-AG's all-gather, GP-A2A's all-to-all (Fig. 2 (a), (b)) and the halo
exchange (only the cut rows; reading of Alg. 3's open set).  beta_c(p) is in seconds per
NODE of the graph (t_comm = beta_c(p) N):
  * allgather, a2a: Fig. 2 sweeps of the collective over node-row counts, log-log fit of t = beta rows;
  * halo: the exchange time of libgt's own halo pattern on the actual graph / N - measured by a plan
    (its fwd_exchange + bwd_exchange stage times, CUDA events) on GPUs; on CPU groups (tests) the same
    all-to-all-v with libgt's send lists (gt_send_list) is run through the group's all_to_all.
The planner's beta_profile (gt_opts.beta_profile, --profile-out) is per MOVED ROW at `row_bytes`.

  torchrun --nproc-per-node P -m paper_2604_16715_b200.agp --t-iter1 0.027 --config C3
  python -m paper_2604_16715_b200.agp --fig5 --config C2 --worlds 2,3,4 --out profiles/r02/fig5.json
"""
from __future__ import annotations

import argparse
import json
import math
import os
import threading
import time

import numpy as np

from . import gt

COLLECTIVES = ("allgather", "a2a", "halo")   # strategy index c = position in this tuple


def _timed(fn, device, reps: int) -> float:
    """Median seconds of `fn` over `reps` calls after one warm-up (CUDA events on GPU)."""
    import torch
    fn()
    ts = []
    for _ in range(reps):
        if device.type == "cuda":
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        else:
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def profile_collective(c: str, p: int, rows: int, row_bytes: int, group, device, reps: int = 5) -> float:
    """Time of one collective c among the first p ranks moving `rows` node rows in total (each rank
    contributes rows / p of them), as in the NCCL tests of Fig. 2.  Ranks >= p return 0."""
    import torch
    import torch.distributed as dist
    if dist.get_rank() >= p:
        return 0.0
    per = max(rows // p, 1)
    elems = per * row_bytes // 4
    x = torch.ones(elems, dtype=torch.float32, device=device)
    if c == "allgather":
        out = torch.empty(elems * p, dtype=torch.float32, device=device)
        return _timed(lambda: dist.all_gather_into_tensor(out, x, group=group), device, reps)
    if c == "a2a":
        elems -= elems % p
        x = x[:elems].contiguous()
        out = torch.empty_like(x)
        return _timed(lambda: dist.all_to_all_single(out, x, group=group), device, reps)
    raise ValueError(c)


def halo_counts(row_ptr, col_idx, p: int, rank: int):
    """Rows rank `rank` sends to / receives from every peer in the forward and backward halo exchanges at
    world p (libgt's host planning: gt_partition + gt_send_list, the lists gt_plan uses)."""
    b = gt.partition(row_ptr, p)
    send, recv = [0] * p, [0] * p
    for s in range(p):
        if s == rank:
            continue
        for inward in (False, True):
            send[s] += len(gt.send_list(row_ptr, col_idx, b[rank], b[rank + 1], b[s], b[s + 1], inward))
            recv[s] += len(gt.send_list(row_ptr, col_idx, b[s], b[s + 1], b[rank], b[rank + 1], inward))
    return send, recv


def profile_halo_group(row_ptr, col_idx, p: int, row_bytes: int, group, device, reps: int = 5):
    """Halo exchange time at world p through the group's all_to_all with libgt's send lists (CPU groups,
    tests).  Returns (seconds, rows moved by the slowest rank)."""
    import torch
    import torch.distributed as dist
    r = dist.get_rank()
    if r >= p:
        return 0.0, 0
    send, recv = halo_counts(row_ptr, col_idx, p, r)
    w = row_bytes // 4
    x = torch.ones(sum(send) * w, dtype=torch.float32, device=device)
    out = torch.empty(sum(recv) * w, dtype=torch.float32, device=device)
    t = _timed(lambda: dist.all_to_all_single(out, x, [c * w for c in recv], [c * w for c in send], group=group),
               device, reps)
    return t, sum(recv)


def profile_halo_plan(row_ptr, col_idx, heads: int, d: int, dtype: str, comm, world: int, rank: int,
                      steps: int = 5):
    """Halo exchange time of libgt's own exchange (GPU): a plan with strategy "halo" is stepped
    (fwd + bwd) with per-stage CUDA events; returns (exchange seconds per step, rows received per step,
    the plan's info).  Collective over `comm`."""
    import torch
    plan = gt.Plan(row_ptr, col_idx, heads, d, dtype=dtype, world=world, rank=rank, comm=comm, strategy="halo",
                   profile=True)
    n = plan.n_local
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = [torch.randn(n, heads, d, device="cuda").to(tdt) for _ in range(4)]
    for _ in range(2):
        y, lse = plan.fwd(*x[:3])
        plan.bwd(*x[:3], y, lse, x[3])
    torch.cuda.synchronize()
    plan.timings()
    for _ in range(steps):
        y, lse = plan.fwd(*x[:3])
        plan.bwd(*x[:3], y, lse, x[3])
    torch.cuda.synchronize()
    st = plan.timings()
    info = plan.info()
    plan.close()
    t = (st["fwd_exchange"][0] + st["bwd_exchange"][0]) * 1e-3 / steps
    elt = 2 if dtype == "bf16" else 4
    kv_row = 2 * heads * d * elt                            # [k | v] rows forward
    in_row = kv_row + (8 * heads + 15) // 16 * 16           # [q | dy | (LSE2, D)] rows backward
    rows = info["exch_fwd_bytes"] / kv_row + info["exch_bwd_bytes"] / in_row
    return t, rows, info


def profile_beta(P: int, sizes, row_bytes: int, device, reps: int = 5, graph=None, N: float = 0.0):
    """beta[c, p] in seconds per node for p = 2..P (Fig. 2 sweeps + the log-log fit; halo: the graph's
    halo exchange / N); columns 0 and 1 unused.  Collective over the default group: every rank calls it;
    p-subgroups are created in order.  `graph` = (row_ptr, col_idx) enables the halo candidate (CPU
    groups: all_to_all with libgt's send lists).  Returns (beta [len(COLLECTIVES), P + 1],
    raw {c: {p: [(rows, seconds)]}}, per-moved-row beta {c: {p: s}})."""
    import torch.distributed as dist
    beta = np.zeros((len(COLLECTIVES), P + 1))
    beta[COLLECTIVES.index("halo"), :] = np.inf if graph is None else 0.0
    raw = {c: {} for c in COLLECTIVES}
    per_row = {c: {} for c in COLLECTIVES}
    for p in range(2, P + 1):
        group = dist.new_group(list(range(p)))
        for ci, c in enumerate(COLLECTIVES):
            if c == "halo":
                if graph is None:
                    continue
                t, rows = profile_halo_group(graph[0], graph[1], p, row_bytes, group, device, reps)
                if dist.get_rank() < p:
                    # the slowest rank's time (max over the subgroup) is the exchange time of the step
                    tmax = _max_over(t, group)
                    raw[c][p] = [(int(rows), tmax)]
                    beta[ci, p] = max(tmax, 1e-12) / max(N, 1.0)
                    per_row[c][p] = max(tmax, 1e-12) / max(rows, 1)
                continue
            pts = []
            for rows in sizes:
                t = profile_collective(c, p, int(rows), row_bytes, group, device, reps)
                pts.append((int(rows), t))
            raw[c][p] = pts
            if dist.get_rank() < p:
                x = np.array([r for r, _ in pts], np.float64)
                y = np.array([max(t, 1e-9) for _, t in pts], np.float64)
                beta[ci, p] = gt.fit_beta(x, y)     # s per node row = s per node (rows = N nodes)
                per_row[c][p] = beta[ci, p]
        dist.barrier()
    # rank 0 is in every subgroup; its table is the one used
    return beta, raw, per_row


def _max_over(t: float, group) -> float:
    import torch
    import torch.distributed as dist
    x = torch.tensor([t], dtype=torch.float64)
    dist.all_reduce(x, op=dist.ReduceOp.MAX, group=group)
    return float(x.item())


def decide(N: float, E: float, t_iter1: float, beta: np.ndarray) -> dict:
    """Alg. 3 decision plus the Eq. 7/8 estimates (the Fig. 5 'estimated' series) and the Eq. 14
    feasibility of every (c, p).  Rows of `beta` follow COLLECTIVES; a candidate with no finite beta is
    left out (beta = +inf never passes the feasibility test)."""
    P = beta.shape[1] - 1
    b = np.where(np.isfinite(beta), beta, 1e300)
    c, s, score = gt.agp_select(N, t_iter1, b)
    alpha1 = t_iter1 / E if E > 0 else 0.0  # Eq. 7 at p = 1 with the communication term 0
    k = t_iter1 / N
    est = {}
    for ci, name in enumerate(COLLECTIVES[:beta.shape[0]]):
        if not np.isfinite(beta[ci, 2:]).any():
            continue
        est[name] = {}
        for p in range(2, P + 1):
            bb = float(beta[ci, p])
            est[name][p] = {"beta_s_per_node": bb,
                            "t_iter_est_s": gt.estimate_iter_time(alpha1, b, ci, p, N, E),
                            "score": p * bb / (p - 1), "feasible": p * bb / (p - 1) <= k}
    return {"strategy": COLLECTIVES[c] if c >= 0 else "single", "gpus": s, "score": score, "k": k,
            "estimates": est}


# --------------------------------------------------------------------------- Fig. 5 analog --
def fig5_loopback(row_ptr, col_idx, heads: int, d: int, dtype: str, worlds, steps: int = 5,
                  strategies=("allgather", "halo", "a2a")):
    """Estimated vs measured iteration time (Fig. 5) over in-process loopback worlds on one GPU.

    For every world p and strategy c: the Eq. 7/8 estimate t(1)/p + beta_c(p) N with beta_c(p) =
    the measured exchange time of that plan / N; the plan's own prediction (gt_plan_info predicted_ms);
    the measured per-step time (max over ranks of the ranks' own stage times, CUDA events); and what
    GT_AUTO picks at that p.  Caveat (one GPU): the p ranks share one device, so their kernels and
    copies interleave - the measured compute is not t(1)/p, and the comparison validates the model's
    bookkeeping (volumes, beta, the choice), not multi-GPU scaling."""
    import torch
    n = len(row_ptr) - 1
    E = int(row_ptr[-1])
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    full = [torch.randn(n, heads, d, device="cuda", generator=torch.Generator("cuda").manual_seed(i)).to(tdt)
            for i in range(4)]

    def run(world, strategy):
        grp = gt.LoopbackGroup(world) if world > 1 else None
        out = [None] * world
        errs = []

        def worker(r):
            try:
                torch.cuda.set_device(0)
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    plan = gt.Plan(row_ptr, col_idx, heads, d, dtype=dtype, world=world, rank=r, comm=grp,
                                   strategy=strategy, profile=True)
                    lo, hi = plan.row_lo, plan.row_hi
                    x = [t[lo:hi].contiguous() for t in full]
                    for _ in range(2):
                        y, lse = plan.fwd(*x[:3])
                        plan.bwd(*x[:3], y, lse, x[3])
                    s.synchronize()
                    plan.timings()
                    for _ in range(steps):
                        y, lse = plan.fwd(*x[:3])
                        plan.bwd(*x[:3], y, lse, x[3])
                    s.synchronize()
                    st = plan.timings()
                    out[r] = ({k: v[0] / steps for k, v in st.items()}, plan.info())
                    plan.close()
            except Exception as e:
                errs.append((r, repr(e)))

        th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if grp:
            grp.close()
        if errs:
            raise RuntimeError(errs)
        return out

    base = run(1, "single")[0][0]
    t1 = sum(base.values()) * 1e-3
    rows = [{"p": 1, "strategy": "single", "measured_ms": t1 * 1e3, "stages_ms": base}]
    for p in worlds:
        auto_info = run(p, "auto")[0][1]        # GT_AUTO probes every candidate: its predictions
        auto = auto_info["strategy_name"]
        for c in strategies:
            try:
                res = run(p, c)
            except Exception as e:  # e.g. GP-A2A needs heads % p == 0
                rows.append({"p": p, "strategy": c, "error": str(e)[:200]})
                continue
            meas = max(sum(st.values()) for st, _ in res) * 1e-3
            exch = max(st["fwd_exchange"] + st["bwd_exchange"] for st, _ in res) * 1e-3
            beta = exch / n
            info = res[0][1]
            ci = {"allgather": 2, "halo": 3, "a2a": 4}[c]
            rows.append({"p": p, "strategy": c, "auto_choice": auto,
                         "eq7_estimate_ms": (t1 / p + beta * n) * 1e3,
                         "plan_predicted_ms": (auto_info["predicted_ms"][ci]
                                               if np.isfinite(auto_info["predicted_ms"][ci]) else None),
                         "measured_ms": meas * 1e3, "measured_exchange_ms": exch * 1e3,
                         "beta_s_per_node": beta, "alg3_score_ms": p * beta * n / (p - 1) * 1e3,
                         "exch_bytes_rank0": info["exch_fwd_bytes"] + info["exch_bwd_bytes"]})
    return {"nodes": n, "nnz": E, "heads": heads, "d": d, "dtype": dtype, "t_iter1_ms": t1 * 1e3,
            "device": torch.cuda.get_device_name(), "rows": rows,
            "caveat": "loopback ranks share one GPU: measured times are not multi-GPU times"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t-iter1", type=float, default=None, help="measured single-GPU step time (s)")
    ap.add_argument("--nodes", type=float, default=None)
    ap.add_argument("--edges", type=float, default=None)
    ap.add_argument("--config", default=None, help="gtgen config (C1..C5): graph for the halo candidate")
    ap.add_argument("--row-bytes", type=int, default=1024, help="bytes per exchanged node row (K||V at D=256 bf16)")
    ap.add_argument("--sizes", default="65536,262144,1048576", help="node rows per collective (sweep)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--profile-out", default=None,
                    help="write {collective: {GPU count: beta per moved row}, row_bytes} for gt_opts.beta_profile")
    ap.add_argument("--fig5", action="store_true", help="Fig. 5 analog over loopback worlds on one GPU")
    ap.add_argument("--worlds", default="2,4")
    args = ap.parse_args()
    import torch
    import gtgen  # seeded input graphs (no method arithmetic)
    graph = None
    if args.config:
        cfg = gtgen.CONFIGS[args.config]
        graph = gtgen.make_graph(cfg.graph)
    if args.fig5:
        res = fig5_loopback(graph[0], graph[1], cfg.heads, cfg.d, cfg.dtype, [int(x) for x in args.worlds.split(",")])
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(line + "\n")
        return
    import torch.distributed as dist
    cuda = torch.cuda.is_available()
    if cuda:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl" if cuda else "gloo")
    device = torch.device("cuda", torch.cuda.current_device()) if cuda else torch.device("cpu")
    P = dist.get_world_size()
    N = args.nodes if args.nodes else (len(graph[0]) - 1 if graph else 0)
    E = args.edges if args.edges else (int(graph[0][-1]) if graph else 0)
    sizes = [int(x) for x in args.sizes.split(",")]
    beta, raw, per_row = profile_beta(P, sizes, args.row_bytes, device, args.reps,
                                      graph=None if cuda else graph, N=N)
    if cuda and graph is not None:
        # the halo candidate through libgt's own exchange: a plan per GPU count p (NCCL sub-communicator)
        hi = COLLECTIVES.index("halo")
        for p in range(2, P + 1):
            group = dist.new_group(list(range(p)))
            if dist.get_rank() < p:
                comm = gt.NcclComm(group)
                t, rows, _ = profile_halo_plan(graph[0], graph[1], cfg.heads, cfg.d, cfg.dtype, comm, p,
                                               dist.get_rank(group))
                comm.close()
                t = _max_over_cuda(t, group)
                beta[hi, p] = t / max(N, 1)
                per_row["halo"][p] = t / max(rows or 1, 1)
                raw["halo"][p] = [(rows, t)]
            dist.barrier()
    if dist.get_rank() == 0:
        t1 = args.t_iter1 if args.t_iter1 else 1.0
        res = decide(N, E, t1, beta)
        res["profile"] = {c: {str(p): pts for p, pts in d.items()} for c, d in raw.items()}
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(line + "\n")
        if args.profile_out:
            prof = {c: {str(p): float(v) for p, v in per_row[c].items()} for c in COLLECTIVES if per_row[c]}
            prof["row_bytes"] = args.row_bytes
            with open(args.profile_out, "w") as f:
                json.dump(prof, f)
    dist.destroy_process_group()


def _max_over_cuda(t: float, group) -> float:
    import torch
    import torch.distributed as dist
    x = torch.tensor([t], dtype=torch.float64, device="cuda")
    dist.all_reduce(x, op=dist.ReduceOp.MAX, group=group)
    return float(x.item())


if __name__ == "__main__":
    main()
