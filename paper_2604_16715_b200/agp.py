"""Automatic graph parallelism over the GPU count.

PAPER.md Section 4:
  * Eq. 7: t_iter(p) = alpha(p) E + beta_c(p) N, with Eq. 8 alpha(s p) = alpha(p) / s;
  * Fig. 2: beta_c(p) is profiled per collective c and GPU count p from message-size sweeps,
    whose time-vs-size relation is linear on log-log axes, so one coefficient per (c, p) (fit: gt_fit_beta);
  * Alg. 3: with k = t_iter(1) / N, keep the candidates i b / (i - 1) <= k over i = 2..P and
    c in {GP-AG, GP-A2A, ...}; return the argmin (c, s) (gt_agp_select; reading Z12 for ties / none);
  * Fig. 5: the model's estimate next to the measured iteration time.

This module is the host-side driver: it profiles beta with the collectives of a torch.distributed group
(NCCL on GPUs; gloo on CPU for tests), measures nothing of the attention itself (the caller passes
t_iter(1), e.g. bench.py's single-GPU step), and evaluates Alg. 3 with the library's C routines.  Beta
is in seconds per node row of `row_bytes` bytes (reading Z14).

  torchrun --nproc-per-node P -m paper_2604_16715_b200.agp --t-iter1 0.0351 --nodes 2449029 --edges 123718280
"""
from __future__ import annotations

import argparse
import json
import os
import time

import numpy as np

from . import gt

COLLECTIVES = ("allgather", "a2a")   # Fig. 2 (a) and (b); strategy index c = position in this tuple


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


def profile_beta(P: int, sizes, row_bytes: int, device, reps: int = 5):
    """beta[c, p] in seconds per node row for p = 2..P (Fig. 2 sweeps + the log-log fit); column 0 and
    1 unused.  Collective over the default group: every rank calls it; p-subgroups are created for
    every p in order.  Returns (beta [len(COLLECTIVES), P + 1], raw {c: {p: [(rows, seconds)]}})."""
    import torch.distributed as dist
    beta = np.zeros((len(COLLECTIVES), P + 1))
    raw = {c: {} for c in COLLECTIVES}
    for p in range(2, P + 1):
        group = dist.new_group(list(range(p)))
        for ci, c in enumerate(COLLECTIVES):
            pts = []
            for rows in sizes:
                t = profile_collective(c, p, int(rows), row_bytes, group, device, reps)
                pts.append((int(rows), t))
            raw[c][p] = pts
            if dist.get_rank() < p:
                x = np.array([r for r, _ in pts], np.float64)
                y = np.array([max(t, 1e-9) for _, t in pts], np.float64)
                beta[ci, p] = gt.fit_beta(x, y)
        dist.barrier()
    # rank 0 is in every subgroup; its table is the one used
    return beta, raw


def decide(N: float, E: float, t_iter1: float, beta: np.ndarray) -> dict:
    """Alg. 3 decision plus the Eq. 7/8 estimates (the Fig. 5 'estimated' series) and the Eq. 14
    feasibility of every (c, p)."""
    P = beta.shape[1] - 1
    c, s, score = gt.agp_select(N, t_iter1, beta)
    alpha1 = t_iter1 / E if E > 0 else 0.0  # Eq. 7 at p = 1 with the communication term 0
    k = t_iter1 / N
    est = {}
    for ci, name in enumerate(COLLECTIVES):
        est[name] = {}
        for p in range(2, P + 1):
            b = float(beta[ci, p])
            est[name][p] = {"beta_s_per_node": b,
                            "t_iter_est_s": gt.estimate_iter_time(alpha1, beta, ci, p, N, E),
                            "score": p * b / (p - 1), "feasible": p * b / (p - 1) <= k}
    return {"strategy": COLLECTIVES[c] if c >= 0 else "single", "gpus": s, "score": score, "k": k,
            "estimates": est}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t-iter1", type=float, required=True, help="measured single-GPU step time (s)")
    ap.add_argument("--nodes", type=float, required=True)
    ap.add_argument("--edges", type=float, required=True)
    ap.add_argument("--row-bytes", type=int, default=1024, help="bytes per exchanged node row (K||V at D=256 bf16)")
    ap.add_argument("--sizes", default="65536,262144,1048576", help="node rows per collective (sweep)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--profile-out", default=None,
                    help="write {collective: {GPU count: beta}} for gt_opts.beta_profile (Plan(beta_profile=...))")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    cuda = torch.cuda.is_available()
    if cuda:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl" if cuda else "gloo")
    device = torch.device("cuda", torch.cuda.current_device()) if cuda else torch.device("cpu")
    P = dist.get_world_size()
    sizes = [int(x) for x in args.sizes.split(",")]
    beta, raw = profile_beta(P, sizes, args.row_bytes, device, args.reps)
    if dist.get_rank() == 0:
        res = decide(args.nodes, args.edges, args.t_iter1, beta)
        res["profile"] = {c: {str(p): pts for p, pts in d.items()} for c, d in raw.items()}
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(line + "\n")
        if args.profile_out:
            prof = {c: {str(p): float(beta[ci, p]) for p in range(2, P + 1)} for ci, c in enumerate(COLLECTIVES)}
            with open(args.profile_out, "w") as f:
                json.dump(prof, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
