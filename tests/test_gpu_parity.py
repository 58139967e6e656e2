"""GPU parity: libgt (C ABI, CUDA sm_100a) vs the fp64 CPU oracle, element by element.

Tolerances (BASELINE.json north_star; reading Z8): normwise max relative error <= 1e-4 (fp32) and
<= 2e-2 (bf16) for Y, dQ, dK, dV; LSE absolute <= 1e-4 / 1e-2 with -inf exactly on empty rows;
integer tables (CSC) bit-exact.
"""
import math

import numpy as np
import pytest

import gtgen
import oracle
from tests._util import TOL, check_lse, inputs, normwise, to_f64, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gt():
    import paper_2604_16715_b200 as g
    return g


def run_case(gt, row_ptr, col_idx, h, d, dtype, seed, scale=None, qk_scale=1.0, heavy=0, q_zero=False,
             edge_state=0):
    import torch
    n = len(row_ptr) - 1
    q, k, v, dy = inputs(n, h, d, dtype, seed, qk_scale)
    if q_zero:
        q = np.zeros_like(q)
    scale = scale if scale is not None else 1.0 / math.sqrt(h * d)
    plan = gt.Plan(row_ptr, col_idx, h, d, dtype=dtype, scale=scale, heavy_threshold=heavy, edge_state=edge_state)
    assert plan.info()["edge_state"] == (0 if edge_state < 0 else 1)
    tq, tk, tv, tdy = (to_torch(x) for x in (q, k, v, dy))
    y, lse = plan.fwd(tq, tk, tv)
    dq, dk, dv = plan.bwd(tq, tk, tv, y, lse, tdy)
    torch.cuda.synchronize()
    Y, LSE = oracle.forward(row_ptr, col_idx, q, k, v, scale)
    DQ, DK, DV, _ = oracle.backward(row_ptr, col_idx, q, k, v, dy, scale)
    errs = {"y": normwise(to_f64(y), Y), "dq": normwise(to_f64(dq), DQ), "dk": normwise(to_f64(dk), DK),
            "dv": normwise(to_f64(dv), DV)}
    check_lse(to_f64(lse), LSE, dtype)
    for name, e in errs.items():
        assert e <= TOL[dtype], f"{name}: normwise error {e:.3e} > {TOL[dtype]}"
    return plan, errs, (tq, tk, tv, tdy), (y, lse, dq, dk, dv)


def test_c1_cora_f32(gt):
    c = gtgen.CONFIGS["C1"]
    rp, ci = gtgen.make_graph(c.graph)
    run_case(gt, rp, ci, c.heads, c.d, c.dtype, seed=101)


def test_c2_arxiv_bf16(gt):
    c = gtgen.CONFIGS["C2"]
    rp, ci = gtgen.make_graph(c.graph)
    run_case(gt, rp, ci, c.heads, c.d, c.dtype, seed=102)


SHAPES = [  # h, d, dtype
    (4, 64, "bf16"), (4, 64, "f32"), (8, 16, "f32"), (8, 32, "bf16"), (1, 128, "bf16"), (2, 64, "f32"),
    (2, 256, "bf16"), (8, 64, "f32"), (1, 256, "f32"), (4, 32, "bf16"),
    (1, 64, "bf16"), (4, 16, "bf16"), (8, 8, "f32"), (2, 32, "f32"),   # heads * d = 64 (4-byte bf16 lane slices)
]


# edge_state 1: materialised logits and (P, dP) (default plan); -1: recompute kernels
@pytest.mark.parametrize("edge_state", [1, -1])
@pytest.mark.parametrize("h,d,dtype", SHAPES)
def test_shapes_power_law_with_chunking(gt, h, d, dtype, edge_state):
    rp, ci = gtgen.random_graph(3000, 45000, seed=7 + h + d, directed=True, power=2.05)
    run_case(gt, rp, ci, h, d, dtype, seed=200 + h * d, heavy=48, edge_state=edge_state)


@pytest.mark.parametrize("edge_state", [1, -1])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_peaked_softmax_logits_x8(gt, dtype, edge_state):
    rp, ci = gtgen.random_graph(2000, 30000, seed=31, power=2.2)
    run_case(gt, rp, ci, 4, 64, dtype, seed=301, scale=8.0 / math.sqrt(64), heavy=64, edge_state=edge_state)


def test_all_equal_logits(gt):
    rp, ci = gtgen.random_graph(1500, 20000, seed=32, power=2.2)
    run_case(gt, rp, ci, 4, 64, "f32", seed=302, q_zero=True, heavy=40)


def test_empty_graph_and_isolated_rows(gt):
    n = 37
    rp = np.zeros(n + 1, np.int64)
    ci = np.zeros(0, np.int32)
    plan, errs, ins, outs = run_case(gt, rp, ci, 4, 32, "bf16", seed=303)
    y, lse, dq, dk, dv = outs
    assert float(y.abs().max()) == 0.0 and float(dq.abs().max()) == 0.0
    assert float(dk.abs().max()) == 0.0 and float(dv.abs().max()) == 0.0


@pytest.mark.parametrize("edge_state", [1, -1])
def test_single_edge_and_star(gt, edge_state):
    rp, ci = gtgen.csr_from_pairs(5, [(3, 1)])
    run_case(gt, rp, ci, 2, 64, "f32", seed=304, edge_state=edge_state)
    n = 700  # hub row 0 -> all, all -> hub column 0: exercises chunked rows and chunked columns
    pairs = [(0, j) for j in range(1, n)] + [(j, 0) for j in range(1, n)]
    rp, ci = gtgen.csr_from_pairs(n, pairs)
    plan, *_ = run_case(gt, rp, ci, 4, 64, "bf16", seed=305, heavy=100, edge_state=edge_state)
    inf = plan.info()
    assert inf["heavy_rows"] == 1 and inf["heavy_cols"] == 1 and inf["heavy_row_chunks"] == 7


def test_one_row_single_node(gt):
    rp, ci = gtgen.csr_from_pairs(1, [(0, 0)])
    run_case(gt, rp, ci, 1, 128, "f32", seed=306)


@pytest.mark.parametrize("edge_state", [1, -1])
def test_csc_bitexact_and_deterministic(gt, edge_state):
    import torch
    rp, ci = gtgen.random_graph(5000, 80000, seed=41, power=2.1)
    plan, errs, ins, outs = run_case(gt, rp, ci, 4, 64, "bf16", seed=401, heavy=128, edge_state=edge_state)
    cp, ri = oracle.transpose(rp, ci)
    np.testing.assert_array_equal(plan.export("csc_ptr"), cp)
    np.testing.assert_array_equal(plan.export("csc_idx"), ri)
    # bitwise run-to-run determinism (no atomics in the numerics)
    tq, tk, tv, tdy = ins
    y2, lse2 = plan.fwd(tq, tk, tv)
    dq2, dk2, dv2 = plan.bwd(tq, tk, tv, y2, lse2, tdy)
    torch.cuda.synchronize()
    for a, b in zip(outs, (y2, lse2, dq2, dk2, dv2)):
        assert torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a,
                           b.view(torch.int16) if b.dtype == torch.bfloat16 else b)


def test_autograd_wrapper(gt):
    import torch
    rp, ci = gtgen.random_graph(800, 9000, seed=51, power=2.3)
    h, d = 4, 32
    q, k, v, dy = inputs(800, h, d, "f32", 501)
    plan = gt.Plan(rp, ci, h, d, dtype="f32")
    tq, tk, tv = (to_torch(x).requires_grad_(True) for x in (q, k, v))
    y = gt.sparse_graph_attention(plan, tq, tk, tv)
    y.backward(to_torch(dy))
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, plan.scale)
    assert normwise(to_f64(tq.grad), DQ) <= 1e-4
    assert normwise(to_f64(tk.grad), DK) <= 1e-4
    assert normwise(to_f64(tv.grad), DV) <= 1e-4


def test_host_buffer_entry_point(gt):
    import torch
    rp, ci = gtgen.random_graph(1200, 15000, seed=61, power=2.2)
    h, d = 4, 64
    q, k, v, dy = inputs(1200, h, d, "bf16", 601)
    plan = gt.Plan(rp, ci, h, d, dtype="bf16")
    pin = lambda x: to_torch(x, "cpu").pin_memory()  # noqa: E731
    tq, tk, tv, tdy = (pin(x) for x in (q, k, v, dy))
    y, dq, dk, dv = (torch.empty_like(tq).pin_memory() for _ in range(4))
    lse = torch.empty((1200, h), dtype=torch.float32).pin_memory()
    plan.fwd_bwd_host(tq, tk, tv, tdy, y, lse, dq, dk, dv)
    Y, LSE = oracle.forward(rp, ci, q, k, v, plan.scale)
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, plan.scale)
    assert normwise(to_f64(y), Y) <= 2e-2 and normwise(to_f64(dq), DQ) <= 2e-2
    assert normwise(to_f64(dk), DK) <= 2e-2 and normwise(to_f64(dv), DV) <= 2e-2
    check_lse(lse.numpy(), LSE, "bf16")


@pytest.mark.parametrize("chunks", ["1", "3", "8", "64"])
def test_host_buffer_streamed_chunks(gt, chunks, monkeypatch):
    """World-1 gt_attn_fwd_bwd_host streams rows (columns) in chunks: heavy rows whole inside a chunk and
    merged with it, rows without entries filled once, outputs copied out per chunk; any chunk count
    gives the oracle's results (power-law graph with empty rows and chunked heavy rows)."""
    import torch
    monkeypatch.setenv("GT_E2E_CHUNKS", chunks)
    rp, ci = gtgen.random_graph(2600, 30000, seed=63, directed=True, power=2.05)
    n, h, d = len(rp) - 1, 4, 64
    assert (np.diff(rp) == 0).any()
    q, k, v, dy = inputs(n, h, d, "bf16", 603)
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", heavy_threshold=48)
    assert plan.info()["heavy_rows"] > 0 and plan.info()["heavy_cols"] > 0
    pin = lambda x: to_torch(x, "cpu").pin_memory()  # noqa: E731
    tq, tk, tv, tdy = (pin(x) for x in (q, k, v, dy))
    Y, LSE = oracle.forward(rp, ci, q, k, v, plan.scale)
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, plan.scale)
    for _ in range(2):
        y, dq, dk, dv = (torch.full_like(tq, float("nan")).pin_memory() for _ in range(4))
        lse = torch.full((n, h), float("nan"), dtype=torch.float32).pin_memory()
        plan.fwd_bwd_host(tq, tk, tv, tdy, y, lse, dq, dk, dv)
        assert normwise(to_f64(y), Y) <= 2e-2 and normwise(to_f64(dq), DQ) <= 2e-2
        assert normwise(to_f64(dk), DK) <= 2e-2 and normwise(to_f64(dv), DV) <= 2e-2
        check_lse(lse.numpy(), LSE, "bf16")
    # bitwise reproducible across calls (the chunk schedule does not change the arithmetic order)
    outs2 = [torch.empty_like(tq).pin_memory() for _ in range(4)]
    lse2 = torch.empty((n, h), dtype=torch.float32).pin_memory()
    plan.fwd_bwd_host(tq, tk, tv, tdy, outs2[0], lse2, outs2[1], outs2[2], outs2[3])
    for a, b in zip((y, dq, dk, dv, lse), (*outs2, lse2)):
        assert torch.equal(a, b)
    # the device API afterwards sees a consistent plan (the host path left the forward state tagged)
    dev = [to_torch(x) for x in (q, k, v, dy)]
    yd, ld = plan.fwd(*dev[:3])
    g = plan.bwd(*dev[:3], yd, ld, dev[3])
    torch.cuda.synchronize()
    assert normwise(to_f64(g[0]), DQ) <= 2e-2 and normwise(to_f64(g[1]), DK) <= 2e-2
    # and the chunked host schedule computes exactly what the device API computes
    for a, b in zip((yd, ld, *g), (y, lse, dq, dk, dv)):
        assert torch.equal(a.cpu(), b)
    plan.close()


@pytest.mark.parametrize("case", ["empty", "one_hub", "single_edge"])
def test_host_buffer_streamed_degenerate(gt, case, monkeypatch):
    """The streamed host path on graphs with no entries, one hub row / column carrying every entry
    (a single chunked row: no row-chunk cut exists), and one edge among isolated nodes."""
    import torch
    monkeypatch.setenv("GT_E2E_CHUNKS", "8")
    if case == "empty":
        rp, ci = np.zeros(40, np.int64), np.zeros(0, np.int32)
    elif case == "one_hub":
        n = 600
        rp, ci = gtgen.csr_from_pairs(n, [(0, j) for j in range(1, n)] + [(j, 0) for j in range(1, n)])
    else:
        rp, ci = gtgen.csr_from_pairs(9, [(4, 7)])
    n, h, d = len(rp) - 1, 4, 64
    q, k, v, dy = inputs(n, h, d, "bf16", 607)
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", heavy_threshold=64)
    pin = lambda x: to_torch(x, "cpu").pin_memory()  # noqa: E731
    tq, tk, tv, tdy = (pin(x) for x in (q, k, v, dy))
    y, dq, dk, dv = (torch.full_like(tq, float("nan")).pin_memory() for _ in range(4))
    lse = torch.full((n, h), float("nan"), dtype=torch.float32).pin_memory()
    plan.fwd_bwd_host(tq, tk, tv, tdy, y, lse, dq, dk, dv)
    Y, LSE = oracle.forward(rp, ci, q, k, v, plan.scale)
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, plan.scale)
    for a, r in ((y, Y), (dq, DQ), (dk, DK), (dv, DV)):
        assert not torch.isnan(a.float()).any()
        assert normwise(to_f64(a), r) <= 2e-2
    check_lse(lse.numpy(), LSE, "bf16")
    plan.close()


@pytest.mark.parametrize("dtype,h,d", [("bf16", 4, 64), ("f32", 8, 16)])
def test_hot_column_table(gt, dtype, h, d):
    """gt_opts.hot_cols: the most referenced columns' K||V rows are read from a packed table under a
    persisting L2 window; outputs are the oracle's, through the device API (incl. a backward of another
    forward's k, v, which re-packs) and the streamed host-buffer step."""
    import torch
    rp, ci = gtgen.random_graph(3000, 45000, seed=64, directed=True, power=1.9)
    n = len(rp) - 1
    A = inputs(n, h, d, dtype, 641)
    B = inputs(n, h, d, dtype, 642, qk_scale=3.0)
    plan = gt.Plan(rp, ci, h, d, dtype=dtype, heavy_threshold=64, hot_cols=200)
    info = plan.info()
    indeg = np.bincount(ci, minlength=n)
    assert info["hot_cols"] == 200 and info["hot_entries"] == np.sort(indeg)[-200:].sum()
    ta, tb = [to_torch(x) for x in A], [to_torch(x) for x in B]
    ya, la = plan.fwd(*ta[:3])
    yb, lb = plan.fwd(*tb[:3])
    ga = plan.bwd(*ta[:3], ya, la, ta[3])      # the table holds B's rows: re-packed
    torch.cuda.synchronize()
    for X, (y, l, g) in ((A, (ya, la, ga)), (B, (yb, lb, None))):
        Y, LSE = oracle.forward(rp, ci, *X[:3], plan.scale)
        assert normwise(to_f64(y), Y) <= TOL[dtype]
        check_lse(to_f64(l), LSE, dtype)
        if g is not None:
            DQ, DK, DV, _ = oracle.backward(rp, ci, *X, plan.scale)
            for a, r in zip(g, (DQ, DK, DV)):
                assert normwise(to_f64(a), r) <= TOL[dtype]
    pin = lambda x: to_torch(x, "cpu").pin_memory()  # noqa: E731
    hq, hk, hv, hdy = (pin(x) for x in B)
    outs = [torch.empty_like(hq).pin_memory() for _ in range(4)]
    hl = torch.empty((n, h), dtype=torch.float32).pin_memory()
    plan.fwd_bwd_host(hq, hk, hv, hdy, outs[0], hl, outs[1], outs[2], outs[3])
    DQ, DK, DV, _ = oracle.backward(rp, ci, *B, plan.scale)
    for a, r in zip(outs[1:], (DQ, DK, DV)):
        assert normwise(to_f64(a), r) <= TOL[dtype]
    plan.close()


def test_errors_are_reported(gt):
    rp, ci = gtgen.csr_from_pairs(4, [(0, 1), (1, 2)])
    bad = ci.copy()
    bad[0] = 7
    with pytest.raises(gt.GTError) as e:
        gt.Plan(rp, bad, 4, 64)
    assert e.value.status == 2  # GT_EGRAPH
    with pytest.raises(gt.GTError) as e:
        gt.Plan(rp, ci, 3, 64)
    assert e.value.status == 3  # GT_ECONFIG
    unsorted = gtgen.csr_from_pairs(3, [(0, 1), (0, 2)])
    uc = unsorted[1][::-1].copy()
    with pytest.raises(gt.GTError):
        gt.Plan(unsorted[0], uc, 4, 64)
    with pytest.raises(gt.GTError) as e:
        gt.Plan(rp, ci, 4, 64, edge_state=2)
    assert e.value.status == 1  # GT_EINVAL
    # shape / dtype / device errors of the binding: GT_EINVAL, no kernel launched
    import torch
    plan = gt.Plan(rp, ci, 4, 64, dtype="f32", edge_state=1)
    z = torch.zeros((4, 4, 64), dtype=torch.float32, device="cuda")
    lz = torch.zeros((4, 4), dtype=torch.float32, device="cuda")
    bad_cases = [
        lambda: plan.fwd(torch.zeros((3, 4, 64), device="cuda"), z, z),                # n_local
        lambda: plan.fwd(z, torch.zeros((4, 2, 128), device="cuda"), z),               # heads, d
        lambda: plan.fwd(z, z, z.to(torch.bfloat16)),                                  # dtype
        lambda: plan.fwd(z, z, torch.zeros((4, 64, 4), device="cuda").transpose(1, 2)),  # layout
        lambda: plan.fwd(z, z, z, y=torch.zeros((2, 4, 64), device="cuda")),            # output shape
        lambda: plan.fwd(z, z, z, lse=torch.zeros((4, 4), dtype=torch.float64, device="cuda")),
        lambda: plan.bwd(z, z, z, z, torch.zeros((4, 3), device="cuda"), z),              # lse shape
        lambda: plan.bwd(z, z, z, z, lz.to(torch.bfloat16), z),                           # lse dtype
        lambda: plan.bwd(z, z, z, z, lz, z, dq=torch.zeros((5, 4, 64), device="cuda")),   # output shape
        lambda: plan.bwd(z.cpu(), z, z, z, lz, z),                                        # device
    ]
    for i, f in enumerate(bad_cases):
        with pytest.raises(gt.GTError) as e:
            f()
        assert e.value.status == 1, i  # GT_EINVAL
    # a backward with no forward before it is no longer an error: it recomputes (test_gpu_state_binding)
    plan.bwd(z, z, z, z, lz, z)
    torch.cuda.synchronize()
    plan.close()


def test_cuda_graph_replay_matches_eager(gt):
    """gt_opts.cuda_graphs: captured and replayed steps (two pointer sets, the cache keyed by them)
    give bitwise the eager results and stay within tolerance of the oracle."""
    import torch
    rp, ci = gtgen.random_graph(1500, 20000, seed=71, power=2.2)
    h, d = 4, 64
    q, k, v, dy = inputs(1500, h, d, "bf16", 701)
    scale = 1.0 / math.sqrt(h * d)
    tq, tk, tv, tdy = (to_torch(x) for x in (q, k, v, dy))
    eager = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, heavy_threshold=64)
    y0, l0 = eager.fwd(tq, tk, tv)
    g0 = eager.bwd(tq, tk, tv, y0, l0, tdy)
    s = torch.cuda.Stream()
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, heavy_threshold=64, cuda_graphs=True)
    outs = []
    with torch.cuda.stream(s):
        bufs = [(torch.empty_like(tq), torch.empty((1500, h), dtype=torch.float32, device="cuda")) for _ in range(2)]
        gbufs = [tuple(torch.empty_like(tq) for _ in range(3)) for _ in range(2)]
    for it in range(5):  # eager warm-up, capture set 0, capture set 1, replay 0, replay 1
        y, lse = bufs[it % 2]
        dq, dk, dv = gbufs[it % 2]
        plan.fwd(tq, tk, tv, y, lse, stream=s)
        plan.bwd(tq, tk, tv, y, lse, tdy, dq, dk, dv, stream=s)
        s.synchronize()
        outs.append(tuple(t.clone() for t in (y, lse, dq, dk, dv)))
    torch.cuda.synchronize()
    ref = (y0, l0) + tuple(g0)
    for o in outs:
        for a, b in zip(o, ref):
            assert torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a,
                               b.view(torch.int16) if b.dtype == torch.bfloat16 else b)
    Y, _ = oracle.forward(rp, ci, q, k, v, scale)
    assert normwise(to_f64(outs[-1][0]), Y) <= 2e-2


def test_host_buffer_entry_point_with_graph_replay(gt):
    """gt_attn_fwd_bwd_host on a cuda_graphs plan and a non-default stream: from the third call on the
    backward is replayed from a graph, and the dQ copy must still wait for the replayed row pass
    (ev_dq is an external event node of the graph)."""
    import torch
    rp, ci = gtgen.random_graph(1500, 22000, seed=62, power=2.2)
    h, d = 4, 64
    n = len(rp) - 1
    q, k, v, dy = inputs(n, h, d, "bf16", 602)
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", cuda_graphs=True, heavy_threshold=64)
    pin = lambda x: to_torch(x, "cpu").pin_memory()  # noqa: E731
    tq, tk, tv, tdy = (pin(x) for x in (q, k, v, dy))
    Y, LSE = oracle.forward(rp, ci, q, k, v, plan.scale)
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, plan.scale)
    s = torch.cuda.Stream()
    for it in range(4):
        y, dq, dk, dv = (torch.full_like(tq, float("nan")).pin_memory() for _ in range(4))
        lse = torch.empty((n, h), dtype=torch.float32).pin_memory()
        plan.fwd_bwd_host(tq, tk, tv, tdy, y, lse, dq, dk, dv, stream=s)
        assert normwise(to_f64(y), Y) <= 2e-2 and normwise(to_f64(dq), DQ) <= 2e-2, it
        assert normwise(to_f64(dk), DK) <= 2e-2 and normwise(to_f64(dv), DV) <= 2e-2, it
        check_lse(lse.numpy(), LSE, "bf16")
    plan.close()


@pytest.mark.parametrize("h,d,dtype,heavy", [(4, 64, "bf16", 48), (8, 32, "bf16", 0), (2, 64, "f32", 40),
                                             (8, 16, "f32", 0), (1, 128, "f32", 30)])
def test_column_first_backward_equals_row_first(gt, h, d, dtype, heavy, monkeypatch):
    """World-1 backward in column-first order (default: the column pass computes dP with its own v_j and
    stores dS, the row pass gathers k_j alone) against the row-first order (GT_COLFIRST=0 at plan time):
    the same products summed in the same trees, so dQ, dK, dV are equal bit for bit; both within tolerance
    of the oracle."""
    import torch
    rp, ci = gtgen.random_graph(1500, 16000, seed=71, directed=True, power=2.0)
    n = len(rp) - 1
    q, k, v, dy = inputs(n, h, d, dtype, 72)
    scale = 1.0 / math.sqrt(h * d)
    tq, tk, tv, tdy = (to_torch(x) for x in (q, k, v, dy))
    outs = []
    for order in ("1", "0"):
        monkeypatch.setenv("GT_COLFIRST", order)
        plan = gt.Plan(rp, ci, h, d, dtype=dtype, scale=scale, heavy_threshold=heavy, edge_state=1)
        assert plan.info()["bwd_colfirst"] == (1 if order == "1" and h * (2 if dtype == "bf16" else 4) >= 4 else 0)
        y, lse = plan.fwd(tq, tk, tv)
        dq, dk, dv = plan.bwd(tq, tk, tv, y, lse, tdy)
        torch.cuda.synchronize()
        outs.append([t.clone() for t in (dq, dk, dv)])
        plan.close()
    for name, a, b in zip(("dq", "dk", "dv"), outs[0], outs[1]):
        assert torch.equal(a, b), f"{name}: column-first and row-first orders differ"
    DQ, DK, DV, _ = oracle.backward(rp, ci, q, k, v, dy, scale)
    for name, got, ref in zip(("dq", "dk", "dv"), outs[0], (DQ, DK, DV)):
        e = normwise(to_f64(got), ref)
        assert e <= TOL[dtype], f"{name}: normwise error {e:.3e} > {TOL[dtype]}"
