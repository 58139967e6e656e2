"""fp8 K/V storage (gt_opts.kv_fp8, reading Z25) against the oracle.

* The quantised table is BYTE work: every e4m3 code and every power-of-two scale of the plan's table
  (GT_EXPORT_KV8) equals oracle/quant.py's quantisation of the same K, V, bit for bit.
* The attention: Y, LSE, dQ, dK, dV of q, dY (bf16) on the dequantised K^, V^ against the fp64 oracle
  (normwise, reading Z8) within the bf16 tolerance 2e-2, on power-law graphs with chunked heavy rows,
  several (heads, d), and peaked logits.
* A backward whose k, v are not the last forward's re-quantises them (fwd(A), fwd(B), bwd(A)).
* Unsupported configurations are GT_ECONFIG before any device work.
* Full size: C3 (products-shaped) with kv_fp8 on the degree-stratified sample.
"""
import math

import numpy as np
import pytest

import gtgen
import oracle
from oracle import quant
from tests._util import TOL, check_lse, inputs, normwise, to_f64, to_torch

pytestmark = pytest.mark.gpu


def f32(x):
    return (x.astype(np.uint32) << 16).view(np.float32) if x.dtype == np.uint16 else x


def reference(rp, ci, q, k, v, dy, scale):
    """The oracle on (q, K^, V^, dY): all fp32 arrays (K^, V^ exactly representable: 3-bit mantissas)."""
    kh, _ = quant.quantize(k)
    vh, _ = quant.quantize(v)
    args = [np.ascontiguousarray(a, np.float32) for a in (f32(q), kh, vh, f32(dy))]
    Y, LSE = oracle.forward(rp, ci, *args[:3], scale)
    DQ, DK, DV, _ = oracle.backward(rp, ci, *args, scale)
    return Y, LSE, DQ, DK, DV


def table_reference(k, v, h):
    """The plan's fp8 table as oracle/quant.py defines it: per row k8 | v8 | 2^ek f32[h] | 2^ev f32[h]."""
    n, _, d = k.shape
    D = h * d
    row = (2 * D + 8 * h + 15) // 16 * 16
    out = np.zeros((n, row), np.uint8)
    import torch
    for j, x in enumerate((k, v)):
        xh, e = quant.quantize(x)
        codes = torch.from_numpy((xh / np.exp2(e)[:, :, None]).astype(np.float32)).to(torch.float8_e4m3fn)
        out[:, j * D:(j + 1) * D] = codes.view(torch.uint8).numpy().reshape(n, D)
        out[:, 2 * D + 4 * h * j:2 * D + 4 * h * (j + 1)] = np.exp2(e).astype(np.float32).view(np.uint8).reshape(n, 4 * h)
    return out


def check_all(got, ref, what=""):
    y, lse, dq, dk, dv = got
    Y, LSE, DQ, DK, DV = ref
    for name, a, r in (("y", y, Y), ("dq", dq, DQ), ("dk", dk, DK), ("dv", dv, DV)):
        e = normwise(a, r)
        assert e <= TOL["bf16"], f"{what} {name}: normwise {e:.3e}"
    check_lse(lse, LSE, "bf16")


@pytest.mark.parametrize("h,d,qk", [(4, 64, 1.0), (8, 32, 1.0), (2, 64, 1.0), (8, 64, 1.0), (1, 128, 1.0),
                                    (4, 64, 6.0)])
def test_fp8_parity_and_table(h, d, qk):
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(3000, 42000, seed=500 + h + d, directed=True, power=2.05)
    n = len(rp) - 1
    q, k, v, dy = inputs(n, h, d, "bf16", 5000 + h, qk_scale=qk)
    # rows of very different magnitudes: scales must follow each (row, head)
    k = (f32(k) * np.exp2(np.random.default_rng(1).integers(-12, 12, (n, h, 1)))).astype(np.float32)
    k = (k.view(np.uint32) >> 16).astype(np.uint16)
    scale = 1.0 / math.sqrt(h * d)
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, heavy_threshold=64, kv_fp8=True)
    info = plan.info()
    assert info["kv_fp8"] == 1 and info["edge_state"] == 1
    tq, tk, tv, tdy = (to_torch(x) for x in (q, k, v, dy))
    y, lse = plan.fwd(tq, tk, tv)
    dq, dk, dv = plan.bwd(tq, tk, tv, y, lse, tdy)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(plan.export("kv8").reshape(n, -1), table_reference(k, v, h))
    check_all([to_f64(t) for t in (y, lse, dq, dk, dv)], reference(rp, ci, q, k, v, dy, scale), f"h{h} d{d}")
    plan.close()


def test_fp8_stale_backward_requantises():
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(2500, 30000, seed=77, directed=True, power=2.1)
    n, h, d = len(rp) - 1, 4, 64
    scale = 1.0 / math.sqrt(h * d)
    A = inputs(n, h, d, "bf16", 71)
    B = inputs(n, h, d, "bf16", 72, qk_scale=3.0)
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, heavy_threshold=64, kv_fp8=True)
    ta, tb = [to_torch(x) for x in A], [to_torch(x) for x in B]
    ya, la = plan.fwd(*ta[:3])
    yb, lb = plan.fwd(*tb[:3])
    ga = plan.bwd(*ta[:3], ya, la, ta[3])      # the table holds B's k, v: re-quantised
    gb = plan.bwd(*tb[:3], yb, lb, tb[3])
    torch.cuda.synchronize()
    check_all([to_f64(t) for t in (ya, la, *ga)], reference(rp, ci, *A, scale), "A")
    check_all([to_f64(t) for t in (yb, lb, *gb)], reference(rp, ci, *B, scale), "B")
    assert plan.info()["stale_bwds"] >= 1
    plan.close()


@pytest.mark.parametrize("case", ["empty", "hub", "zero_rows"])
def test_fp8_degenerate(case):
    """fp8 on graphs without entries, with one hub row / column, and with all-zero K / V rows (scale
    exponent -126, codes 0) next to ordinary ones."""
    import torch
    import paper_2604_16715_b200 as gt
    h, d = 4, 64
    if case == "empty":
        rp, ci = np.zeros(50, np.int64), np.zeros(0, np.int32)
    elif case == "hub":
        n = 500
        rp, ci = gtgen.csr_from_pairs(n, [(0, j) for j in range(1, n)] + [(j, 0) for j in range(1, n)])
    else:
        rp, ci = gtgen.random_graph(800, 9000, seed=81, directed=True, power=2.2)
    n = len(rp) - 1
    q, k, v, dy = inputs(n, h, d, "bf16", 811)
    if case == "zero_rows":
        k[::7] = 0
        v[::5, 1] = 0
    scale = 1.0 / math.sqrt(h * d)
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, heavy_threshold=64, kv_fp8=True)
    tq, tk, tv, tdy = (to_torch(x) for x in (q, k, v, dy))
    y, lse = plan.fwd(tq, tk, tv)
    dq, dk, dv = plan.bwd(tq, tk, tv, y, lse, tdy)
    torch.cuda.synchronize()
    if n:
        np.testing.assert_array_equal(plan.export("kv8").reshape(n, -1), table_reference(k, v, h))
    check_all([to_f64(t) for t in (y, lse, dq, dk, dv)], reference(rp, ci, q, k, v, dy, scale), case)
    plan.close()


def test_fp8_bitwise_deterministic():
    """No atomics in the numerics: two fp8 steps on the same inputs are bitwise identical."""
    import torch
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(2500, 40000, seed=91, directed=True, power=2.0)
    n, h, d = len(rp) - 1, 4, 64
    ins = [to_torch(x) for x in inputs(n, h, d, "bf16", 911)]
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", heavy_threshold=48, kv_fp8=True)
    outs = []
    for _ in range(2):
        y, lse = plan.fwd(*ins[:3])
        g = plan.bwd(*ins[:3], y, lse, ins[3])
        torch.cuda.synchronize()
        outs.append([t.clone() for t in (y, lse, *g)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    plan.close()


def test_fp8_config_errors():
    import paper_2604_16715_b200 as gt
    rp, ci = gtgen.random_graph(300, 2000, seed=5, power=2.3)
    for kw in ({"dtype": "f32"}, {"edge_state": -1}):
        with pytest.raises(gt.GTError) as e:
            gt.Plan(rp, ci, 4, 64, kv_fp8=True, **{"dtype": "bf16", **kw})
        assert e.value.status == 3
    with pytest.raises(gt.GTError) as e:          # heads * d = 64 < 128
        gt.Plan(rp, ci, 2, 32, dtype="bf16", kv_fp8=True)
    assert e.value.status == 3
    grp = gt.LoopbackGroup(2)
    try:
        with pytest.raises(gt.GTError) as e:      # world > 1 (rejected before any collective)
            gt.Plan(rp, ci, 4, 64, dtype="bf16", world=2, rank=0, comm=grp, strategy="halo", kv_fp8=True)
        assert e.value.status == 3
    finally:
        grp.close()


@pytest.mark.slow
def test_fp8_fullsize_c3_sampled():
    import torch
    import paper_2604_16715_b200 as gt
    from tests.test_gpu_fullsize import stratified_ids
    cfg = gtgen.CONFIGS["C3"]
    rp, ci = gtgen.make_graph(cfg.graph)
    n, h, d = len(rp) - 1, cfg.heads, cfg.d
    scale = 1.0 / math.sqrt(h * d)
    feats = {nm: gtgen.features(77, nm, n, h, d, "bf16") for nm in ("q", "k", "v", "dy")}
    plan = gt.Plan(rp, ci, h, d, dtype="bf16", scale=scale, kv_fp8=True)
    dev = {nm: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda() for nm, x in feats.items()}
    y, lse = plan.fwd(dev["q"], dev["k"], dev["v"])
    dq, dk, dv = plan.bwd(dev["q"], dev["k"], dev["v"], y, lse, dev["dy"])
    torch.cuda.synchronize()
    del dev
    rng = np.random.default_rng(5)
    rows = stratified_ids(np.diff(rp), rng)
    cols = stratified_ids(np.bincount(ci, minlength=n), rng)
    kh, _ = quant.quantize(feats["k"])
    vh, _ = quant.quantize(feats["v"])
    ref = oracle.sample(rp, ci, f32(feats["q"]), kh.astype(np.float32), vh.astype(np.float32), f32(feats["dy"]),
                        scale, rows, cols)
    del kh, vh
    ti = lambda idx: torch.from_numpy(idx).cuda()  # noqa: E731
    for name, t, idx in (("y", y, rows), ("dq", dq, rows), ("dk", dk, cols), ("dv", dv, cols)):
        e = normwise(t[ti(idx)].double().cpu().numpy(), ref[name])
        print(f"C3 fp8 {name}: normwise {e:.3e}")
        assert e <= TOL["bf16"], f"{name}: {e}"
    check_lse(lse[ti(rows)].double().cpu().numpy(), ref["lse"], "bf16")
    plan.close()
