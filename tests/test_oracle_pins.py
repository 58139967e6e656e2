"""Pins for the CPU fp64 oracle (oracle/): it is checked against things other than itself.

P1 textbook special case: dense masked softmax attention in torch fp64 (Eq. 4-5),
   backward by torch autograd of the dense graph (independent of the oracle's hand backward).
P2 worked examples: tests/golden/spec_worked_examples.json (cited per case).
P3 closed forms: Q=0 -> neighbour mean and LSE = ln deg; complete graph = unmasked SDPA; scale invariance.
P4 invariants: sum_e U_e = 1, sum_e dZ_e = 0 (dQ invariant to K + c), sum_j dV_j = sum_{deg>0} dY_i,
   D_i = <dY_i, Y_i>, empty rows / zero in-degree columns, linearity, relabel equivariance.
P5 central finite differences, eps = 1e-5, loss L = <dY, Y>.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import gtgen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")


def rand_inputs(n, h, d, seed, dtype="f32"):
    q = gtgen.features(seed, "q", n, h, d, dtype)
    k = gtgen.features(seed, "k", n, h, d, dtype)
    v = gtgen.features(seed, "v", n, h, d, dtype)
    dy = gtgen.features(seed, "dy", n, h, d, dtype)
    return q, k, v, dy


def as64(x):
    return gtgen.bf16_bits_to_f32(x).astype(np.float64) if x.dtype == np.uint16 else x.astype(np.float64)


def dense_reference(row_ptr, col_idx, q, k, v, dy, scale):
    """Dense masked softmax attention per head in torch fp64 + autograd (P1)."""
    n, h, d = q.shape
    mask = torch.zeros(n, n, dtype=torch.bool)
    for i in range(n):
        for e in range(row_ptr[i], row_ptr[i + 1]):
            mask[i, col_idx[e]] = True
    Q = torch.tensor(as64(q), requires_grad=True)
    K = torch.tensor(as64(k), requires_grad=True)
    V = torch.tensor(as64(v), requires_grad=True)
    S = scale * torch.einsum("ihc,jhc->hij", Q, K)
    S = S.masked_fill(~mask.unsqueeze(0), float("-inf"))
    nonempty = mask.any(dim=1)
    S = torch.where(nonempty.view(1, n, 1), S, torch.zeros_like(S))
    Pm = torch.softmax(S, dim=-1)
    Pm = torch.where(nonempty.view(1, n, 1), Pm, torch.zeros_like(Pm))
    Y = torch.einsum("hij,jhc->ihc", Pm, V)
    lse = torch.logsumexp(S, dim=-1).T  # [n, h]
    lse = torch.where(nonempty.view(n, 1), lse, torch.full_like(lse, float("-inf")))
    L = (Y * torch.tensor(as64(dy))).sum()
    L.backward()
    return (Y.detach().numpy(), lse.detach().numpy(), Q.grad.numpy(), K.grad.numpy(), V.grad.numpy())


CASES = [  # n, m, h, d, seed, directed, scale_kind
    (1, 0, 1, 4, 11, True, "hd"),
    (7, 12, 1, 4, 12, True, "hd"),
    (16, 40, 2, 8, 13, True, "d"),
    (33, 120, 4, 16, 14, False, "hd"),
    (64, 300, 4, 8, 15, True, "x8"),
    (64, 900, 2, 16, 16, True, "hd"),
    (40, 0, 2, 4, 17, True, "hd"),
]


def pick_scale(kind, h, d):
    if kind == "hd":
        return 1.0 / math.sqrt(h * d)
    if kind == "d":
        return 1.0 / math.sqrt(d)
    return 8.0 / math.sqrt(h * d)


@pytest.mark.parametrize("n,m,h,d,seed,directed,sk", CASES)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_p1_dense_bruteforce(n, m, h, d, seed, directed, sk, dtype):
    row_ptr, col_idx = gtgen.random_graph(n, m, seed, directed=directed) if m else (
        np.zeros(n + 1, np.int64), np.zeros(0, np.int32))
    q, k, v, dy = rand_inputs(n, h, d, seed, dtype)
    scale = pick_scale(sk, h, d)
    y, lse = oracle.forward(row_ptr, col_idx, q, k, v, scale)
    dq, dk, dv, dstat = oracle.backward(row_ptr, col_idx, q, k, v, dy, scale)
    Y, LSE, DQ, DK, DV = dense_reference(row_ptr, col_idx, q, k, v, dy, scale)
    np.testing.assert_allclose(y, Y, rtol=0, atol=1e-12)
    fin = np.isfinite(LSE)
    assert np.array_equal(fin, np.isfinite(lse))
    assert np.all(np.isneginf(lse[~fin]))
    np.testing.assert_allclose(lse[fin], LSE[fin], rtol=0, atol=1e-12)
    np.testing.assert_allclose(dq, DQ, rtol=0, atol=1e-12)
    np.testing.assert_allclose(dk, DK, rtol=0, atol=1e-12)
    np.testing.assert_allclose(dv, DV, rtol=0, atol=1e-12)


def test_p1_sdpa_nonempty_rows():
    """torch's own scaled_dot_product_attention with a boolean mask, on rows with >= 1 edge."""
    n, h, d, seed = 48, 2, 8, 21
    row_ptr, col_idx = gtgen.random_graph(n, 200, seed)
    q, k, v, _ = rand_inputs(n, h, d, seed)
    scale = 0.3
    y, _ = oracle.forward(row_ptr, col_idx, q, k, v, scale)
    mask = torch.zeros(n, n, dtype=torch.bool)
    for i in range(n):
        mask[i, col_idx[row_ptr[i]:row_ptr[i + 1]]] = True
    ne = mask.any(1)
    Q = torch.tensor(as64(q)).permute(1, 0, 2)
    K = torch.tensor(as64(k)).permute(1, 0, 2)
    V = torch.tensor(as64(v)).permute(1, 0, 2)
    Ys = torch.nn.functional.scaled_dot_product_attention(Q[:, ne], K, V, attn_mask=mask[ne], scale=scale)
    np.testing.assert_allclose(y[ne.numpy()], Ys.permute(1, 0, 2).numpy(), rtol=0, atol=1e-12)


def _load_golden():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _load_golden(), ids=lambda c: c["id"])
def test_p2_worked_examples(case):
    row_ptr, col_idx = gtgen.csr_from_pairs(case["n"], case["pairs"])
    q = np.array(case["q"], np.float32)
    k = np.array(case["k"], np.float32)
    v = np.array(case["v"], np.float32)
    y, lse = oracle.forward(row_ptr, col_idx, q, k, v, case["scale"])
    for i, val in case.get("expect_y", {}).items():
        np.testing.assert_allclose(y[int(i)], np.array(val, np.float64), rtol=1e-15, atol=1e-15)
    for i, val in case.get("expect_lse", {}).items():
        exp = np.array([float(x) for x in val])
        got = lse[int(i)]
        if np.isneginf(exp).any():
            assert np.array_equal(np.isneginf(got), np.isneginf(exp))
        else:
            np.testing.assert_allclose(got, exp, rtol=1e-15, atol=1e-12)
    assert np.all(np.isfinite(y))


def test_p3_q_zero_is_neighbour_mean():
    n, h, d, seed = 50, 4, 8, 31
    row_ptr, col_idx = gtgen.random_graph(n, 160, seed)
    _, k, v, _ = rand_inputs(n, h, d, seed)
    q = np.zeros((n, h, d), np.float32)
    y, lse = oracle.forward(row_ptr, col_idx, q, k, v, 0.7)
    for i in range(n):
        cols = col_idx[row_ptr[i]:row_ptr[i + 1]]
        if len(cols) == 0:
            assert np.all(y[i] == 0) and np.all(np.isneginf(lse[i]))
            continue
        np.testing.assert_allclose(y[i], v[cols].astype(np.float64).mean(0), atol=1e-13)
        np.testing.assert_allclose(lse[i], math.log(len(cols)), atol=1e-13)


def test_p3_complete_graph_is_unmasked_attention():
    n, h, d, seed = 24, 2, 8, 32
    pairs = [(i, j) for i in range(n) for j in range(n)]
    row_ptr, col_idx = gtgen.csr_from_pairs(n, pairs)
    q, k, v, _ = rand_inputs(n, h, d, seed)
    y, _ = oracle.forward(row_ptr, col_idx, q, k, v, 0.25)
    Q, K, V = (torch.tensor(as64(x)).permute(1, 0, 2) for x in (q, k, v))
    Ys = torch.nn.functional.scaled_dot_product_attention(Q, K, V, scale=0.25).permute(1, 0, 2)
    np.testing.assert_allclose(y, Ys.numpy(), atol=1e-12)


def test_p3_scale_invariance_and_single_edge():
    n, h, d, seed = 30, 2, 4, 33
    row_ptr, col_idx = gtgen.random_graph(n, 70, seed)
    q, k, v, dy = rand_inputs(n, h, d, seed)
    y1, _ = oracle.forward(row_ptr, col_idx, q, k, v, 0.5)
    y2, _ = oracle.forward(row_ptr, col_idx, (q * 4).astype(np.float32), k, v, 0.125)
    np.testing.assert_allclose(y1, y2, atol=1e-12)
    # single-edge rows: Y_i = v_j, dQ_i = 0, and that edge's dK contribution is 0
    deg = np.diff(row_ptr)
    dq, dk, dv, _ = oracle.backward(row_ptr, col_idx, q, k, v, dy, 0.5)
    for i in np.nonzero(deg == 1)[0]:
        j = col_idx[row_ptr[i]]
        np.testing.assert_allclose(y1[i], v[j], atol=1e-13)
        np.testing.assert_allclose(dq[i], 0, atol=1e-13)


def test_p4_invariants():
    n, h, d, seed = 60, 4, 8, 41
    row_ptr, col_idx = gtgen.random_graph(n, 240, seed, power=2.3)
    q, k, v, dy = rand_inputs(n, h, d, seed)
    scale = 0.35
    deg = np.diff(row_ptr)
    indeg = np.bincount(col_idx, minlength=n)
    ones = np.ones_like(v)
    y1, _ = oracle.forward(row_ptr, col_idx, q, k, ones, scale)
    np.testing.assert_allclose(y1[deg > 0], 1.0, atol=1e-13)          # sum_e U_e = 1
    assert np.all(y1[deg == 0] == 0)
    y, lse = oracle.forward(row_ptr, col_idx, q, k, v, scale)
    dq, dk, dv, dstat = oracle.backward(row_ptr, col_idx, q, k, v, dy, scale)
    # D_i = <dY_i, Y_i>
    np.testing.assert_allclose(dstat, np.einsum("ihc,ihc->ih", dy.astype(np.float64), y), atol=1e-12)
    # sum_e dZ_e = 0  <=>  dQ unchanged when every k_j is shifted by the same vector c
    # k from bf16-representable values plus dyadic c keeps k + c exact in fp32
    kb = gtgen.bf16_bits_to_f32(gtgen.f32_to_bf16_bits(k))
    c = np.random.default_rng(0).choice([-1.0, -0.5, 0.25, 0.5, 1.0], size=(1, h, d)).astype(np.float32)
    k2 = (kb + c).astype(np.float32)
    assert np.array_equal(k2.astype(np.float64) - kb.astype(np.float64), np.broadcast_to(c, k2.shape))
    dq, _, _, _ = oracle.backward(row_ptr, col_idx, q, kb, v, dy, scale)
    dq2, _, _, _ = oracle.backward(row_ptr, col_idx, q, k2, v, dy, scale)
    np.testing.assert_allclose(dq2, dq, atol=1e-11)
    dq, dk, dv, dstat = oracle.backward(row_ptr, col_idx, q, k, v, dy, scale)
    # sum_j dV_j = sum_{i: deg>0} dY_i
    np.testing.assert_allclose(dv.sum(0), dy[deg > 0].astype(np.float64).sum(0), atol=1e-11)
    # empty rows and zero in-degree columns
    assert np.all(dq[deg == 0] == 0) and np.all(np.isneginf(lse[deg == 0]))
    assert np.all(dk[indeg == 0] == 0) and np.all(dv[indeg == 0] == 0)
    # linearity in V (forward) and in dY (backward)
    y3, _ = oracle.forward(row_ptr, col_idx, q, k, (2 * v).astype(np.float32), scale)
    np.testing.assert_allclose(y3, 2 * y, atol=1e-12)
    dqb, dkb, dvb, _ = oracle.backward(row_ptr, col_idx, q, k, v, (4 * dy).astype(np.float32), scale)
    np.testing.assert_allclose(dqb, 4 * dq, atol=1e-11)
    np.testing.assert_allclose(dkb, 4 * dk, atol=1e-11)
    np.testing.assert_allclose(dvb, 4 * dv, atol=1e-11)


def test_p4_relabel_equivariance():
    n, h, d, seed = 40, 2, 4, 42
    row_ptr, col_idx = gtgen.random_graph(n, 150, seed)
    q, k, v, dy = rand_inputs(n, h, d, seed)
    perm = np.random.default_rng(1).permutation(n)  # new id of old node i is perm[i]
    pairs = [(perm[i], perm[col_idx[e]]) for i in range(n) for e in range(row_ptr[i], row_ptr[i + 1])]
    rp2, ci2 = gtgen.csr_from_pairs(n, pairs)
    inv = np.argsort(perm)
    q2, k2, v2, dy2 = q[inv], k[inv], v[inv], dy[inv]
    y, _ = oracle.forward(row_ptr, col_idx, q, k, v, 0.4)
    y2, _ = oracle.forward(rp2, ci2, q2, k2, v2, 0.4)
    np.testing.assert_allclose(y2[perm], y, atol=1e-12)
    g = oracle.backward(row_ptr, col_idx, q, k, v, dy, 0.4)
    g2 = oracle.backward(rp2, ci2, q2, k2, v2, dy2, 0.4)
    for a, b in zip(g[:3], g2[:3]):
        np.testing.assert_allclose(b[perm], a, atol=1e-11)


@pytest.mark.parametrize("seed", [51, 52, 53])
def test_p5_finite_differences(seed):
    n, h, d = 10, 2, 3
    row_ptr, col_idx = gtgen.random_graph(n, 30, seed)
    q, k, v, dy = rand_inputs(n, h, d, seed)
    # The oracle reads fp32 inputs, so the step is a power of two (~1e-5) that is added exactly
    # to the fp32 input; the assert below checks the perturbed input moved by exactly +/- eps.
    scale = 0.45
    dq, dk, dv, _ = oracle.backward(row_ptr, col_idx, q, k, v, dy, scale)
    eps = 2.0 ** -17  # ~7.6e-6, exactly representable offsets on inputs of magnitude < 4
    rng = np.random.default_rng(seed)
    grads = {"q": dq, "k": dk, "v": dv}
    for name in ("q", "k", "v"):
        for _ in range(12):
            idx = tuple(rng.integers(0, s) for s in q.shape)
            base = {"q": q.copy(), "k": k.copy(), "v": v.copy()}
            vals = []
            for sgn in (+1, -1):
                x = {kk: vv.copy() for kk, vv in base.items()}
                x[name][idx] = np.float32(np.float64(x[name][idx]) + sgn * eps)
                assert np.float64(x[name][idx]) - np.float64(base[name][idx]) == sgn * eps
                y, _ = oracle.forward(row_ptr, col_idx, x["q"], x["k"], x["v"], scale)
                vals.append(float((y * dy.astype(np.float64)).sum()))
            fd = (vals[0] - vals[1]) / (2 * eps)
            an = grads[name][idx]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (name, idx, fd, an)


def test_bf16_decode_matches_f32():
    n, h, d, seed = 20, 2, 8, 61
    row_ptr, col_idx = gtgen.random_graph(n, 60, seed)
    qb, kb, vb, dyb = rand_inputs(n, h, d, seed, "bf16")
    q, k, v, dy = (gtgen.bf16_bits_to_f32(x) for x in (qb, kb, vb, dyb))
    a = oracle.forward(row_ptr, col_idx, qb, kb, vb, 0.3)
    b = oracle.forward(row_ptr, col_idx, q, k, v, 0.3)
    np.testing.assert_array_equal(a[0], b[0])
    assert gtgen.f32_to_bf16_bits(np.array([1.0, -2.0], np.float32)).tolist() == [0x3F80, 0xC000]
    # round-to-nearest-even tie: 1 + 2^-8 is halfway between bf16 neighbours 1 and 1 + 2^-7 -> even (1.0)
    assert gtgen.f32_to_bf16_bits(np.array([1.0 + 2.0 ** -8], np.float32)).tolist() == [0x3F80]
    assert gtgen.f32_to_bf16_bits(np.array([1.0 + 3 * 2.0 ** -8], np.float32)).tolist() == [0x3F82]


def test_sampled_oracle_matches_full():
    n, h, d, seed = 300, 4, 8, 71
    row_ptr, col_idx = gtgen.random_graph(n, 2500, seed, power=2.2)
    q, k, v, dy = rand_inputs(n, h, d, seed)
    y, lse = oracle.forward(row_ptr, col_idx, q, k, v, 0.3)
    dq, dk, dv, ds = oracle.backward(row_ptr, col_idx, q, k, v, dy, 0.3)
    rows = np.array([0, 5, 17, 299, 150])
    cols = np.array([3, 0, 299, 77])
    s = oracle.sample(row_ptr, col_idx, q, k, v, dy, 0.3, rows, cols)
    np.testing.assert_allclose(s["y"], y[rows], atol=1e-13)
    np.testing.assert_allclose(s["lse"], lse[rows], atol=1e-13)
    np.testing.assert_allclose(s["dq"], dq[rows], atol=1e-13)
    np.testing.assert_allclose(s["dstat"], ds[rows], atol=1e-13)
    np.testing.assert_allclose(s["dk"], dk[cols], atol=1e-12)
    np.testing.assert_allclose(s["dv"], dv[cols], atol=1e-12)


def test_oracle_transpose_vs_scipy():
    import scipy.sparse as sp
    n = 200
    row_ptr, col_idx = gtgen.random_graph(n, 1500, 81, power=2.2)
    col_ptr, row_idx = oracle.transpose(row_ptr, col_idx)
    A = sp.csr_matrix((np.ones(len(col_idx)), col_idx, row_ptr), shape=(n, n))
    T = A.T.tocsr()
    T.sort_indices()
    np.testing.assert_array_equal(col_ptr, T.indptr)
    np.testing.assert_array_equal(row_idx, T.indices)
    # involution
    rp2, ci2 = oracle.transpose(col_ptr, row_idx)
    np.testing.assert_array_equal(rp2, row_ptr)
    np.testing.assert_array_equal(ci2, col_idx)


def sparse_library_reference(row_ptr, col_idx, q, k, v, dy, scale):
    """P1 at scale: the same attention written with torch.sparse library ops in fp64 and
    differentiated by torch autograd — a COO pattern per head, torch.sparse.softmax over each row's
    stored entries, torch.sparse.mm with V; SDDMM as an explicit gather-dot.  Empty rows give
    Y = 0 and no gradient contribution.  Shares nothing with the oracle's hand-written C."""
    n, h, d = q.shape
    rows = torch.repeat_interleave(torch.arange(n), torch.tensor(np.diff(row_ptr)))
    cols = torch.tensor(col_idx.astype(np.int64))
    Q = torch.tensor(as64(q), requires_grad=True)
    K = torch.tensor(as64(k), requires_grad=True)
    V = torch.tensor(as64(v), requires_grad=True)
    Ys = []
    for t in range(h):
        s = scale * (Q[rows, t, :] * K[cols, t, :]).sum(-1)                     # SDDMM on the pattern
        S = torch.sparse_coo_tensor(torch.stack([rows, cols]), s, (n, n)).coalesce()
        U = torch.sparse.softmax(S, dim=1)                                       # edge softmax per row
        Ys.append(torch.sparse.mm(U, V[:, t, :]))                                # SpMM
    Y = torch.stack(Ys, dim=1)
    (Y * torch.tensor(as64(dy))).sum().backward()
    return Y.detach().numpy(), Q.grad.numpy(), K.grad.numpy(), V.grad.numpy()


@pytest.mark.parametrize("n,m,h,d,power,seed,dtype", [
    (1500, 24000, 2, 8, 2.05, 31, "f32"),    # power law: hub rows / columns of several hundred entries
    (2000, 16000, 1, 16, 0.0, 32, "bf16"),   # uniform degrees, bf16 inputs
    (900, 30000, 4, 4, 2.3, 33, "f32"),      # dense rows
])
def test_p1_sparse_library_at_scale(n, m, h, d, power, seed, dtype):
    row_ptr, col_idx = gtgen.random_graph(n, m, seed, directed=True, power=power)
    q, k, v, dy = rand_inputs(n, h, d, seed, dtype)
    scale = 1.0 / math.sqrt(h * d)
    y, _ = oracle.forward(row_ptr, col_idx, q, k, v, scale)
    dq, dk, dv, _ = oracle.backward(row_ptr, col_idx, q, k, v, dy, scale)
    Y, DQ, DK, DV = sparse_library_reference(row_ptr, col_idx, q, k, v, dy, scale)
    if power:
        assert np.diff(row_ptr).max() > 50  # heavy rows exercised
    for got, ref in ((y, Y), (dq, DQ), (dk, DK), (dv, DV)):
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-11 * max(1.0, np.abs(ref).max()))
