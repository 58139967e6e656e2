"""Pins for the SGA-block / graph-transformer oracle (oracle/sga.py), checked against things other than
itself (Eq. 3-5, and the backward census P:98):

S1 the whole model written densely in torch fp64 - matmuls for Eq. 3, a masked softmax per head for
   Eq. 4, Eq. 5 with the residual, relu, classifier, cross-entropy - differentiated by autograd
   (independent of the oracle's hand-written chain rule and of its sparse attention backward);
S2 central finite differences of the loss in random parameter directions;
S3 closed form: W_Q = 0 makes every row's attention uniform over its neighbours, so
   X' = X W_o + mean_{j in N(i)} X_j W_V;
S4 the SGD trajectory equals repeated S1 gradient steps.
"""
import math

import numpy as np
import torch

import gtgen
import oracle.sga as osga


def small_problem(n=40, m=150, dim=16, heads=2, classes=5, layers=3, seed=3):
    rp, ci = gtgen.random_graph(n, m, seed=seed, directed=True, power=2.0)
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, dim))
    mk = lambda: rng.standard_normal((dim, dim)) / math.sqrt(dim)  # noqa: E731
    params = {"layers": [{"wq": mk(), "wk": mk(), "wv": mk(), "wo": mk()} for _ in range(layers)],
              "wc": rng.standard_normal((dim, classes)) / math.sqrt(dim)}
    labels = rng.integers(0, classes, n)
    return rp, ci, X, params, labels, heads, 1.0 / math.sqrt(dim)


def dense_model(rp, ci, X, params, labels, heads, scale):
    """S1: the model in dense torch fp64; returns (loss tensor, leaf parameter tensors)."""
    n, dim = X.shape
    mask = torch.zeros(n, n, dtype=torch.bool)
    for i in range(n):
        mask[i, ci[rp[i]:rp[i + 1]]] = True
    nonempty = mask.any(dim=1).view(1, n, 1)
    leaves = {"wc": torch.tensor(params["wc"], requires_grad=True),
              "layers": [{k: torch.tensor(w, requires_grad=True) for k, w in W.items()} for W in params["layers"]]}
    H = torch.tensor(X)
    L = len(params["layers"])
    for li, W in enumerate(leaves["layers"]):
        Q, K, V = H @ W["wq"], H @ W["wk"], H @ W["wv"]
        dh = dim // heads
        Qh, Kh, Vh = (t.view(n, heads, dh) for t in (Q, K, V))
        S = scale * torch.einsum("ihc,jhc->hij", Qh, Kh)
        S = S.masked_fill(~mask.unsqueeze(0), float("-inf"))
        S = torch.where(nonempty, S, torch.zeros_like(S))
        P = torch.where(nonempty, torch.softmax(S, dim=-1), torch.zeros_like(S))
        Y = torch.einsum("hij,jhc->ihc", P, Vh).reshape(n, dim)
        Xp = H @ W["wo"] + Y
        H = torch.relu(Xp) if li < L - 1 else Xp
    logits = H @ leaves["wc"]
    loss = torch.nn.functional.cross_entropy(logits, torch.tensor(labels))
    return loss, leaves


def test_s1_dense_autograd():
    rp, ci, X, params, labels, heads, scale = small_problem()
    loss, g = osga.model_loss_grads(rp, ci, X, params, labels, heads, scale)
    tl, leaves = dense_model(rp, ci, X, params, labels, heads, scale)
    tl.backward()
    assert abs(loss - tl.item()) <= 1e-12 * max(1.0, abs(loss))
    np.testing.assert_allclose(g["wc"], leaves["wc"].grad.numpy(), rtol=0, atol=1e-12)
    for gW, W in zip(g["layers"], leaves["layers"]):
        for k in ("wq", "wk", "wv", "wo"):
            ref = W[k].grad.numpy()
            assert np.max(np.abs(gW[k] - ref)) <= 1e-11 * max(1.0, np.max(np.abs(ref))), k


def test_s1_block_input_gradient():
    """dX of one block against autograd of the dense block (the gradient the next layer down sees)."""
    rp, ci, X, params, labels, heads, scale = small_problem(layers=1)
    W = params["layers"][0]
    Xp, cache = osga.block_forward(rp, ci, X, W, heads, scale)
    G = np.random.default_rng(9).standard_normal(Xp.shape)
    dX, _ = osga.block_backward(rp, ci, W, cache, G, heads, scale)
    n, dim = X.shape
    mask = torch.zeros(n, n, dtype=torch.bool)
    for i in range(n):
        mask[i, ci[rp[i]:rp[i + 1]]] = True
    ne = mask.any(dim=1).view(1, n, 1)
    tX = torch.tensor(X, requires_grad=True)
    Tw = {k: torch.tensor(w) for k, w in W.items()}
    Qh, Kh, Vh = ((tX @ Tw[k]).view(n, heads, dim // heads) for k in ("wq", "wk", "wv"))
    S = torch.where(ne, (scale * torch.einsum("ihc,jhc->hij", Qh, Kh)).masked_fill(~mask.unsqueeze(0), -math.inf), 0.0)
    P = torch.where(ne, torch.softmax(S, dim=-1), 0.0)
    out = tX @ Tw["wo"] + torch.einsum("hij,jhc->ihc", P, Vh).reshape(n, dim)
    np.testing.assert_allclose(Xp, out.detach().numpy(), rtol=0, atol=1e-12)
    (out * torch.tensor(G)).sum().backward()
    np.testing.assert_allclose(dX, tX.grad.numpy(), rtol=0, atol=1e-11)


def test_s2_finite_differences():
    rp, ci, X, params, labels, heads, scale = small_problem(n=24, m=80, dim=8, heads=2, classes=3)
    _, g = osga.model_loss_grads(rp, ci, X, params, labels, heads, scale)
    rng = np.random.default_rng(4)
    eps = 2.0 ** -17
    for li, k in ((0, "wq"), (1, "wk"), (2, "wv"), (0, "wo"), (2, "wo")):
        Dm = rng.standard_normal(params["layers"][li][k].shape)

        def loss_at(t):
            p = {"wc": params["wc"], "layers": [dict(W) for W in params["layers"]]}
            p["layers"][li][k] = params["layers"][li][k] + t * Dm
            return osga.model_loss_grads(rp, ci, X, p, labels, heads, scale)[0]

        fd = (loss_at(eps) - loss_at(-eps)) / (2 * eps)
        an = float(np.sum(g["layers"][li][k] * Dm))
        assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)), (li, k, fd, an)


def test_s3_zero_query_is_neighbour_mean():
    rp, ci, X, params, labels, heads, scale = small_problem(layers=1)
    W = dict(params["layers"][0])
    W["wq"] = np.zeros_like(W["wq"])
    Xp, _ = osga.block_forward(rp, ci, X, W, heads, scale)
    V = X @ W["wv"]
    ref = X @ W["wo"]
    for i in range(len(rp) - 1):
        nb = ci[rp[i]:rp[i + 1]]
        if len(nb):
            ref[i] += V[nb].mean(axis=0)
    np.testing.assert_allclose(Xp, ref, rtol=0, atol=1e-12)


def test_s4_sgd_trajectory_matches_dense_steps():
    rp, ci, X, params, labels, heads, scale = small_problem(n=30, m=100)
    lr = 0.3
    losses, final = osga.sgd_trajectory(rp, ci, X, params, labels, heads, scale, lr, 3)
    p = {"wc": params["wc"].copy(), "layers": [{k: w.copy() for k, w in W.items()} for W in params["layers"]]}
    for step in range(3):
        tl, leaves = dense_model(rp, ci, X, p, labels, heads, scale)
        tl.backward()
        assert abs(tl.item() - losses[step]) <= 1e-12
        p["wc"] = p["wc"] - lr * leaves["wc"].grad.numpy()
        for W, TW in zip(p["layers"], leaves["layers"]):
            for k in W:
                W[k] = W[k] - lr * TW[k].grad.numpy()
    np.testing.assert_allclose(final["wc"], p["wc"], rtol=0, atol=1e-11)
    assert losses[-1] < losses[0]
