"""fp64 oracle of the sparse graph transformer around the attention core.

TEST INFRASTRUCTURE ONLY (same rule as ``oracle/__init__.py``): only ``tests/`` may import it.  It
shares no code with ``paper_2604_16715_b200``; the attention itself is ``oracle.forward`` /
``oracle.backward`` (plain fp64 C, pinned in tests/test_oracle_pins.py), fed fp64 Q, K, V.

What it computes, in the paper's notation (Section 2.1):
  Eq. 3  Q = X W_Q,  K = X W_K,  V = X W_V                (W: d x d)
  Eq. 4  Z = (Q K^T) (.) A,  U = Softmax(Z scale)        (per head, over row i's entries)
  Eq. 5  Y = U V,  X' = X W_o + Y                        (the SGA block)
  Multi-head: the d columns of Q, K, V are h heads of d' = d / h consecutive columns.
Backward (P:98 for the attention; the dense products by the chain rule):
  dY = dX';  (dQ, dK, dV) = attention backward;  dW_o = X^T dX';  dW_Q = X^T dQ;  dW_K = X^T dK;
  dW_V = X^T dV;  dX = dX' W_o^T + dQ W_Q^T + dK W_K^T + dV W_V^T.
The model (reading Z23 in DESIGN.md; the paper trains "a 3-layer Graph Transformer", hidden
128, 8 heads, without further detail): H_0 = X, H_{l+1} = relu(SGA_l(H_l)) for l < L - 1,
H_L = SGA_{L-1}(H_{L-1}); logits = H_L W_c; loss = mean over nodes of the softmax cross-entropy
with integer labels; plain SGD W <- W - lr dW.

Pins: tests/test_oracle_sga.py (dense masked attention + matmuls in torch fp64 differentiated by
autograd, central finite differences, the W_Q = 0 closed form).
"""
from __future__ import annotations

import numpy as np

import oracle


def _heads(x, h):
    n, dim = x.shape
    return np.ascontiguousarray(x.reshape(n, h, dim // h))


def block_forward(row_ptr, col_idx, X, W, heads: int, scale: float):
    """One SGA block (Eq. 3-5).  W = {"wq", "wk", "wv", "wo"} (d x d fp64).  Returns X' and a cache."""
    X = np.asarray(X, np.float64)
    Q, K, V = X @ W["wq"], X @ W["wk"], X @ W["wv"]                       # Eq. 3
    Yh, lse = oracle.forward(row_ptr, col_idx, _heads(Q, heads), _heads(K, heads), _heads(V, heads), scale)
    Y = Yh.reshape(X.shape)                                                # Eq. 4-5: Y = U V
    Xp = X @ W["wo"] + Y                                                   # Eq. 5: X' = X W_o + Y
    return Xp, {"X": X, "Q": Q, "K": K, "V": V, "Y": Y, "lse": lse}


def block_backward(row_ptr, col_idx, W, cache, dXp, heads: int, scale: float):
    """Gradients of <dX', X'> w.r.t. X and the four weights of the block."""
    X, Q, K, V = cache["X"], cache["Q"], cache["K"], cache["V"]
    dXp = np.asarray(dXp, np.float64)
    dQh, dKh, dVh, _ = oracle.backward(row_ptr, col_idx, _heads(Q, heads), _heads(K, heads), _heads(V, heads),
                                       _heads(dXp, heads), scale)          # dY = dX'
    dQ, dK, dV = (t.reshape(X.shape) for t in (dQh, dKh, dVh))
    g = {"wo": X.T @ dXp, "wq": X.T @ dQ, "wk": X.T @ dK, "wv": X.T @ dV}
    dX = dXp @ W["wo"].T + dQ @ W["wq"].T + dK @ W["wk"].T + dV @ W["wv"].T
    return dX, g


def model_loss_grads(row_ptr, col_idx, X, params, labels, heads: int, scale: float):
    """Loss (mean cross-entropy) and gradients of every parameter of the L-layer model."""
    layers = params["layers"]
    L = len(layers)
    H = np.asarray(X, np.float64)
    caches, pre = [], []
    for li, W in enumerate(layers):
        Xp, c = block_forward(row_ptr, col_idx, H, W, heads, scale)
        caches.append(c)
        pre.append(Xp)
        H = np.maximum(Xp, 0.0) if li < L - 1 else Xp
    logits = H @ params["wc"]
    n = logits.shape[0]
    z = logits - logits.max(axis=1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    loss = -logp[np.arange(n), labels].mean()
    dlogits = np.exp(logp)
    dlogits[np.arange(n), labels] -= 1.0
    dlogits /= n
    grads = {"wc": H.T @ dlogits, "layers": [None] * L}
    dH = dlogits @ params["wc"].T
    for li in range(L - 1, -1, -1):
        dXp = dH * (pre[li] > 0) if li < L - 1 else dH
        dH, grads["layers"][li] = block_backward(row_ptr, col_idx, layers[li], caches[li], dXp, heads, scale)
    return float(loss), grads


def sgd_trajectory(row_ptr, col_idx, X, params, labels, heads: int, scale: float, lr: float, steps: int):
    """Losses of `steps` plain SGD steps (loss before each update) and the final parameters."""
    p = {"wc": params["wc"].copy(), "layers": [{k: w.copy() for k, w in W.items()} for W in params["layers"]]}
    losses = []
    for _ in range(steps):
        loss, g = model_loss_grads(row_ptr, col_idx, X, p, labels, heads, scale)
        losses.append(loss)
        p["wc"] -= lr * g["wc"]
        for W, gW in zip(p["layers"], g["layers"]):
            for k in W:
                W[k] -= lr * gW[k]
    return losses, p
