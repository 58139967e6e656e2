"""Sparse graph transformer around the libgt attention core.

PAPER.md Section 2.1: one SGA block is
  Eq. 3  Q = X W_Q, K = X W_K, V = X W_V
  Eq. 4  U = Softmax((Q K^T) (.) A  scale)           -> libgt (gt_attn_fwd)
  Eq. 5  Y = U V, X' = X W_o + Y
and the model the paper trains is "a 3-layer Graph Transformer" (hidden 128, 8 heads):
H_{l+1} = relu(SGA_l(H_l)) (no relu after the last block), logits = H_L W_c, mean cross-entropy
(reading Z23).  The dense products run in PyTorch (cuBLAS GEMMs, the compute dtype of the
plan: bf16 with fp32 accumulation, or fp32); every sparse operation - the SDDMM, softmax and SpMM of the
forward and the SDDMM + 3 SpMM of the backward - runs in libgt.  All layers share one plan (one
graph); each backward is bound to the forward of its layer by libgt.

Forward and backward are written out (the chain rule of Eq. 3-5; dX = dX' W_o^T + dQ W_Q^T + dK W_K^T
+ dV W_V^T, dW_* = X^T d*) rather than left to torch.autograd: a multi-rank step issues collective
libgt calls in the same order on every rank, and the autograd engine runs the backward of all host
threads of one device on a single worker thread, which would serialise the in-process loopback ranks.

Data parallelism over graph rows (Alg. 1): rank r holds rows [row_lo, row_hi) of X, the
labels and every activation; the weights are replicated; the attention exchange is libgt's; weight
gradients and the loss are summed over ranks by the caller's `allreduce` (torch.distributed over NCCL,
or the loopback helper of the tests) before the SGD update.
"""
from __future__ import annotations

import math

import torch

from .gt import Plan

KEYS = ("wq", "wk", "wv", "wo")


class GraphTransformer:
    """L SGA blocks + a linear classifier; parameters fp32 on the plan's device."""

    def __init__(self, params: dict, heads: int, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        conv = lambda w: torch.as_tensor(w, dtype=torch.float32).to(dev).contiguous()  # noqa: E731
        self.layers = [{k: conv(W[k]) for k in KEYS} for W in params["layers"]]
        self.wc = conv(params["wc"])
        self.heads = heads
        self.dim = self.wc.shape[0]
        if self.dim % heads:
            raise ValueError("dim must be a multiple of heads")

    @classmethod
    def init(cls, dim: int, heads: int, layers: int, classes: int, seed: int = 0, device=None):
        g = torch.Generator().manual_seed(seed)
        mk = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64) / math.sqrt(dim)  # noqa: E731
        params = {"layers": [{k: mk(dim, dim) for k in KEYS} for _ in range(layers)], "wc": mk(dim, classes)}
        return cls(params, heads, device)

    def parameters(self):
        return [w for W in self.layers for w in (W[k] for k in KEYS)] + [self.wc]

    # -- forward / backward of one block --
    def _block_fwd(self, plan: Plan, W, X):
        cd = plan._torch_dtype()
        n = X.shape[0]
        h, dh = self.heads, self.dim // self.heads
        Xc = X.to(cd)
        Q, K, V = (Xc @ W[k].to(cd) for k in ("wq", "wk", "wv"))           # Eq. 3 (cuBLAS)
        Qh, Kh, Vh = (t.view(n, h, dh) for t in (Q, K, V))
        Y, lse = plan.fwd(Qh, Kh, Vh)                                         # Eq. 4-5: Y = U V (libgt)
        Xp = Xc @ W["wo"].to(cd) + Y.view(n, self.dim)                        # Eq. 5: X' = X W_o + Y
        return Xp, (Xc, Qh, Kh, Vh, Y, lse)

    def _block_bwd(self, plan: Plan, W, cache, dXp):
        Xc, Qh, Kh, Vh, Y, lse = cache
        cd = Xc.dtype
        n = Xc.shape[0]
        dXp = dXp.to(cd).contiguous()
        dQ, dK, dV = plan.bwd(Qh, Kh, Vh, Y, lse, dXp.view(n, self.heads, -1))  # P:98 (libgt)
        dQ, dK, dV = (t.view(n, self.dim) for t in (dQ, dK, dV))
        Xf = Xc.float()
        g = {"wo": Xf.T @ dXp.float(), "wq": Xf.T @ dQ.float(), "wk": Xf.T @ dK.float(), "wv": Xf.T @ dV.float()}
        dX = dXp @ W["wo"].to(cd).T + dQ @ W["wq"].to(cd).T + dK @ W["wk"].to(cd).T + dV @ W["wv"].to(cd).T
        return dX, g

    def forward(self, plan: Plan, X):
        """Logits (fp32) of this rank's rows and the activations the backward needs."""
        H, caches, pre = X, [], []
        L = len(self.layers)
        for li, W in enumerate(self.layers):
            Xp, c = self._block_fwd(plan, W, H)
            caches.append(c)
            pre.append(Xp)
            H = torch.relu(Xp) if li < L - 1 else Xp
        logits = H.float() @ self.wc
        return logits, (H, caches, pre)

    def loss_and_grads(self, plan: Plan, X, labels, n_total: int):
        """Sum over this rank's rows of the cross-entropy / n_total (so that the sum over ranks is the
        mean over all nodes) and its gradients w.r.t. every parameter (this rank's contribution)."""
        logits, (H, caches, pre) = self.forward(plan, X)
        loss = torch.nn.functional.cross_entropy(logits, labels, reduction="sum") / n_total
        dlogits = torch.softmax(logits, dim=1)
        dlogits[torch.arange(len(labels), device=labels.device), labels] -= 1.0
        dlogits /= n_total
        grads = {"wc": H.float().T @ dlogits, "layers": [None] * len(self.layers)}
        dH = dlogits @ self.wc.T
        for li in range(len(self.layers) - 1, -1, -1):   # last layer first: its forward state is the plan's
            dXp = dH * (pre[li] > 0) if li < len(self.layers) - 1 else dH
            dH, grads["layers"][li] = self._block_bwd(plan, self.layers[li], caches[li], dXp)
        return loss, grads

    def sgd_step(self, plan: Plan, X, labels, n_total: int, lr: float, allreduce=None) -> float:
        """One training step; `allreduce(list_of_tensors)` sums in place over ranks (None at world 1).
        Returns the loss over all nodes (before the update)."""
        loss, g = self.loss_and_grads(plan, X, labels, n_total)
        flat = [g["wc"]] + [gW[k] for gW in g["layers"] for k in KEYS] + [loss.reshape(1)]
        if allreduce is not None:
            allreduce(flat)
        with torch.no_grad():
            self.wc -= lr * flat[0]
            i = 1
            for W in self.layers:
                for k in KEYS:
                    W[k] -= lr * flat[i]
                    i += 1
        return float(flat[-1].item())


def nccl_allreduce(tensors):
    """Sum over the default torch.distributed group (one process per GPU)."""
    import torch.distributed as dist
    for t in tensors:
        dist.all_reduce(t)
