"""Shared helpers for the GPU parity tests: seeded inputs (gtgen) and error metrics."""
from __future__ import annotations

import numpy as np

import gtgen


def inputs(n, h, d, dtype, seed, qk_scale=1.0):
    """q, k, v, dy as numpy (fp32 or bf16 bit patterns)."""
    q = gtgen.features(seed, "q", n, h, d, dtype, scale=qk_scale)
    k = gtgen.features(seed, "k", n, h, d, dtype)
    v = gtgen.features(seed, "v", n, h, d, dtype)
    dy = gtgen.features(seed, "dy", n, h, d, dtype)
    return q, k, v, dy


def to_torch(x, device="cuda"):
    import torch
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(x)).to(device)


def to_f64(t):
    import torch
    return t.detach().to(torch.float64).cpu().numpy()


def normwise(x, r):
    """Reading Z8: max_i |x_i - r_i| / max_i |r_i| (0 when both are identically 0)."""
    x = np.asarray(x, np.float64)
    r = np.asarray(r, np.float64)
    den = np.max(np.abs(r)) if r.size else 0.0
    num = np.max(np.abs(x - r)) if r.size else 0.0
    if den == 0.0:
        return num
    return num / den


def elementwise(x, r, floor=1e-3):
    """Reading Z8's diagnostic: max |x - r| / |r| over entries with |r| >= floor * max|r|."""
    x = np.asarray(x, np.float64).ravel()
    r = np.asarray(r, np.float64).ravel()
    if r.size == 0 or np.max(np.abs(r)) == 0.0:
        return 0.0
    m = np.abs(r) >= floor * np.max(np.abs(r))
    return float(np.max(np.abs(x[m] - r[m]) / np.abs(r[m])))


TOL = {"f32": 1e-4, "bf16": 2e-2}
LSE_TOL = {"f32": 1e-4, "bf16": 1e-2}


def check_lse(lse_gpu, lse_ref, dtype):
    lse_gpu = np.asarray(lse_gpu, np.float64)
    inf_r = np.isneginf(lse_ref)
    assert np.array_equal(np.isneginf(lse_gpu), inf_r), "empty-row LSE must be exactly -inf"
    if (~inf_r).any():
        err = np.max(np.abs(lse_gpu[~inf_r] - lse_ref[~inf_r]))
        assert err <= LSE_TOL[dtype], f"LSE abs err {err}"
