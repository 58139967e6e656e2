"""fp8 (e4m3) K/V quantiser of the NEXT-4 fp8 storage option (gt_opts.kv_fp8; reading Z25).

TEST INFRASTRUCTURE ONLY (same rule as ``oracle/__init__.py``).  It shares no code with the CUDA path.

Per row i and head t of K (and of V), with x the head's d values (fp32 of the stored bf16 bits):
  e      = the smallest integer with max_c |x_c| <= 448 * 2^e   (448 = largest finite e4m3 value;
           max |x| = 0 gives e = -126), clamped to [-126, 126]
  x8_c   = RNE_e4m3(x_c * 2^-e)                                (exact scaling, one rounding)
  x^_c   = x8_c * 2^e                                           (the dequantised value)
The attention of the option is that of q, dY (bf16) on K^, V^ (the oracle reads K^, V^ as fp64).
RNE to e4m3 is torch's float8_e4m3fn conversion (a library primitive); pinned in
tests/test_oracle_quant.py against an exhaustive decode of the 256 codes, round-to-nearest-even on
the midpoints, and closed forms of the exponent rule.
"""
from __future__ import annotations

import math

import numpy as np
import torch

E4M3_MAX = 448.0


def exponent(amax: float) -> int:
    """Smallest integer e with amax <= 448 * 2^e (exact, by fp64 comparisons of powers of two)."""
    if amax == 0.0:
        return -126
    e = int(math.ceil(math.log2(amax / E4M3_MAX)))
    while amax > E4M3_MAX * 2.0 ** e:
        e += 1
    while amax <= E4M3_MAX * 2.0 ** (e - 1):
        e -= 1
    return max(-126, min(126, e))


def rne_e4m3(x: np.ndarray) -> np.ndarray:
    """Round float32 values (|x| <= 448) to the nearest e4m3 value, ties to even; returned as fp64."""
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.float8_e4m3fn).to(torch.float64).numpy()


def _f32(x: np.ndarray) -> np.ndarray:
    if x.dtype == np.uint16:   # bf16 bit patterns
        return (x.astype(np.uint32) << 16).view(np.float32)
    return np.asarray(x, np.float32)


def exponents(amax: np.ndarray) -> np.ndarray:
    """`exponent` over an array (the same fp64 comparisons, vectorised; checked against it in the pins)."""
    a = np.asarray(amax, np.float64)
    with np.errstate(divide="ignore"):
        e = np.ceil(np.log2(np.where(a > 0, a, 1.0) / E4M3_MAX))
    for _ in range(2):
        e = e + (a > E4M3_MAX * np.exp2(e))
        e = e - (a <= E4M3_MAX * np.exp2(e - 1))
    e = np.where(a > 0, e, -126)
    return np.clip(e, -126, 126).astype(np.int64)


def quantize(x: np.ndarray):
    """x: [n, h, d] (bf16 bits as uint16, or float32).  Returns (dequantised fp64 [n, h, d], e int[n, h])."""
    f = _f32(x)
    n, h, _ = f.shape
    amax = np.abs(f).max(axis=2) if f.size else np.zeros((n, h), np.float32)
    e = exponents(amax)
    scaled = f.astype(np.float64) * np.ldexp(1.0, -e)[:, :, None]     # exact: power-of-two scaling
    q8 = rne_e4m3(scaled.astype(np.float32))                           # the one rounding
    return q8 * np.ldexp(1.0, e)[:, :, None], e
