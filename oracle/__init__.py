"""CPU fp64 oracle for sparse graph attention (forward + backward) and the partition/halo sets.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares no code
with the CUDA path (``paper_2604_16715_b200``) and neither imports the other.

Each function follows the paper's definitions (Eq. 2, Eq. 4 P:86-89,
Eq. 5, Section 2.2) as restated in ``oracle/oracle.c``; readings Z1-Z22 are
listed in DESIGN.md.  Pins: ``tests/test_oracle_pins.py`` (dense brute force in torch fp64,
SPEC worked examples, closed forms, invariants, finite differences) and
``tests/test_oracle_partition.py`` (hand-computed partitions and halos, brute force).
Every function here is pinned; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

F32, BF16, F64 = 0, 1, 2


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.oracle_fwd.argtypes = [_I64, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P,
                                   ctypes.c_double, _P, _P]
        lib.oracle_bwd.argtypes = [_I64, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P,
                                   ctypes.c_double, _P, _P, _P, _P]
        lib.oracle_sample.argtypes = [_I64, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P,
                                      ctypes.c_double, _I64, _P, _P, _P, _P, _P, _I64, _P, _P, _P]
        lib.oracle_transpose.argtypes = [_I64, _P, _P, _P, _P, _P]
        lib.oracle_partition.argtypes = [_I64, _P, ctypes.c_int, ctypes.c_int, _P]
        lib.oracle_halo.argtypes = [_I64, _P, _P, _I64, _I64, ctypes.c_int, _P, _I64]
        lib.oracle_halo.restype = _I64
        _lib = lib
    return _lib


def _dt(x: np.ndarray) -> int:
    if x.dtype == np.float32:
        return F32
    if x.dtype == np.uint16:
        return BF16
    if x.dtype == np.float64:
        return F64
    raise TypeError(f"oracle inputs are float32, bf16 bits (uint16) or float64, got {x.dtype}")


def _c(x, dtype=None):
    return np.ascontiguousarray(x if dtype is None else x.astype(dtype, copy=False))


def _ptr(x):
    return None if x is None else x.ctypes.data


def forward(row_ptr, col_idx, q, k, v, scale: float):
    """Y [n,h,d] fp64 and LSE [n,h] fp64 (LSE = -inf on empty rows)."""
    lib = _load()
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    q, k, v = _c(q), _c(k), _c(v)
    n, h, d = q.shape
    y = np.zeros((n, h, d), np.float64)
    lse = np.zeros((n, h), np.float64)
    lib.oracle_fwd(n, row_ptr.ctypes.data, col_idx.ctypes.data, h, d, _dt(q), q.ctypes.data, k.ctypes.data,
                   v.ctypes.data, float(scale), y.ctypes.data, lse.ctypes.data)
    return y, lse


def backward(row_ptr, col_idx, q, k, v, dy, scale: float):
    """dQ, dK, dV [n,h,d] fp64 and Dstat [n,h] fp64 (D_i = sum_e U_e dU_e)."""
    lib = _load()
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    q, k, v, dy = _c(q), _c(k), _c(v), _c(dy)
    n, h, d = q.shape
    dq = np.zeros((n, h, d), np.float64)
    dk = np.zeros((n, h, d), np.float64)
    dv = np.zeros((n, h, d), np.float64)
    ds = np.zeros((n, h), np.float64)
    lib.oracle_bwd(n, row_ptr.ctypes.data, col_idx.ctypes.data, h, d, _dt(q), q.ctypes.data, k.ctypes.data,
                   v.ctypes.data, dy.ctypes.data, float(scale), dq.ctypes.data, dk.ctypes.data, dv.ctypes.data,
                   ds.ctypes.data)
    return dq, dk, dv, ds


def sample(row_ptr, col_idx, q, k, v, dy, scale: float, rows, cols):
    """Oracle outputs restricted to sampled rows (Y, LSE, dQ, Dstat) and columns (dK, dV)."""
    lib = _load()
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    q, k, v = _c(q), _c(k), _c(v)
    dy = None if dy is None else _c(dy)
    n, h, d = q.shape
    rows = _c(np.asarray(rows), np.int64)
    cols = _c(np.asarray(cols), np.int64)
    nr, nc = len(rows), len(cols)
    y = np.zeros((nr, h, d)); lse = np.zeros((nr, h))
    dq = np.zeros((nr, h, d)) if dy is not None else None
    dst = np.zeros((nr, h)) if dy is not None else None
    dk = np.zeros((nc, h, d)) if dy is not None else None
    dv = np.zeros((nc, h, d)) if dy is not None else None
    lib.oracle_sample(n, row_ptr.ctypes.data, col_idx.ctypes.data, h, d, _dt(q), q.ctypes.data, k.ctypes.data,
                      v.ctypes.data, _ptr(dy), float(scale), nr, rows.ctypes.data, y.ctypes.data,
                      lse.ctypes.data, _ptr(dq), _ptr(dst), nc, cols.ctypes.data, _ptr(dk), _ptr(dv))
    return {"y": y, "lse": lse, "dq": dq, "dstat": dst, "dk": dk, "dv": dv}


def transpose(row_ptr, col_idx):
    """Oracle's own counting-sort transpose: (col_ptr int64[n+1], row_idx int32[nnz]); rows ascending
    within each column."""
    lib = _load()
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    n = len(row_ptr) - 1
    nnz = int(row_ptr[-1])
    col_ptr = np.zeros(n + 1, np.int64)
    row_idx = np.zeros(max(nnz, 1), np.int32)
    lib.oracle_transpose(n, row_ptr.ctypes.data, col_idx.ctypes.data, col_ptr.ctypes.data, row_idx.ctypes.data,
                         None)
    return col_ptr, row_idx[:nnz]


def partition(row_ptr, p: int, mode: int = 0) -> np.ndarray:
    """bounds int64[p+1]; mode 0 = rows+edges balanced (reading Z9), 1 = SPEC node-balanced."""
    lib = _load()
    row_ptr = _c(row_ptr, np.int64)
    n = len(row_ptr) - 1
    b = np.zeros(p + 1, np.int64)
    if lib.oracle_partition(n, row_ptr.ctypes.data, p, mode, b.ctypes.data) != 0:
        raise ValueError("bad partition arguments")
    return b


def halo(row_ptr, col_idx, lo: int, hi: int, inward: bool = False) -> np.ndarray:
    """Out-halo (remote columns touched by rows [lo,hi)) or in-halo (remote rows with an edge into a
    column in [lo,hi)); sorted ascending int32."""
    lib = _load()
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    n = len(row_ptr) - 1
    cnt = lib.oracle_halo(n, row_ptr.ctypes.data, col_idx.ctypes.data, lo, hi, int(inward), None, 0)
    out = np.zeros(max(cnt, 1), np.int32)
    lib.oracle_halo(n, row_ptr.ctypes.data, col_idx.ctypes.data, lo, hi, int(inward), out.ctypes.data, cnt)
    return out[:cnt]


def send_list(halo_r: np.ndarray, bounds: np.ndarray, s: int) -> np.ndarray:
    """send[s -> r] = H_r intersected with rank s's owned range [b_s, b_{s+1})."""
    return halo_r[(halo_r >= bounds[s]) & (halo_r < bounds[s + 1])]
