"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module draws random numbers and assembles input graphs (canonical CSR) and
feature tensors.  It contains none of the method's arithmetic.  Recipes are the
ones stated in DESIGN.md ("Input recipe"), following SURVEY.md section 8(d) G1-G5:
shapes, sizes, degree distributions and community structure of the paper's
benchmark graphs (Table 2; configs in BASELINE.json).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "gen.c")
_LIB = os.path.join(_HERE, "libgtgen.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("directed", ctypes.c_int32),
        ("n", ctypes.c_int64), ("m", ctypes.c_int64), ("seed", ctypes.c_uint64),
        ("wdist_out", ctypes.c_int32), ("wdist_in", ctypes.c_int32),
        ("wparam_out", ctypes.c_double), ("wmean_out", ctypes.c_double), ("wcap_out", ctypes.c_double),
        ("wparam_in", ctypes.c_double), ("wmean_in", ctypes.c_double), ("wcap_in", ctypes.c_double),
        ("comm_size", ctypes.c_int64), ("f_in", ctypes.c_double),
        ("scale", ctypes.c_int32), ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double),
        ("permute", ctypes.c_int32), ("oversample", ctypes.c_double),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.gen_graph.restype = ctypes.c_int64
        _lib.gen_graph.argtypes = [ctypes.POINTER(_Params), ctypes.POINTER(ctypes.c_void_p),
                                   ctypes.POINTER(ctypes.c_void_p)]
        _lib.gen_free.argtypes = [ctypes.c_void_p]
        _lib.gen_normal_f32.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, ctypes.c_void_p]
        _lib.gen_normal_f32_range.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_void_p]
        _lib.gen_f32_to_bf16.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        _lib.gen_num_threads.restype = ctypes.c_int
    return _lib


PARETO, LOGNORMAL, CONSTANT = 0, 1, 2


@dataclass
class GraphSpec:
    """One synthetic graph recipe (Input recipe)."""
    name: str
    n: int
    m: int                       # unique pairs (undirected) / edges (directed)
    directed: bool
    seed: int
    kind: int = 0                # 0 Chung-Lu, 1 R-MAT
    wdist_out: int = PARETO
    wparam_out: float = 2.5
    wmean_out: float = 4.0
    wcap_out: float = 0.0
    wdist_in: int = PARETO
    wparam_in: float = 2.5
    wmean_in: float = 4.0
    wcap_in: float = 0.0
    comm_size: int = 0
    f_in: float = 0.0
    scale: int = 0
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    permute: bool = False
    oversample: float = 1.1

    @property
    def nnz(self) -> int:
        return self.m if self.directed else 2 * self.m


@dataclass
class Config:
    """A benchmark/parity configuration: graph + heads x head_dim + dtype (BASELINE.json configs)."""
    name: str
    graph: GraphSpec
    heads: int
    d: int
    dtype: str                   # "f32" | "bf16"


# BASELINE.json configs[0..4]; SURVEY.md section 8(d) G1-G5.
GRAPHS = {
    # Cora: 2,708 nodes, 5,278 undirected pairs -> 10,556 nnz; power-law, max degree ~168.
    "cora": GraphSpec("cora", 2708, 5278, False, 1, wdist_out=PARETO, wparam_out=2.5,
                      wmean_out=2 * 5278 / 2708, wcap_out=168.0),
    # ogbn-arxiv: 169,343 nodes, 1,166,243 directed edges; lognormal out-weights (mean 6.9),
    # power-law in-weights (citations), capped at arxiv's max in-degree.
    "arxiv": GraphSpec("arxiv", 169343, 1166243, True, 2, wdist_out=LOGNORMAL, wparam_out=1.0,
                       wmean_out=6.9, wcap_out=500.0, wdist_in=PARETO, wparam_in=2.1,
                       wmean_in=6.9, wcap_in=13161.0),
    # ogbn-products: 2,449,029 nodes, 61,859,140 undirected pairs -> 123,718,280 nnz (Table 2's 123M);
    # community Chung-Lu, communities of 4,096 consecutive ids, f_in = 0.9, Pareto(2.2) capped at 17,481.
    "products": GraphSpec("products", 2449029, 61859140, False, 3, wdist_out=PARETO, wparam_out=2.2,
                          wmean_out=2 * 61859140 / 2449029, wcap_out=17481.0, comm_size=4096,
                          f_in=0.9, oversample=1.12),
    # Reddit: 232,965 nodes, 57,307,946 undirected pairs -> 114,615,892 nnz; 50 communities, f_in=0.5,
    # lognormal weights (mean degree 492, cap 21,657).
    "reddit": GraphSpec("reddit", 232965, 57307946, False, 4, wdist_out=LOGNORMAL, wparam_out=1.0,
                        wmean_out=2 * 57307946 / 232965, wcap_out=21657.0, comm_size=4660, f_in=0.5,
                        oversample=1.25),
    # R-MAT scale 24, 2^28 unique directed edges (Graph500 a,b,c,d = .57,.19,.19,.05), labels permuted.
    "rmat": GraphSpec("rmat", 1 << 24, 1 << 28, True, 5, kind=1, scale=24, permute=True, oversample=1.03),
}

CONFIGS = {
    "C1": Config("C1-cora", GRAPHS["cora"], 8, 16, "f32"),
    "C2": Config("C2-arxiv", GRAPHS["arxiv"], 8, 32, "bf16"),
    "C3": Config("C3-products", GRAPHS["products"], 4, 64, "bf16"),
    "C3f": Config("C3f-products-f32", GRAPHS["products"], 4, 64, "f32"),
    "C4": Config("C4-reddit", GRAPHS["reddit"], 4, 64, "bf16"),
    "C5": Config("C5-rmat", GRAPHS["rmat"], 4, 64, "bf16"),
}

# feature tensor ids (Philox stream per tensor)
TENSOR_IDS = {"q": 0, "k": 1, "v": 2, "dy": 3}


def make_graph(spec: GraphSpec) -> tuple[np.ndarray, np.ndarray]:
    """Returns canonical CSR (row_ptr int64[n+1], col_idx int32[nnz])."""
    lib = _load()
    p = _Params(spec.kind, int(spec.directed), spec.n, spec.m, spec.seed,
                spec.wdist_out, spec.wdist_in, spec.wparam_out, spec.wmean_out, spec.wcap_out,
                spec.wparam_in, spec.wmean_in, spec.wcap_in, spec.comm_size, spec.f_in,
                spec.scale, spec.a, spec.b, spec.c, int(spec.permute), spec.oversample)
    rp = ctypes.c_void_p()
    ci = ctypes.c_void_p()
    nnz = lib.gen_graph(ctypes.byref(p), ctypes.byref(rp), ctypes.byref(ci))
    if nnz < 0:
        raise RuntimeError(f"gen_graph({spec.name}) failed: {nnz}")
    row_ptr = np.ctypeslib.as_array((ctypes.c_int64 * (spec.n + 1)).from_address(rp.value)).copy()
    col_idx = (np.ctypeslib.as_array((ctypes.c_int32 * nnz).from_address(ci.value)).copy()
               if nnz > 0 else np.zeros(0, np.int32))
    lib.gen_free(rp)
    lib.gen_free(ci)
    return row_ptr, col_idx


def random_graph(n: int, m: int, seed: int, directed: bool = True, power: float = 0.0,
                 comm_size: int = 0, f_in: float = 0.0) -> tuple[np.ndarray, np.ndarray]:
    """Small/medium random graph for parity tests: m unique pairs; uniform weights (power=0)
    or Pareto(power) weights; optional communities."""
    spec = GraphSpec("random", n, m, directed, seed,
                     wdist_out=(PARETO if power else CONSTANT), wparam_out=power or 2.0, wmean_out=1.0,
                     wdist_in=(PARETO if power else CONSTANT), wparam_in=power or 2.0, wmean_in=1.0,
                     comm_size=comm_size, f_in=f_in, oversample=1.5)
    return make_graph(spec)


def csr_from_pairs(n: int, pairs) -> tuple[np.ndarray, np.ndarray]:
    """Canonical CSR from an explicit list of directed (u, v) pairs (hand-built test graphs)."""
    pairs = sorted(set((int(u), int(v)) for u, v in pairs))
    row_ptr = np.zeros(n + 1, np.int64)
    for u, _ in pairs:
        row_ptr[u + 1] += 1
    row_ptr = np.cumsum(row_ptr).astype(np.int64)
    col_idx = np.array([v for _, v in pairs], np.int32)
    return row_ptr, col_idx


def normal_f32(seed: int, tensor_id: int, shape) -> np.ndarray:
    """i.i.d. N(0,1) float32 (Philox4x32-10 keyed by seed, stream = tensor id, counter = flat index)."""
    lib = _load()
    n = int(np.prod(shape))
    out = np.empty(n, np.float32)
    if n:
        lib.gen_normal_f32(ctypes.c_uint64(seed), tensor_id, n, out.ctypes.data)
    return out.reshape(shape)


def normal_f32_rows(seed: int, tensor_id: int, row_lo: int, row_hi: int, row_elems: int) -> np.ndarray:
    """Rows [row_lo, row_hi) of the [n, row_elems] tensor normal_f32(seed, tensor_id, (n, row_elems))."""
    lib = _load()
    n = (row_hi - row_lo) * row_elems
    out = np.empty(n, np.float32)
    if n:
        lib.gen_normal_f32_range(ctypes.c_uint64(seed), tensor_id, row_lo * row_elems, n, out.ctypes.data)
    return out.reshape(row_hi - row_lo, row_elems)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    lib = _load()
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(x.shape, np.uint16)
    if x.size:
        lib.gen_f32_to_bf16(x.ctypes.data, x.size, out.ctypes.data)
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def features(seed: int, name: str, n: int, heads: int, d: int, dtype: str, scale: float = 1.0,
             row_lo: int = 0, row_hi: int | None = None):
    """Feature tensor rows [row_lo, row_hi) of [n, heads, d]: fp32 array, or uint16 bf16 bits when
    dtype == 'bf16'.  Any row slice equals the same rows of the full tensor."""
    row_hi = n if row_hi is None else row_hi
    x = normal_f32_rows(seed, TENSOR_IDS[name], row_lo, row_hi, heads * d).reshape(row_hi - row_lo, heads, d)
    if scale != 1.0:
        x = (x * np.float32(scale)).astype(np.float32)
    if dtype == "bf16":
        return f32_to_bf16_bits(x)
    return x


def num_threads() -> int:
    return _load().gen_num_threads()
