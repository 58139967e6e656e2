"""Thin ctypes binding of libgt.so (include/gt.h).  Argument marshalling only: every step of the
sparse attention path runs in the library's CUDA kernels.  PyTorch supplies device memory,
streams and process groups.  If libgt.so is missing this module raises; there is no fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GT_LIB") or os.path.join(_HERE, "libgt.so")

GT_OK, GT_EINVAL, GT_EGRAPH, GT_ECONFIG, GT_ENOMEM, GT_ECUDA, GT_ENCCL, GT_ESTATE = range(8)
STATUS_NAMES = ["GT_OK", "GT_EINVAL", "GT_EGRAPH", "GT_ECONFIG", "GT_ENOMEM", "GT_ECUDA", "GT_ENCCL", "GT_ESTATE"]
GT_F32, GT_BF16 = 0, 1
GT_AUTO, GT_SINGLE, GT_ALLGATHER, GT_HALO = range(4)
STRATEGIES = {"auto": GT_AUTO, "single": GT_SINGLE, "allgather": GT_ALLGATHER, "halo": GT_HALO, "a2a": 4}
STRATEGY_NAMES = {v: k for k, v in STRATEGIES.items()}
GT_COMM_NONE, GT_COMM_NCCL, GT_COMM_LOOPBACK, GT_COMM_HOSTIPC = range(4)
EXPORT = {"bounds": 0, "halo_out": 1, "halo_in": 2, "send_out": 3, "send_in": 4, "csc_ptr": 5, "csc_idx": 6,
          "heavy_rows": 7, "heavy_cols": 8, "kv8": 9}
_EXPORT_I64 = {"bounds", "csc_ptr"}


class GTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")


class _Csr(ctypes.Structure):
    _fields_ = [("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p)]


class _Opts(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("comm_kind", ctypes.c_int), ("comm", ctypes.c_void_p),
                ("dtype", ctypes.c_int), ("scale", ctypes.c_float), ("strategy", ctypes.c_int),
                ("validate", ctypes.c_int), ("partition", ctypes.c_int), ("device", ctypes.c_int),
                ("heavy_threshold", ctypes.c_int), ("beta_profile", ctypes.c_char_p), ("profile", ctypes.c_int),
                ("edge_state", ctypes.c_int), ("bwd_mode", ctypes.c_int), ("transport", ctypes.c_int),
                ("cuda_graphs", ctypes.c_int), ("kv_fp8", ctypes.c_int), ("reserve_sms", ctypes.c_int),
                ("hot_cols", ctypes.c_int)]


class _Info(ctypes.Structure):
    _fields_ = ([(f, ctypes.c_int) for f in ("world", "rank", "strategy", "dtype", "heads", "d")]
                + [("scale", ctypes.c_float)]
                + [(f, ctypes.c_int64) for f in (
                    "n", "nnz", "row_lo", "row_hi", "n_local", "nnz_local", "nnz_in_local", "halo_out_rows",
                    "halo_in_rows", "exch_fwd_bytes", "exch_bwd_bytes", "send_fwd_bytes", "send_bwd_bytes",
                    "device_bytes", "heavy_rows", "heavy_row_chunks", "heavy_cols", "heavy_col_chunks")]
                + [("launches_fwd", ctypes.c_int), ("launches_bwd", ctypes.c_int)]
                + [("beta_s_per_row", ctypes.c_double * 5), ("predicted_ms", ctypes.c_double * 5),
                   ("agp_score", ctypes.c_double * 5), ("agp_feasible", ctypes.c_int * 5),
                   ("alpha_s_per_unit", ctypes.c_double), ("edge_state", ctypes.c_int),
                   ("edge_state_bytes", ctypes.c_int64), ("bwd_mode", ctypes.c_int),
                   ("transport", ctypes.c_int), ("fwd_gen", ctypes.c_int64), ("stale_bwds", ctypes.c_int64),
                   ("kv_fp8", ctypes.c_int), ("kv_fp8_bytes", ctypes.c_int64), ("hot_cols", ctypes.c_int64),
                   ("hot_entries", ctypes.c_int64), ("bwd_colfirst", ctypes.c_int)])


_lib = None
_lock = threading.Lock()
_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def _nccl_hint():
    if os.environ.get("GT_NCCL_LIB"):
        return
    try:
        import nvidia.nccl  # torch's bundled NCCL
        for base in nvidia.nccl.__path__:
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["GT_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def lib():
    """Loads libgt.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                               "(there is no CPU or PyTorch fallback)")
        try:
            import torch  # noqa: F401  (loads CUDA runtime + NCCL first)
        except Exception:
            pass
        _nccl_hint()
        L = ctypes.CDLL(LIB_PATH)
        L.gt_default_opts.argtypes = [ctypes.POINTER(_Opts)]
        L.gt_plan.argtypes = [ctypes.POINTER(_Csr), _I64, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.POINTER(_Opts), ctypes.POINTER(_P)]
        L.gt_plan_info_get.argtypes = [_P, ctypes.POINTER(_Info)]
        L.gt_plan_export.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _I64, ctypes.POINTER(_I64)]
        L.gt_attn_fwd.argtypes = [_P, _P, _P, _P, _P, _P, _P]
        L.gt_attn_bwd.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]
        L.gt_attn_fwd_bwd_host.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]
        L.gt_plan_timings.argtypes = [_P, _P, _P]
        L.gt_free.argtypes = [_P]
        L.gt_free.restype = None
        L.gt_last_error.restype = ctypes.c_char_p
        L.gt_version.restype = ctypes.c_char_p
        L.gt_nccl_unique_id.argtypes = [_P]
        L.gt_nccl_comm_create.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]
        L.gt_nccl_comm_destroy.argtypes = [_P]
        L.gt_nccl_comm_destroy.restype = None
        L.gt_loopback_create.argtypes = [ctypes.c_int, ctypes.POINTER(_P)]
        L.gt_loopback_destroy.argtypes = [_P]
        L.gt_loopback_destroy.restype = None
        L.gt_hostipc_create.argtypes = [ctypes.POINTER(_HostColl), ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]
        L.gt_hostipc_destroy.argtypes = [_P]
        L.gt_hostipc_destroy.restype = None
        L.gt_partition.argtypes = [_I64, _P, ctypes.c_int, ctypes.c_int, _P]
        L.gt_halo.argtypes = [_I64, _P, _P, _I64, _I64, ctypes.c_int, _P, _I64, ctypes.POINTER(_I64)]
        L.gt_send_list.argtypes = [_I64, _P, _P, _I64, _I64, _I64, _I64, ctypes.c_int, _P, _I64,
                                   ctypes.POINTER(_I64)]
        L.gt_estimate_iter_time.argtypes = [ctypes.c_double, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.gt_estimate_iter_time.restype = ctypes.c_double
        L.gt_agp_select.argtypes = [ctypes.c_double, ctypes.c_double, _P, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_double)]
        L.gt_fit_beta.argtypes = [_P, _P, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        _lib = L
        return L


def _check(status: int):
    if status != GT_OK:
        raise GTError(status, lib().gt_last_error().decode(errors="replace"))


def version() -> str:
    return lib().gt_version().decode()


# ---------------------------------------------------------------- host-only planning helpers --
def partition(row_ptr: np.ndarray, p: int, mode: int = 0) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    out = np.zeros(p + 1, np.int64)
    _check(lib().gt_partition(len(row_ptr) - 1, row_ptr.ctypes.data, p, mode, out.ctypes.data))
    return out


def halo(row_ptr: np.ndarray, col_idx: np.ndarray, lo: int, hi: int, inward: bool = False) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    n = len(row_ptr) - 1
    ln = _I64()
    _check(lib().gt_halo(n, row_ptr.ctypes.data, col_idx.ctypes.data, lo, hi, int(inward), None, 0, ctypes.byref(ln)))
    out = np.zeros(max(ln.value, 1), np.int32)
    _check(lib().gt_halo(n, row_ptr.ctypes.data, col_idx.ctypes.data, lo, hi, int(inward), out.ctypes.data,
                         ln.value, ctypes.byref(ln)))
    return out[:ln.value]


def send_list(row_ptr: np.ndarray, col_idx: np.ndarray, lo: int, hi: int, peer_lo: int, peer_hi: int,
              inward: bool = False) -> np.ndarray:
    """Rows the owner of [lo, hi) sends to the owner of [peer_lo, peer_hi) (gt_send_list)."""
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    n = len(row_ptr) - 1
    ln = _I64()
    _check(lib().gt_send_list(n, row_ptr.ctypes.data, col_idx.ctypes.data, lo, hi, peer_lo, peer_hi, int(inward),
                              None, 0, ctypes.byref(ln)))
    out = np.zeros(max(ln.value, 1), np.int32)
    _check(lib().gt_send_list(n, row_ptr.ctypes.data, col_idx.ctypes.data, lo, hi, peer_lo, peer_hi, int(inward),
                              out.ctypes.data, ln.value, ctypes.byref(ln)))
    return out[:ln.value]


def estimate_iter_time(alpha1: float, beta: np.ndarray, c: int, p: int, N: float, E: float) -> float:
    """Eq. 7 with Eq. 8.  beta: [n_strategies, P + 1] seconds per node."""
    beta = np.ascontiguousarray(beta, np.float64)
    ns, P1 = beta.shape
    return lib().gt_estimate_iter_time(alpha1, beta.ctypes.data, ns, P1 - 1, c, p, N, E)


def agp_select(N: float, t_iter1: float, beta: np.ndarray):
    """Algorithm 3.  beta: [n_strategies, P + 1].  Returns (c, s, score); c = -1 means single GPU."""
    beta = np.ascontiguousarray(beta, np.float64)
    ns, P1 = beta.shape
    c, s, sc = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    _check(lib().gt_agp_select(N, t_iter1, beta.ctypes.data, ns, P1 - 1, ctypes.byref(c), ctypes.byref(s),
                               ctypes.byref(sc)))
    return c.value, s.value, sc.value


def fit_beta(x, t) -> float:
    x = np.ascontiguousarray(x, np.float64)
    t = np.ascontiguousarray(t, np.float64)
    b = ctypes.c_double()
    _check(lib().gt_fit_beta(x.ctypes.data, t.ctypes.data, len(x), ctypes.byref(b)))
    return b.value


# ----------------------------------------------------------------------- multi-rank plumbing --
class LoopbackGroup:
    """In-process group of `world` ranks driven by `world` host threads on one device (tests)."""

    def __init__(self, world: int):
        h = _P()
        _check(lib().gt_loopback_create(world, ctypes.byref(h)))
        self.handle = h.value
        self.world = world

    def close(self):
        if self.handle:
            lib().gt_loopback_destroy(self.handle)
            self.handle = None


_ALLGATHER_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


class _HostColl(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allgather", _ALLGATHER_CB)]


class HostIpcGroup:
    """GT_COMM_HOSTIPC: one process per rank, device data moved by CUDA IPC (gt_hostipc_create), host
    collectives over a torch.distributed process group (gloo): several processes can share ONE GPU,
    which NCCL refuses.  Create it with the rank's CUDA device current; close it after every plan."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

        def allgather(_ctx, send, recv, nbytes):
            try:
                t = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)), dtype=torch.uint8)
                out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(out, t, group=self.group)
                flat = torch.cat(out).numpy()
                ctypes.memmove(recv, flat.ctypes.data, self.world * nbytes)
                return 0
            except Exception:  # reported to the library as a failed collective (GT_ENCCL)
                return 1

        self._cb = _ALLGATHER_CB(allgather)      # kept alive as long as the group
        self._coll = _HostColl(None, self._cb)
        h = _P()
        _check(lib().gt_hostipc_create(ctypes.byref(self._coll), self.world, self.rank, ctypes.byref(h)))
        self.handle = h.value

    def close(self):
        if self.handle:
            lib().gt_hostipc_destroy(self.handle)
            self.handle = None


class NcclComm:
    """NCCL communicator bootstrapped over a torch.distributed process group (rank 0's unique id is
    broadcast through the group)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = bytearray(128)
        if rank == 0:
            buf = (ctypes.c_char * 128).from_buffer(uid)
            _check(lib().gt_nccl_unique_id(ctypes.addressof(buf)))
        backend = dist.get_backend(group)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=0, group=group)
        uid = bytes(t.cpu().tolist())
        ubuf = ctypes.create_string_buffer(uid, 128)
        h = _P()
        _check(lib().gt_nccl_comm_create(ctypes.addressof(ubuf), world, rank, ctypes.byref(h)))
        self.handle = h.value
        self.world, self.rank = world, rank

    def close(self):
        if self.handle:
            lib().gt_nccl_comm_destroy(self.handle)
            self.handle = None


def _dtype_code(dtype) -> int:
    if dtype in ("f32", "float32", GT_F32):
        return GT_F32
    if dtype in ("bf16", "bfloat16", GT_BF16):
        return GT_BF16
    try:
        import torch
        if dtype == torch.float32:
            return GT_F32
        if dtype == torch.bfloat16:
            return GT_BF16
    except Exception:
        pass
    raise ValueError(f"unsupported dtype {dtype!r}")


class Plan:
    """A gt_plan_t: the graph prepared for sparse attention on this rank's device (gt_plan).

    row_ptr / col_idx: the GLOBAL CSR (int64 / int32), identical on every rank.  heads, d: the
    [N, heads, d] layout of every feature tensor.  Options map one to one onto gt_opts (include/gt.h):
    dtype "bf16" | "f32"; scale (0 -> 1 / sqrt(heads d)); world / rank / comm (LoopbackGroup or
    NcclComm) for multi-rank plans; strategy "auto" | "single" | "allgather" | "halo" | "a2a";
    heavy_threshold (0 -> 512); partition 0 (rows + edges) | 1 (nodes); edge_state 0 | 1 | -1
    (materialised logits and (P, dS): auto / on / off); bwd_mode 0 (transposed owner) | 1
    (reduce-scatter); transport 0 (copies) | 1 (fused peer gather); cuda_graphs (world-1 graph
    replay); beta_profile (JSON of measured beta per strategy for GT_AUTO instead of plan-time probes);
    profile (per-stage CUDA events); kv_fp8 (fp8 K||V storage, gt_opts.kv_fp8: world 1, bf16, entry state);
    hot_cols (hot-column K||V table under a persisting L2 window, gt_opts.hot_cols: world 1); reserve_sms
    (world > 1: SMs left to the communication kernels during the forward's overlap; 0 -> 16, -1 -> none).
    """

    def __init__(self, row_ptr, col_idx, heads: int, d: int, dtype="bf16", scale: float = 0.0, world: int = 1,
                 rank: int = 0, comm=None, strategy="auto", heavy_threshold: int = 0, partition: int = 0,
                 validate: bool = True, device: int = -1, profile: bool = False, edge_state: int = 0,
                 bwd_mode: int = 0, transport: int = 0, cuda_graphs: bool = False, beta_profile=None,
                 kv_fp8: bool = False, hot_cols: int = 0, reserve_sms: int = 0):
        L = lib()
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, np.int32)
        n = len(self.row_ptr) - 1
        nnz = int(self.row_ptr[-1]) if n >= 0 else 0
        opts = _Opts()
        L.gt_default_opts(ctypes.byref(opts))
        opts.rank = rank
        opts.dtype = _dtype_code(dtype)
        opts.scale = float(scale)
        opts.strategy = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
        opts.validate = int(validate)
        opts.partition = int(partition)
        opts.device = int(device)
        opts.heavy_threshold = int(heavy_threshold)
        opts.profile = int(profile)
        opts.edge_state = int(edge_state)
        opts.bwd_mode = int(bwd_mode)
        opts.transport = int(transport)
        opts.cuda_graphs = int(cuda_graphs)
        opts.kv_fp8 = int(kv_fp8)
        opts.hot_cols = int(hot_cols)
        opts.reserve_sms = int(reserve_sms)
        self._beta_profile = str(beta_profile).encode() if beta_profile else None  # kept alive for gt_plan
        opts.beta_profile = self._beta_profile
        if world > 1:
            if isinstance(comm, LoopbackGroup):
                opts.comm_kind, opts.comm = GT_COMM_LOOPBACK, comm.handle
            elif isinstance(comm, NcclComm):
                opts.comm_kind, opts.comm = GT_COMM_NCCL, comm.handle
            elif isinstance(comm, HostIpcGroup):
                opts.comm_kind, opts.comm = GT_COMM_HOSTIPC, comm.handle
            else:
                raise ValueError("world > 1 needs a LoopbackGroup, NcclComm or HostIpcGroup")
        csr = _Csr(self.row_ptr.ctypes.data, self.col_idx.ctypes.data if nnz else None)
        h = _P()
        _check(L.gt_plan(ctypes.byref(csr), n, nnz, heads, d, world, ctypes.byref(opts), ctypes.byref(h)))
        self.handle = h.value
        self.heads, self.d, self.dtype_code = heads, d, opts.dtype
        self.device = int(device)
        if self.device < 0:
            import torch
            self.device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        inf = self.info()
        self.n_local = inf["n_local"]
        self.row_lo, self.row_hi = inf["row_lo"], inf["row_hi"]
        self.scale = inf["scale"]

    # -- introspection --
    def info(self) -> dict:
        I = _Info()
        _check(lib().gt_plan_info_get(self.handle, ctypes.byref(I)))
        out = {}
        for name, _ in _Info._fields_:
            v = getattr(I, name)
            out[name] = list(v) if hasattr(v, "__len__") else v
        out["strategy_name"] = STRATEGY_NAMES.get(out["strategy"], "?")
        return out

    def export(self, what: str, peer: int = 0) -> np.ndarray:
        code = EXPORT[what]
        ln = _I64()
        _check(lib().gt_plan_export(self.handle, code, peer, None, 0, ctypes.byref(ln)))
        dt = np.int64 if what in _EXPORT_I64 else (np.uint8 if what == "kv8" else np.int32)
        out = np.zeros(max(ln.value, 1), dt)
        _check(lib().gt_plan_export(self.handle, code, peer, out.ctypes.data, ln.value, ctypes.byref(ln)))
        return out[:ln.value]

    STAGES = ("fwd_exchange", "fwd", "bwd_rows", "bwd_exchange", "bwd_cols")

    def timings(self) -> dict:
        """Per-stage device ms summed since the last call (plan built with profile=True)."""
        ms = np.zeros(5, np.float64)
        calls = np.zeros(5, np.int64)
        _check(lib().gt_plan_timings(self.handle, ms.ctypes.data, calls.ctypes.data))
        return {s: (float(ms[i]), int(calls[i])) for i, s in enumerate(self.STAGES)}

    # -- compute --
    def _torch_dtype(self):
        import torch
        return torch.float32 if self.dtype_code == GT_F32 else torch.bfloat16

    def _check_tensor(self, t, name, lse=False):
        """Shape, dtype, layout and device of a tensor passed to the C ABI (which sees only pointers):
        feature tensors are [n_local, heads, d] of the plan dtype, lse is float32 [n_local, heads],
        all contiguous and on the plan's device.  Raises GTError(GT_EINVAL) (SPEC.md S:56, S:66
        "shape error") instead of letting a kernel read or write out of bounds."""
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise GTError(GT_EINVAL, f"{name} must be a CUDA tensor")
        want_dt = torch.float32 if lse else self._torch_dtype()
        want_shape = (self.n_local, self.heads) if lse else (self.n_local, self.heads, self.d)
        if t.dtype != want_dt:
            raise GTError(GT_EINVAL, f"{name}: dtype {t.dtype} != {want_dt}")
        if tuple(t.shape) != want_shape:
            raise GTError(GT_EINVAL, f"{name}: shape {tuple(t.shape)} != {want_shape} (n_local, heads"
                                     f"{'' if lse else ', d'})")
        if not t.is_contiguous():
            raise GTError(GT_EINVAL, f"{name} must be contiguous")
        if t.device.index != self.device:
            raise GTError(GT_EINVAL, f"{name} is on cuda:{t.device.index}, the plan on cuda:{self.device}")

    @staticmethod
    def _stream(stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return s.cuda_stream

    def fwd(self, q, k, v, y=None, lse=None, stream=None):
        import torch
        for t, nm in ((q, "q"), (k, "k"), (v, "v")):
            self._check_tensor(t, nm)
        y = torch.empty_like(q) if y is None else y
        lse = torch.empty((self.n_local, self.heads), dtype=torch.float32, device=q.device) if lse is None else lse
        self._check_tensor(y, "y")
        self._check_tensor(lse, "lse", lse=True)
        _check(lib().gt_attn_fwd(self.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), y.data_ptr(),
                                 lse.data_ptr(), self._stream(stream)))
        return y, lse

    def bwd(self, q, k, v, y, lse, dy, dq=None, dk=None, dv=None, stream=None):
        """Gradients of sum <dy, Y> w.r.t. q, k, v; y and lse are the forward's outputs for q, k, v."""
        import torch
        for t, nm in ((q, "q"), (k, "k"), (v, "v"), (y, "y"), (dy, "dy")):
            self._check_tensor(t, nm)
        self._check_tensor(lse, "lse", lse=True)
        dq = torch.empty_like(q) if dq is None else dq
        dk = torch.empty_like(k) if dk is None else dk
        dv = torch.empty_like(v) if dv is None else dv
        for t, nm in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
            self._check_tensor(t, nm)
        _check(lib().gt_attn_bwd(self.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), y.data_ptr(), lse.data_ptr(),
                                 dy.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), self._stream(stream)))
        return dq, dk, dv

    def fwd_bwd_host(self, q, k, v, dy, y, lse, dq, dk, dv, stream=None):
        """End-to-end step through the C-ABI with host buffers (pinned CPU tensors)."""
        import torch
        for t, nm in ((q, "q"), (k, "k"), (v, "v"), (dy, "dy"), (y, "y"), (lse, "lse"), (dq, "dq"), (dk, "dk"),
                      (dv, "dv")):
            if t is None and nm not in ("q", "k", "v", "dy"):
                continue
            want_dt = torch.float32 if nm == "lse" else self._torch_dtype()
            want = (self.n_local, self.heads) if nm == "lse" else (self.n_local, self.heads, self.d)
            if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != want_dt or tuple(t.shape) != want \
                    or not t.is_contiguous():
                raise GTError(GT_EINVAL, f"{nm}: expected a contiguous host tensor {want_dt} {want}")
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        _check(lib().gt_attn_fwd_bwd_host(self.handle, ptr(q), ptr(k), ptr(v), ptr(dy), ptr(y), ptr(lse),
                                          ptr(dq), ptr(dk), ptr(dv), self._stream(stream)))

    def close(self):
        if getattr(self, "handle", None):
            lib().gt_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _autograd():
    import torch

    class SparseGraphAttention(torch.autograd.Function):
        """Y = softmax_rows((Q K^T) (.) A * scale) V on the plan's graph (Eq. 4-5)."""

        @staticmethod
        def forward(ctx, plan: Plan, q, k, v):
            q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
            y, lse = plan.fwd(q, k, v)
            ctx.plan = plan
            ctx.save_for_backward(q, k, v, y, lse)
            return y

        @staticmethod
        def backward(ctx, dy):
            q, k, v, y, lse = ctx.saved_tensors
            dq, dk, dv = ctx.plan.bwd(q, k, v, y, lse, dy.contiguous())
            return None, dq, dk, dv

    return SparseGraphAttention


_SGA = None


def sparse_graph_attention(plan: Plan, q, k, v):
    """Autograd-aware sparse graph attention on `plan` (forward and backward through libgt)."""
    global _SGA
    if _SGA is None:
        _SGA = _autograd()
    return _SGA.apply(plan, q, k, v)
