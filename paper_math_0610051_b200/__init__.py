"""paper_math_0610051_b200 -- B200-native fast Fourier integral operator apply.

Thin ctypes binding over the C ABI of include/fio.h (libfio_b200.so, built
in-tree for sm_100a by paper_math_0610051_b200/build.py).  This module only
marshals arguments: the plan's heavy steps and every step of fio_apply run in
the library's CUDA kernels.  There is no CPU fallback -- if the library or a
CUDA device is missing, calls raise.

    Plan(N, c1, c2, ...)      fio_plan
    Plan.apply(f)             fio_apply, device tensors
    Plan.apply_host(f, out)   fio_apply_host (host buffers, copies included)
    Plan.apply_host_stream(fs, outs)  fio_apply_host_stream (a stream of host inputs, copies pipelined)
    Plan(..., nranks=R, group=g)  wedge-sharded plan; the library's NCCL communicator sums the
                              ranks' partials (fio_apply returns this rank's row slab)
    nccl_unique_id()          fio_nccl_unique_id (host only)
    broadcast_nccl_id(group)  rank 0's id to every rank of a torch.distributed group
    geometry(N, W)            fio_geometry (host only)
    assign_wedges(cost, R)    fio_assign_wedges (host only)
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

__all__ = ["FioError", "Plan", "geometry", "assign_wedges", "partition_weights", "nccl_unique_id", "broadcast_nccl_id", "row_slab",
           "library_path", "load_library", "SYMBOLS", "STAGES"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfio_b200.so")
_lib = None

FIO_C64, FIO_C128 = 1, 2
FIO_OK, FIO_WNOTCERT = 0, 1

# every entry point declared in include/fio.h
SYMBOLS = ["fio_default_opts", "fio_plan", "fio_plan_save", "fio_plan_load", "fio_apply", "fio_apply_batch", "fio_apply_adjoint", "fio_apply_host", "fio_apply_host_stream", "fio_destroy", "fio_plan_info",
           "fio_plan_wedges", "fio_geometry", "fio_assign_wedges", "fio_profile_begin", "fio_profile_end",
           "fio_last_error", "fio_version", "fio_nccl_unique_id", "fio_partition_weights"]
NCCL_ID_BYTES = 128
STAGES = ["K0_rows", "K0_cols", "K1_rowpass", "K2_colpass", "K3_interp"]


class FioError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fio error {code}: {msg}")
        self.code = code


class _Phase(ctypes.Structure):
    _fields_ = [("c1", ctypes.c_void_p), ("c2", ctypes.c_void_p), ("b1", ctypes.c_void_p), ("b2", ctypes.c_void_p),
                ("rho_sign", ctypes.c_int)]


class _Amp(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int), ("px", ctypes.c_void_p), ("pxi", ctypes.c_void_p), ("kind", ctypes.c_int)]


class _Opts(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("n_wedges", ctypes.c_int), ("nufft_w", ctypes.c_int),
                ("nufft_beta", ctypes.c_double), ("seed", ctypes.c_uint64), ("device", ctypes.c_int),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("r_init", ctypes.c_int),
                ("r_max", ctypes.c_int), ("certify", ctypes.c_int), ("skeleton", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p), ("wedge_overlap", ctypes.c_double), ("paper_accept", ctypes.c_int),
                ("allgather", ctypes.c_int)]


class _Info(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int), ("W", ctypes.c_int), ("nufft_w", ctypes.c_int), ("dtype", ctypes.c_int),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("n_owned", ctypes.c_int),
                ("sum_q", ctypes.c_int), ("certified", ctypes.c_int), ("nufft_beta", ctypes.c_double),
                ("max_sep_err", ctypes.c_double), ("plan_seconds", ctypes.c_double),
                ("alpha_bytes", ctypes.c_size_t), ("beta_bytes", ctypes.c_size_t),
                ("workspace_bytes", ctypes.c_size_t), ("fine_elems", ctypes.c_size_t),
                ("p1_elems", ctypes.c_size_t), ("launches_per_apply", ctypes.c_int),
                ("meta_bytes", ctypes.c_size_t), ("slots", ctypes.c_longlong),
                ("max_tile_cap", ctypes.c_longlong), ("k3_thread_slots", ctypes.c_longlong),
                ("rank_balance", ctypes.c_double), ("slot_terms", ctypes.c_longlong), ("group_p", ctypes.c_int),
                ("k3_window_rows", ctypes.c_int), ("skeleton_bytes", ctypes.c_size_t),
                ("k3_window_cols", ctypes.c_int), ("k3_streams", ctypes.c_int), ("has_comm", ctypes.c_int),
                ("out_rows", ctypes.c_int), ("wedge_overlap", ctypes.c_double), ("members", ctypes.c_longlong)]


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libfio_b200.so (building it first if its sources are newer).  Raises if it cannot."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    if not _build.up_to_date():
        _build.build()
    lib = ctypes.CDLL(_LIB_PATH)
    P, I = ctypes.c_void_p, ctypes.c_int
    lib.fio_default_opts.argtypes = [ctypes.POINTER(_Opts)]
    lib.fio_default_opts.restype = None
    lib.fio_plan.argtypes = [ctypes.POINTER(P), I, ctypes.POINTER(_Phase), ctypes.POINTER(_Amp), ctypes.c_double,
                             ctypes.POINTER(_Opts)]
    lib.fio_plan_save.argtypes = [P, ctypes.c_char_p]
    lib.fio_plan_load.argtypes = [ctypes.POINTER(P), ctypes.c_char_p, I, ctypes.POINTER(_Phase), ctypes.POINTER(_Amp),
                                  ctypes.c_double, ctypes.POINTER(_Opts)]
    lib.fio_apply.argtypes = [P, P, P, P]
    lib.fio_apply_host.argtypes = [P, P, P, P]
    lib.fio_apply_host_stream.argtypes = [P, I, P, P, P]
    lib.fio_apply_adjoint.argtypes = [P, P, P, P]
    lib.fio_apply_batch.argtypes = [P, I, P, P, P]
    lib.fio_destroy.argtypes = [P]
    lib.fio_plan_info.argtypes = [P, ctypes.POINTER(_Info)]
    lib.fio_plan_wedges.argtypes = [P, P, P, P, P, P, P, P]
    lib.fio_geometry.argtypes = [I, I, P, P, P, P]
    lib.fio_assign_wedges.argtypes = [I, P, I, P]
    lib.fio_profile_begin.argtypes = [P, I]
    lib.fio_profile_end.argtypes = [P, P, P]
    lib.fio_nccl_unique_id.argtypes = [P]
    lib.fio_partition_weights.argtypes = [I, ctypes.c_double, I, I, P]
    lib.fio_last_error.restype = ctypes.c_char_p
    lib.fio_version.restype = ctypes.c_char_p
    for name in ["fio_plan", "fio_apply", "fio_apply_batch", "fio_apply_adjoint", "fio_apply_host",
                 "fio_apply_host_stream", "fio_destroy", "fio_plan_info", "fio_plan_wedges",
                 "fio_geometry", "fio_assign_wedges", "fio_profile_begin", "fio_profile_end", "fio_nccl_unique_id",
                 "fio_partition_weights"]:
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(code: int) -> int:
    if code < 0:
        raise FioError(code, load_library().fio_last_error().decode())
    return code


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> Optional[np.ndarray]:
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _c128(a) -> Optional[np.ndarray]:
    return None if a is None else np.ascontiguousarray(a, dtype=np.complex128)


def geometry(N: int, W: int) -> dict:
    """Wedge partition and lattice boxes chosen by the plan (host only, no GPU)."""
    lib = load_library()
    wo = np.empty(N * N, np.int32)
    M = np.empty((W, 4), np.int32)
    xc = np.empty((W, 2), np.int32)
    box = np.empty((W, 4), np.int32)
    _check(lib.fio_geometry(N, W, _ptr(wo), _ptr(M), _ptr(xc), _ptr(box)))
    return {"wedge_of": wo.reshape(N, N), "M": M.reshape(W, 2, 2), "xc": xc, "box": box[:, :2],
            "fine": box[:, 2:]}


def partition_weights(W: int, overlap: float, xi1: int, xi2: int) -> np.ndarray:
    """fio_partition_weights: chi_l(xi) for l < W (indicator for overlap 0, smooth taper otherwise)."""
    out = np.empty(W, np.float64)
    _check(load_library().fio_partition_weights(int(W), float(overlap), int(xi1), int(xi2), _ptr(out)))
    return out


def assign_wedges(cost, nranks: int) -> np.ndarray:
    lib = load_library()
    cost = _f64(cost)
    owner = np.empty(cost.shape[0], np.int32)
    _check(lib.fio_assign_wedges(cost.shape[0], _ptr(cost), int(nranks), _ptr(owner)))
    return owner


def nccl_unique_id() -> bytes:
    """fio_nccl_unique_id: a fresh NCCL unique id (host only; the library loads libnccl.so.2)."""
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    _check(load_library().fio_nccl_unique_id(buf))
    return buf.raw


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0 of the torch.distributed group draws the id, every rank returns the same bytes.  This
    is the only collective the binding performs; the cross-GPU sum of the apply runs inside the
    library (fio_apply's NCCL reduce-scatter)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    if not isinstance(obj[0], (bytes, bytearray)) or len(obj[0]) != NCCL_ID_BYTES:
        raise FioError(-4, "NCCL id broadcast failed")
    return bytes(obj[0])


def row_slab(N: int, nranks: int, rank: int):
    """Rows [start, stop) of L f that rank `rank` receives from a communicator plan (include/fio.h)."""
    if N % nranks:
        raise FioError(-1, "nranks must divide N")
    rows = N // nranks
    return rank * rows, (rank + 1) * rows


class Plan:
    """fio_plan: preprocessing of Phi(x,xi) = x.xi + b(x).xi + sqrt(c1(x)^2 xi1^2 + c2(x)^2 xi2^2)
    and a(x,xi) = sum_k px[k](x) pxi[k](xi) at accuracy eps (include/fio.h)."""

    def __init__(self, N: int, c1, c2, b1=None, b2=None, px=None, pxi=None, eps: float = 1e-6,
                 dtype: str = "c128", n_wedges: int = 0, nufft_w: int = 0, nufft_beta: float = 0.0,
                 seed: int = 0x5EED, device: Optional[int] = None, rank: int = 0, nranks: int = 1,
                 r_init: int = 32, r_max: int = 512, certify: bool = True, rho_sign: int = 1,
                 amplitude: str = "separable", skeleton: bool = False, load: Optional[str] = None,
                 group=None, nccl_id: Optional[bytes] = None, wedge_overlap: float = 0.0,
                 paper_accept: bool = False, allgather: bool = False):
        import torch
        if not torch.cuda.is_available():
            raise FioError(-3, "no CUDA device: the FIO apply runs only on the GPU (no CPU fallback)")
        lib = load_library()
        self._lib = lib
        self.N = int(N)
        self.dtype = dtype
        self.c64 = dtype == "c64"
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        keep = [_f64(c1), _f64(c2), _f64(b1), _f64(b2)]
        for k in keep:
            if k is not None and k.size != N * N:
                raise FioError(-1, "phase arrays must have N*N entries")
        ph = _Phase(*[_ptr(k) for k in keep], -1 if rho_sign < 0 else 1)
        pxa, pxia = _c128(px), _c128(pxi)
        K = 0 if pxa is None else int(pxa.reshape(-1, N * N).shape[0])
        if amplitude not in ("separable", "bessel"):
            raise FioError(-1, "amplitude must be 'separable' or 'bessel'")
        amp = _Amp(K, _ptr(pxa), _ptr(pxia), 1 if amplitude == "bessel" else 0)
        o = _Opts()
        lib.fio_default_opts(ctypes.byref(o))
        o.dtype = FIO_C64 if self.c64 else FIO_C128
        o.n_wedges, o.nufft_w, o.nufft_beta, o.seed = int(n_wedges), int(nufft_w), float(nufft_beta), int(seed)
        o.device, o.rank, o.nranks = self.device, int(rank), int(nranks)
        o.r_init, o.r_max, o.certify = int(r_init), int(r_max), int(bool(certify))
        o.skeleton = int(bool(skeleton))
        o.wedge_overlap = float(wedge_overlap)
        o.paper_accept = int(bool(paper_accept))
        o.allgather = int(bool(allgather))  # with a communicator: the full N x N on every rank
        # wedge-sharded with a communicator: the id comes from rank 0 (broadcast over `group`, or given)
        if nranks > 1 and nccl_id is None and group is not None:
            nccl_id = broadcast_nccl_id(group)
        idbuf = None
        if nccl_id is not None:
            if len(nccl_id) != NCCL_ID_BYTES:
                raise FioError(-1, f"nccl_id must be {NCCL_ID_BYTES} bytes")
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), NCCL_ID_BYTES)
            o.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            if load is None:
                self.status = _check(lib.fio_plan(ctypes.byref(h), self.N, ctypes.byref(ph), ctypes.byref(amp),
                                                  float(eps), ctypes.byref(o)))
            else:  # reuse a saved separation (fio_plan_load): same operator, N, eps and options required
                self.status = _check(lib.fio_plan_load(ctypes.byref(h), os.fsencode(load), self.N, ctypes.byref(ph),
                                                       ctypes.byref(amp), float(eps), ctypes.byref(o)))
        self._h = h
        self.eps = eps
        self.rank, self.nranks = int(rank), int(nranks)
        self.torch_dtype = torch.complex64 if self.c64 else torch.complex128
        self.out_rows = self.info["out_rows"]  # N, or N / nranks with a communicator (row slab, no allgather)

    def save(self, path: str) -> None:
        """fio_plan_save: write this plan's separation (per wedge C, V S^-1, R, U_R^+) to path;
        Plan(..., load=path) rebuilds the identical plan without the randomized separation."""
        _check(self._lib.fio_plan_save(self._h, os.fsencode(path)))

    # ------------------------------------------------------------ evaluation
    def _dev_tensor(self, t, name, shape, writable=False):
        """Check a device operand against the plan: CUDA, plan dtype, exact shape, the plan's device;
        outputs must already be contiguous (the library writes through the raw pointer)."""
        if not (t.is_cuda and t.dtype == self.torch_dtype and tuple(t.shape) == tuple(shape)
                and t.device.index == self.device):
            raise FioError(-1, f"{name} must be a {self.torch_dtype} tensor of shape {tuple(shape)} on "
                               f"cuda:{self.device}")
        if writable and not t.is_contiguous():
            raise FioError(-1, f"{name} must be contiguous")
        return t if writable else t.contiguous()

    def _host_tensor(self, t, name, rows=None):
        """Check a host operand of apply_host: CPU, contiguous, plan dtype, exactly rows*N elements."""
        rows = self.N if rows is None else rows
        if t.is_cuda or t.dtype != self.torch_dtype or not t.is_contiguous() or t.numel() != rows * self.N:
            raise FioError(-1, f"{name} must be a contiguous CPU {self.torch_dtype} tensor of {rows}x{self.N} "
                               f"elements")
        return t

    def apply(self, f, out=None, stream=None):
        """Lf for a device tensor f (N x N, complex64/complex128 matching the plan dtype)."""
        import torch
        f = self._dev_tensor(f, "f", (self.N, self.N))
        if out is None:
            out = torch.empty((self.out_rows, self.N), dtype=f.dtype, device=f.device)
        out = self._dev_tensor(out, "out", (self.out_rows, self.N), writable=True)
        if stream is None:
            stream = torch.cuda.current_stream(f.device)
        _check(self._lib.fio_apply(self._h, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                   ctypes.c_void_p(stream.cuda_stream)))
        return out

    def apply_batch(self, f, out=None, stream=None):
        """L f_b for a device tensor f of shape (B, N, N) (plan dtype): one fio_apply_batch call."""
        import torch
        if f.dim() != 3 or f.shape[0] < 1:
            raise FioError(-1, f"f must have shape (B, {self.N}, {self.N})")
        f = self._dev_tensor(f, "f", (f.shape[0], self.N, self.N))
        if out is None:
            out = torch.empty((f.shape[0], self.out_rows, self.N), dtype=f.dtype, device=f.device)
        out = self._dev_tensor(out, "out", (f.shape[0], self.out_rows, self.N), writable=True)
        if stream is None:
            stream = torch.cuda.current_stream(f.device)
        _check(self._lib.fio_apply_batch(self._h, int(f.shape[0]), ctypes.c_void_p(f.data_ptr()),
                                         ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
        return out

    def apply_adjoint(self, g, out=None, stream=None):
        """L~* g for a device tensor g (N x N, plan dtype)."""
        import torch
        g = self._dev_tensor(g, "g", (self.N, self.N))
        if out is None:
            out = torch.empty((self.out_rows, self.N), dtype=g.dtype, device=g.device)
        out = self._dev_tensor(out, "out", (self.out_rows, self.N), writable=True)
        if stream is None:
            stream = torch.cuda.current_stream(g.device)
        _check(self._lib.fio_apply_adjoint(self._h, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                           ctypes.c_void_p(stream.cuda_stream)))
        return out

    def apply_host(self, f_host, out_host, stream=None):
        """End-to-end apply from host (pinned) tensors; copies in both directions inside the call."""
        import torch
        self._host_tensor(f_host, "f_host")
        self._host_tensor(out_host, "out_host", rows=self.out_rows)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        _check(self._lib.fio_apply_host(self._h, ctypes.c_void_p(f_host.data_ptr()),
                                        ctypes.c_void_p(out_host.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
        return out_host


    def apply_host_stream(self, f_host, out_host, stream=None):
        """L f_i for a stream of host (pinned) inputs f_host (count, N, N) into out_host (count, out_rows, N):
        one fio_apply_host_stream call; every copy happens inside it, pipelined with the applies."""
        import torch
        count = int(f_host.shape[0]) if f_host.dim() == 3 else -1
        if count < 0 or out_host.dim() != 3 or out_host.shape[0] != count:
            raise FioError(-1, "apply_host_stream: f_host (count, N, N) and out_host (count, out_rows, N)")
        if count and (f_host.is_cuda or f_host.dtype != self.torch_dtype or not f_host.is_contiguous()
                      or tuple(f_host.shape[1:]) != (self.N, self.N)):
            raise FioError(-1, f"f_host must be a contiguous CPU {self.torch_dtype} tensor (count, {self.N}, {self.N})")
        if count and (out_host.is_cuda or out_host.dtype != self.torch_dtype or not out_host.is_contiguous()
                      or tuple(out_host.shape[1:]) != (self.out_rows, self.N)):
            raise FioError(-1, f"out_host must be a contiguous CPU {self.torch_dtype} tensor "
                               f"(count, {self.out_rows}, {self.N})")
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        _check(self._lib.fio_apply_host_stream(self._h, count, ctypes.c_void_p(f_host.data_ptr()),
                                               ctypes.c_void_p(out_host.data_ptr()),
                                               ctypes.c_void_p(stream.cuda_stream)))
        return out_host

    def profile_begin(self, max_applies: int):
        """Record per-stage CUDA events for the next max_applies applies (on their stream)."""
        _check(self._lib.fio_profile_begin(self._h, int(max_applies)))

    def profile_end(self) -> dict:
        """Synchronize and return {stage: total ms} over the recorded applies, plus 'n'."""
        ms = np.zeros(len(STAGES), np.float64)
        n = ctypes.c_int(0)
        _check(self._lib.fio_profile_end(self._h, _ptr(ms), ctypes.byref(n)))
        out = {k: float(v) for k, v in zip(STAGES, ms)}
        out["n"] = n.value
        return out

    # ------------------------------------------------------------ introspection
    @property
    def info(self) -> dict:
        i = _Info()
        _check(self._lib.fio_plan_info(self._h, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in _Info._fields_}

    def wedges(self) -> dict:
        n = self.info["n_owned"]
        l, q, r = (np.zeros(n, np.int32) for _ in range(3))
        box, M = np.zeros((n, 4), np.int32), np.zeros((n, 4), np.int32)
        xc, err = np.zeros((n, 2), np.int32), np.zeros(n, np.float64)
        _check(self._lib.fio_plan_wedges(self._h, _ptr(l), _ptr(q), _ptr(box), _ptr(M), _ptr(xc), _ptr(r),
                                         _ptr(err)))
        return {"l": l, "q": q, "box": box[:, :2], "fine": box[:, 2:], "M": M.reshape(n, 2, 2), "xc": xc,
                "r": r, "sep_err": err}

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.fio_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
