"""CPU FP64 oracle for arXiv math/0610051 -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (the `cpu_baseline` leg and
the `--impl reference` arm) may import this package.  The product
(paper_math_0610051_b200) never imports it and it never imports the product:
the two share no code.  The arithmetic lives in fio_oracle.c (plain C, FP64,
OpenMP over output points); this module only marshals numpy arrays.

Functions and the passages they restate:
  dft2            eq. (dft)
  fio             eq. (dfio) PAPER.md:165-168 (full grid or sampled points;
                  optionally restricted to a wedge set = sum of L_l);
                  phases Phi_+- (op.sign) and the Bessel amplitude of eq. ellipses_amp
                  (op.amp == "bessel")
  wedge_of        wedges W_l PAPER.md:210-217 (W wedges, reading R1)
  smooth_wedge_weights  the smooth polar-wedge partition chi_l of DESIGN.md reading R2 (numpy, from
                  its definition); sum_l chi_l = 1, so L_l f = fio(op, fhat=chi_l fhat)
  nudft2          the Fourier series of evaluation step 3, PAPER.md:1299-1311
  fio_adjoint_hat widehat(L* g)(xi)
  rel_l2          the error estimator of PAPER.md:1549-1555
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fio_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc -O2 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.oracle_dft2.argtypes = [ctypes.c_int, P, P]
        lib.oracle_wedge_of.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.oracle_wedge_of.restype = ctypes.c_int
        lib.oracle_fio_points.argtypes = [ctypes.c_int, P, P, P, P, ctypes.c_int, P, P, P, I64, P,
                                          ctypes.c_int, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_nudft2.argtypes = [ctypes.c_int, ctypes.c_int, P, I64, P, P]
        lib.oracle_fio_adjoint_freq.argtypes = [ctypes.c_int, P, P, P, P, ctypes.c_int, P, P, P, I64,
                                                P, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _amp_kind(op) -> int:
    return 1 if getattr(op, "amp", "separable") == "bessel" else 0


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def dft2(f: np.ndarray) -> np.ndarray:
    """fhat(xi) = (1/N) sum_x e^{-2 pi i x.xi} f(x) in FFT-natural order (eq. dft)."""
    f = _c(f, np.complex128)
    N = f.shape[0]
    out = np.empty_like(f)
    _load().oracle_dft2(N, _ptr(f), _ptr(out))
    return out


def wedge_of(W: int, xi1: int, xi2: int) -> int:
    return int(_load().oracle_wedge_of(int(W), int(xi1), int(xi2)))


def fio(op, f: Optional[np.ndarray] = None, pts: Optional[np.ndarray] = None,
        fhat: Optional[np.ndarray] = None, wedges: Optional[Sequence[int]] = None, W: int = 0,
        include_dc: bool = True) -> np.ndarray:
    """(Lf)(x) of eq. (dfio) at flat output indices pts (default: the whole grid, returned N x N).

    op: workloads.Operator.  wedges: restrict the xi-sum to the union of W_l, l in wedges
    (W wedges), plus xi = 0 iff include_dc."""
    N = op.N
    if fhat is None:
        fhat = dft2(f)
    fhat = _c(fhat, np.complex128)
    full = pts is None
    if full:
        pts = np.arange(N * N, dtype=np.int64)
    pts = _c(pts, np.int64)
    c1, c2 = _c(op.c1, np.float64), _c(op.c2, np.float64)
    b1 = None if op.b1 is None else _c(op.b1, np.float64)
    b2 = None if op.b2 is None else _c(op.b2, np.float64)
    K = op.K
    px = None if K == 0 else _c(op.px, np.complex128)
    pxi = None if K == 0 else _c(op.pxi, np.complex128)
    sel = None
    if wedges is not None:
        sel = np.zeros(W, dtype=np.int32)
        sel[list(wedges)] = 1
    out = np.empty(pts.shape[0], dtype=np.complex128)
    _load().oracle_fio_points(N, _ptr(c1), _ptr(c2), _ptr(b1), _ptr(b2), K, _ptr(px), _ptr(pxi),
                              _ptr(fhat), pts.shape[0], _ptr(pts), int(W), _ptr(sel),
                              int(bool(include_dc)), int(getattr(op, "sign", 1)), _amp_kind(op), _ptr(out))
    return out.reshape(N, N) if full else out


def fio_adjoint_hat(op, g: np.ndarray, fidx: Optional[np.ndarray] = None) -> np.ndarray:
    """widehat(L* g)(xi) at FFT-natural flat frequency indices."""
    N = op.N
    g = _c(g, np.complex128)
    full = fidx is None
    if full:
        fidx = np.arange(N * N, dtype=np.int64)
    fidx = _c(fidx, np.int64)
    c1, c2 = _c(op.c1, np.float64), _c(op.c2, np.float64)
    b1 = None if op.b1 is None else _c(op.b1, np.float64)
    b2 = None if op.b2 is None else _c(op.b2, np.float64)
    K = op.K
    px = None if K == 0 else _c(op.px, np.complex128)
    pxi = None if K == 0 else _c(op.pxi, np.complex128)
    out = np.empty(fidx.shape[0], dtype=np.complex128)
    _load().oracle_fio_adjoint_freq(N, _ptr(c1), _ptr(c2), _ptr(b1), _ptr(b2), K, _ptr(px),
                                    _ptr(pxi), _ptr(g), fidx.shape[0], _ptr(fidx),
                                    int(getattr(op, "sign", 1)), _amp_kind(op), _ptr(out))
    return out.reshape(N, N) if full else out


def _smooth_step(tau):
    """S(tau) = g(u) / (g(u) + g(1 - u)), u = (1 + tau)/2, g(u) = exp(-1/u) for u > 0 (else 0):
    0 for tau <= -1, 1 for tau >= 1, infinitely differentiable, S(tau) + S(-tau) = 1."""
    tau = np.asarray(tau, dtype=np.float64)
    u = np.clip(0.5 * (1.0 + tau), 0.0, 1.0)
    with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
        gu = np.where(u > 0, np.exp(-1.0 / np.where(u > 0, u, 1.0)), 0.0)
        gv = np.where(u < 1, np.exp(-1.0 / np.where(u < 1, 1.0 - u, 1.0)), 0.0)
        out = gu / (gu + gv)
    return np.where(tau <= -1, 0.0, np.where(tau >= 1, 1.0, out))


def smooth_chi_angle(W: int, overlap: float, l: int, theta):
    """chi_l at polar angle theta (reading R2): with D = 2 pi / W and the paper's boundary
    rays b_l = (l - 1/2) D, h = overlap D / 2,
        chi_l = S(((theta - b_l) mod 2 pi) / h) * (1 - S(((theta - b_{l+1}) mod 2 pi) / h)),
    angle differences taken in (-pi, pi]."""
    D = 2 * np.pi / W
    h = 0.5 * overlap * D

    def wrap(a):  # to (-pi, pi]
        a = np.mod(np.asarray(a, dtype=np.float64), 2 * np.pi)
        return np.where(a > np.pi, a - 2 * np.pi, a)
    return _smooth_step(wrap(theta - (l - 0.5) * D) / h) * (1.0 - _smooth_step(wrap(theta - (l + 0.5) * D) / h))


def smooth_wedge_weights(N: int, W: int, overlap: float) -> np.ndarray:
    """chi_l(xi) on Omega in FFT-natural order, shape (W, N, N); chi_l(0) = 0 (xi = 0 is the DC term)."""
    k = np.arange(N)
    k = np.where(k >= N // 2, k - N, k)
    xi1, xi2 = np.meshgrid(k, k, indexing="ij")
    th = np.arctan2(xi2.astype(np.float64), xi1.astype(np.float64))
    chi = np.stack([smooth_chi_angle(W, overlap, l, th) for l in range(W)])
    chi[:, 0, 0] = 0.0
    return chi


def nudft2(coeffs: np.ndarray, y: np.ndarray) -> np.ndarray:
    """F(y) = sum_{k in box} c_k e^{2 pi i y.k}, box k_a in [-n_a/2, n_a/2), coeffs[k1+n1/2, k2+n2/2]."""
    coeffs = _c(coeffs, np.complex128)
    y = _c(y, np.float64).reshape(-1, 2)
    out = np.empty(y.shape[0], dtype=np.complex128)
    n1, n2 = coeffs.shape
    _load().oracle_nudft2(n1, n2, _ptr(coeffs), y.shape[0], _ptr(y), _ptr(out))
    return out


def rel_l2(approx: np.ndarray, exact: np.ndarray) -> float:
    """sqrt(sum |Lf - L~f|^2 / sum |Lf|^2)."""
    a = np.asarray(approx, dtype=np.complex128).ravel()
    e = np.asarray(exact, dtype=np.complex128).ravel()
    den = np.sqrt(np.sum(np.abs(e) ** 2))
    return float(np.sqrt(np.sum(np.abs(a - e) ** 2)) / (den if den > 0 else 1.0))
