"""Seeded synthetic workloads for arXiv math/0610051 (the five BASELINE.json configs).

This module is shared by the CUDA path (tests, bench.py) and the CPU oracle
(oracle/).  It holds only INPUT generation -- the grids, the operator
coefficients sampled on the grid X, the input images f and the sampled output
points -- and none of the fast method's arithmetic (no wedges, no separation,
no NUFFT, no FIO sum).  Both sides consume the identical bytes produced here.

The operator family (the phase and amplitude are data on the grids):

    Phi(x, xi) = x.xi + b(x).xi + sqrt(c1(x)^2 xi1^2 + c2(x)^2 xi2^2)
    a(x, xi)   = sum_k px[k](x) * pxi[k](xi)          (K = 0  ->  a == 1)

x = (n1/N, n2/N), axis 0 of every spatial array is n1 <-> x1
(reading R14).  pxi arrays are in FFT-natural frequency order
(index k <-> xi = k - N[k >= N/2]).

Input recipe: numpy.random.default_rng(seed) (PCG64);
white noise = standard_normal((N, N)) float64; the complex64 configuration
rounds f to float32 first and both sides consume the rounded values.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

__all__ = [
    "Operator", "CONFIGS", "config", "grid", "freqs", "grt_operator", "wave_operator",
    "identity_operator", "const_ellipse_operator", "shift_operator", "paper_ellipse_operator",
    "white_noise", "gaussian_bumps", "sample_points", "make_operator", "make_input", "bessel_grt_operator",
]


@dataclasses.dataclass
class Operator:
    """Discrete FIO description on an N x N grid (all arrays float64 / complex128)."""

    N: int
    c1: np.ndarray
    c2: np.ndarray
    b1: Optional[np.ndarray] = None
    b2: Optional[np.ndarray] = None
    px: Optional[np.ndarray] = None   # (K, N, N) complex128, spatial factors
    pxi: Optional[np.ndarray] = None  # (K, N, N) complex128, frequency factors, FFT order
    name: str = ""
    sign: int = 1                     # Phi = x.xi + b.xi + sign * rho (Phi_+- of PAPER.md:1600-1603)
    amp: str = "separable"            # "separable" (px, pxi) or "bessel" (eq. ellipses_amp)

    @property
    def K(self) -> int:
        return 0 if self.px is None else int(self.px.shape[0])


# ---------------------------------------------------------------- the configs
# BASELINE.json "configs" (index 3 is run in two precisions).
CONFIGS = {
    "cfg0": dict(N=64, dtype="c128", eps=1e-6, phase="grt", input="white", seed=0),
    "cfg1": dict(N=256, dtype="c128", eps=1e-6, phase="grt", input="bumps", seed=0),
    "cfg2": dict(N=512, dtype="c128", eps=1e-6, phase="wave", input="white", seed=0),
    "cfg3_c64": dict(N=1024, dtype="c64", eps=1e-4, phase="grt", input="white", seed=0),
    "cfg3_c128": dict(N=1024, dtype="c128", eps=1e-6, phase="grt", input="white", seed=0),
    "cfg4": dict(N=2048, dtype="c128", eps=1e-6, phase="grt", input="white", seed=0),
}


def config(name: str) -> dict:
    c = dict(CONFIGS[name])
    c["name"] = name
    return c


# ---------------------------------------------------------------- grids
def grid(N: int):
    """x1, x2 arrays (N, N), x = (n1/N, n2/N)."""
    n = np.arange(N, dtype=np.float64) / N
    return np.meshgrid(n, n, indexing="ij")


def freqs(N: int):
    """xi1, xi2 integer arrays (N, N) in FFT-natural order."""
    k = np.arange(N)
    k = np.where(k >= N // 2, k - N, k)
    return np.meshgrid(k, k, indexing="ij")


# ---------------------------------------------------------------- operators
def grt_operator(N: int) -> Operator:
    """Generalized-Radon phase of BASELINE configs 0,1,3,4: c1 = (2 + sin2pi x1 sin2pi x2)/3,
    c2 = (2 + cos2pi x1 cos2pi x2)/3, a == 1."""
    x1, x2 = grid(N)
    c1 = (2.0 + np.sin(2 * np.pi * x1) * np.sin(2 * np.pi * x2)) / 3.0
    c2 = (2.0 + np.cos(2 * np.pi * x1) * np.cos(2 * np.pi * x2)) / 3.0
    return Operator(N, c1, c2, name="grt")


def wave_operator(N: int, t: float = 0.1) -> Operator:
    """Config 2: Phi = x.xi + c(x)|xi| t, c = 1 + 0.2 sin(2pi x1) cos(2pi x2);
    a = 1 + 0.1 cos(2pi x1) xi1/|xi|, a(x,0) = 1 -- a rank-2 separable amplitude."""
    x1, x2 = grid(N)
    c = (1.0 + 0.2 * np.sin(2 * np.pi * x1) * np.cos(2 * np.pi * x2)) * t
    xi1, xi2 = freqs(N)
    r = np.sqrt(xi1.astype(np.float64) ** 2 + xi2.astype(np.float64) ** 2)
    ratio = np.where(r > 0, xi1 / np.where(r > 0, r, 1.0), 0.0)
    px = np.stack([np.ones((N, N)), 0.1 * np.cos(2 * np.pi * x1)]).astype(np.complex128)
    pxi = np.stack([np.ones((N, N)), ratio]).astype(np.complex128)
    return Operator(N, c.copy(), c.copy(), px=px, pxi=pxi, name="wave")


def identity_operator(N: int) -> Operator:
    """Phi = x.xi, a = 1: L is the inverse of the DFT."""
    z = np.zeros((N, N))
    return Operator(N, z, z.copy(), name="identity")


def const_ellipse_operator(N: int, c1: float, c2: float) -> Operator:
    """Phi = x.xi + sqrt(c1^2 xi1^2 + c2^2 xi2^2), constant radii: a Fourier multiplier
    (the FFT-multiply-iFFT propagator of PAPER.md:109-119 when c1 = c2 = c t)."""
    return Operator(N, np.full((N, N), float(c1)), np.full((N, N), float(c2)),
                    name=f"const_ellipse({c1},{c2})")


def shift_operator(N: int, k1, k2) -> Operator:
    """Phi = (x + b(x)).xi with b = (k1/N, k2/N) (k1, k2 scalars or (N,N) integer arrays):
    Lf[n1, n2] = f[n1 + k1, n2 + k2] (indices mod N)."""
    z = np.zeros((N, N))
    b1 = np.broadcast_to(np.asarray(k1, dtype=np.float64) / N, (N, N)).copy()
    b2 = np.broadcast_to(np.asarray(k2, dtype=np.float64) / N, (N, N)).copy()
    return Operator(N, z, z.copy(), b1, b2, name="shift")


def paper_ellipse_operator(N: int) -> Operator:
    """The paper's own ellipse phase Phi_+ (eq. nrphase):
    r1 = (2+sin4pi x1)(2+sin4pi x2)/9, r2 = (2+cos4pi x1)(2+cos4pi x2)/9."""
    x1, x2 = grid(N)
    r1 = (2 + np.sin(4 * np.pi * x1)) * (2 + np.sin(4 * np.pi * x2)) / 9.0
    r2 = (2 + np.cos(4 * np.pi * x1)) * (2 + np.cos(4 * np.pi * x2)) / 9.0
    return Operator(N, r1, r2, name="paper_ellipse")


def bessel_grt_operator(N: int, sign: int = 1) -> Operator:
    """L_+ (sign = 1) or L_- of the circle-averaging GRT: Phi_+- = x.xi +- r(x)|xi|,
    r = (3 + sin 4pi x1)(3 + sin 4pi x2)/16 (eq. circlerad), amplitude a_+- of eq. ellipses_amp."""
    x1, x2 = grid(N)
    r = (3 + np.sin(4 * np.pi * x1)) * (3 + np.sin(4 * np.pi * x2)) / 16.0
    return Operator(N, r, r.copy(), name=f"bessel_grt{'+' if sign > 0 else '-'}", sign=int(sign), amp="bessel")


def make_operator(cfg: dict) -> Operator:
    N = cfg["N"]
    if cfg["phase"] == "grt":
        return grt_operator(N)
    if cfg["phase"] == "wave":
        return wave_operator(N)
    raise ValueError(cfg["phase"])


# ---------------------------------------------------------------- inputs
def white_noise(N: int, seed: int = 0, dtype: str = "c128") -> np.ndarray:
    """iid N(0,1) real image as complex128 (c64: rounded to float32 first)."""
    f = np.random.default_rng(seed).standard_normal((N, N))
    if dtype == "c64":
        f = f.astype(np.float32).astype(np.float64)
    return f.astype(np.complex128)


def gaussian_bumps(N: int, seed: int = 0, nbumps: int = 64, dtype: str = "c128") -> np.ndarray:
    """Config 1 input: sum of 64 isotropic periodic Gaussian bumps, centres U[0,1)^2,
    widths U[0.005, 0.02], amplitudes N(0,1) (draw order: centres, widths, amplitudes)."""
    rng = np.random.default_rng(seed)
    centres = rng.random((nbumps, 2))
    widths = rng.uniform(0.005, 0.02, nbumps)
    amps = rng.standard_normal(nbumps)
    x1, x2 = grid(N)
    f = np.zeros((N, N))
    for (cx, cy), s, a in zip(centres, widths, amps):
        d1 = x1 - cx
        d1 -= np.round(d1)
        d2 = x2 - cy
        d2 -= np.round(d2)
        f += a * np.exp(-(d1 * d1 + d2 * d2) / (2 * s * s))
    if dtype == "c64":
        f = f.astype(np.float32).astype(np.float64)
    return f.astype(np.complex128)


def make_input(cfg: dict) -> np.ndarray:
    N = cfg["N"]
    if cfg["input"] == "white":
        return white_noise(N, cfg.get("seed", 0), cfg["dtype"])
    if cfg["input"] == "bumps":
        return gaussian_bumps(N, cfg.get("seed", 0), dtype=cfg["dtype"])
    raise ValueError(cfg["input"])


def sample_points(N: int, n: int = 4096, seed: int = 1) -> np.ndarray:
    """Sorted distinct flat output indices n1*N + n2 (default_rng(seed).choice)."""
    n = min(n, N * N)
    return np.sort(np.random.default_rng(seed).choice(N * N, n, replace=False)).astype(np.int64)
