"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

None of these compares the oracle with itself: every expected value is a
closed form of the paper (identity, FFT-multiply-iFFT propagator, lattice
shift), a library routine the definition reduces to (numpy FFT), an exact
invariant (Parseval, partition of unity, adjoint pairing, linearity) or a
printed/worked value (tests/golden/spec_examples.json).  Each test names the
mistake it would catch.
"""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as wl

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
rng = np.random.default_rng(1234)


def crandn(*shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def multiplier(N, m):
    """N * ifft2(m * fhat): (1/N) sum_xi e^{2 pi i x.xi} m(xi) fhat(xi) for a Fourier multiplier."""
    return lambda fhat: N * np.fft.ifft2(m * fhat)


# ------------------------------------------------------------------ DFT (eq. dft)
def test_dft_impulse_golden():
    g = GOLD["dft_impulse_N4"]
    f = np.zeros((g["N"], g["N"]), complex)
    f[0, 0] = 1
    np.testing.assert_allclose(oracle.dft2(f), g["value"], atol=1e-15)


def test_dft_constant_golden():
    g = GOLD["dft_constant_N8"]
    N = g["N"]
    fh = oracle.dft2(np.ones((N, N), complex))
    assert abs(fh[0, 0] - g["dc"]) < 1e-13
    fh[0, 0] = 0
    assert np.abs(fh).max() < 1e-13


@pytest.mark.parametrize("N", [6, 16, 30])
def test_dft_matches_library_fft_and_parseval(N):
    # catches: sign of the exponent, 1/N normalisation, transposed axes, index wrap
    f = crandn(N, N)
    fh = oracle.dft2(f)
    np.testing.assert_allclose(fh, np.fft.fft2(f) / N, atol=1e-12)
    assert abs(np.linalg.norm(fh) / np.linalg.norm(f) - 1) < 1e-13
    f2 = np.zeros((N, N), complex)
    f2[1, 0] = 1.0  # x = (1/N, 0): fhat(xi) = e^{-2 pi i xi1/N}/N depends on k1 only
    k = np.arange(N)
    np.testing.assert_allclose(oracle.dft2(f2)[:, 3], np.exp(-2j * np.pi * k / N) / N, atol=1e-14)


# ------------------------------------------------------------------ eq. dfio closed forms
@pytest.mark.parametrize("N", [8, 16, 22])
def test_identity_phase_is_inverse_dft(N):
    # Phi = x.xi makes L the inverse DFT, so L(f) = f
    f = crandn(N, N)
    np.testing.assert_allclose(oracle.fio(wl.identity_operator(N), f), f, atol=1e-12)


@pytest.mark.parametrize("c1,c2", [(0.7, 0.7), (0.3, 1.7)])
def test_constant_radii_is_fourier_multiplier(c1, c2):
    # PAPER.md:109-119 (c1 = c2 = c t is the wave propagator); c1 != c2 pins xi1 <-> axis 0
    N = 16
    f = crandn(N, N)
    fh = np.fft.fft2(f) / N
    xi1, xi2 = wl.freqs(N)
    m = np.exp(2j * np.pi * np.sqrt(c1 ** 2 * xi1 ** 2 + c2 ** 2 * xi2 ** 2))
    np.testing.assert_allclose(oracle.fio(wl.const_ellipse_operator(N, c1, c2), f),
                               multiplier(N, m)(fh), atol=1e-11)


def test_constant_shift_is_roll():
    # Phi = (x + d).xi, d = k/N: Lf[n] = f[n + k] exactly (reading R12)
    N = 16
    f = crandn(N, N)
    out = oracle.fio(wl.shift_operator(N, 3, -5), f)
    np.testing.assert_allclose(out, np.roll(f, (-3, 5), axis=(0, 1)), atol=1e-12)


def test_pointwise_shift_pins_spatial_indexing():
    # b(x) varies with x: Lf[n1,n2] = f[n1 + k1(n), n2 + k2(n)] -- catches a transposed or
    # mis-indexed spatial coefficient array
    N = 12
    f = crandn(N, N)
    n1, n2 = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    k1 = (n1 + 2 * n2) % 3 - 1
    k2 = (n1 * n2) % 5 - 2
    out = oracle.fio(wl.shift_operator(N, k1, k2), f)
    np.testing.assert_allclose(out, f[(n1 + k1) % N, (n2 + k2) % N], atol=1e-12)


def test_piecewise_radii_pins_c1_c2_indexing():
    # c1, c2 piecewise constant in x: at each x, Lf(x) is the constant-radius multiplier
    # with the radii of that x (the sum over xi is local in x) -- catches c1/c2 swapped,
    # a transposed c array, or a dropped square
    N = 16
    f = crandn(N, N)
    fh = np.fft.fft2(f) / N
    n1, n2 = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    ma = (n1 < 5)
    mb = ((n1 + 3 * n2) % 4 == 0)
    A1, B1, A2, B2 = 0.3, 1.1, 0.9, 0.45
    c1 = np.where(ma, A1, B1)
    c2 = np.where(mb, A2, B2)
    op = wl.Operator(N, c1, c2)
    xi1, xi2 = wl.freqs(N)
    exp_ = np.zeros((N, N), complex)
    for v1 in (A1, B1):
        for v2 in (A2, B2):
            P = multiplier(N, np.exp(2j * np.pi * np.sqrt(v1 ** 2 * xi1 ** 2 + v2 ** 2 * xi2 ** 2)))(fh)
            sel = (c1 == v1) & (c2 == v2)
            exp_[sel] = P[sel]
    np.testing.assert_allclose(oracle.fio(op, f), exp_, atol=1e-11)


def test_wave_amplitude_closed_form():
    # config 2's amplitude a = 1 + 0.1 cos(2 pi x1) xi1/|xi| with constant c: L = M0 + 0.1 cos(2 pi x1) M1
    # (a complex spatial factor is used so that a dropped conj/imag part shows)
    N = 16
    t = 0.1
    f = crandn(N, N)
    fh = np.fft.fft2(f) / N
    base = wl.wave_operator(N, t)
    c = 1.37 * t
    px = base.px.copy()
    px[1] = px[1] * np.exp(0.4j)
    op = wl.Operator(N, np.full((N, N), c), np.full((N, N), c), px=px, pxi=base.pxi)
    xi1, xi2 = wl.freqs(N)
    r = np.sqrt(xi1 ** 2 + xi2 ** 2)
    m0 = np.exp(2j * np.pi * c * r)
    ratio = np.where(r > 0, xi1 / np.where(r > 0, r, 1), 0)
    x1, _ = wl.grid(N)
    exp_ = multiplier(N, m0)(fh) + 0.1 * np.exp(0.4j) * np.cos(2 * np.pi * x1) * multiplier(N, m0 * ratio)(fh)
    np.testing.assert_allclose(oracle.fio(op, f), exp_, atol=1e-11)


def test_single_mode():
    # fhat = delta_{xi0}: (Lf)(x) = (1/N) a(x,xi0) e^{2 pi i Phi(x, xi0)} -- the GRT phase at
    # one frequency; checks the per-term phase reduction against numpy at large |xi|
    N = 32
    op = wl.grt_operator(N)
    fh = np.zeros((N, N), complex)
    xi0 = (-16, 11)
    fh[xi0[0] % N, xi0[1] % N] = 1.0
    x1, x2 = wl.grid(N)
    phi = x1 * xi0[0] + x2 * xi0[1] + np.sqrt(op.c1 ** 2 * xi0[0] ** 2 + op.c2 ** 2 * xi0[1] ** 2)
    np.testing.assert_allclose(oracle.fio(op, fhat=fh), np.exp(2j * np.pi * phi) / N, atol=1e-13)


# ------------------------------------------------------------------ invariants
def test_linearity_and_sampling_consistency():
    N = 16
    op = wl.grt_operator(N)
    f, g = crandn(N, N), crandn(N, N)
    a, b = 0.3 - 1.2j, 2.1
    Lf, Lg = oracle.fio(op, f), oracle.fio(op, g)
    np.testing.assert_allclose(oracle.fio(op, a * f + b * g), a * Lf + b * Lg, atol=1e-12)
    pts = wl.sample_points(N, 40, seed=3)
    # sampled mode must equal the full grid bit for bit (same sum order)
    assert np.array_equal(oracle.fio(op, f, pts=pts), Lf.ravel()[pts])


def test_partition_of_unity():
    # sum_l chi_l = 1: sum of per-wedge partial operators + DC = L
    N, W = 16, 8
    op = wl.grt_operator(N)
    f = crandn(N, N)
    full = oracle.fio(op, f)
    acc = oracle.fio(op, f, wedges=[], W=W, include_dc=True)
    parts = []
    for l in range(W):
        p = oracle.fio(op, f, wedges=[l], W=W, include_dc=False)
        parts.append(np.linalg.norm(p))
        acc = acc + p
    np.testing.assert_allclose(acc, full, atol=1e-12)
    assert min(parts) > 1e-3 * max(parts)


def test_adjoint_pairing():
    # <L f, g>_X = <fhat, widehat(L* g)>_Omega (DFT unitary)
    N = 12
    op = wl.wave_operator(N)
    f, g = crandn(N, N), crandn(N, N)
    lhs = np.vdot(g, oracle.fio(op, f))
    rhs = np.vdot(oracle.fio_adjoint_hat(op, g), oracle.dft2(f))
    assert abs(lhs - rhs) < 1e-11 * abs(lhs)


# ------------------------------------------------------------------ wedges
def test_wedge_golden_examples():
    g = GOLD["wedges_N64"]
    for xi1, xi2, l in g["members"]:
        assert oracle.wedge_of(g["W"], xi1, xi2) == l
    assert oracle.wedge_of(8, 0, 0) == -1


@pytest.mark.parametrize("N,W", [(16, 8), (64, 8), (32, 12)])
def test_wedge_membership_by_cross_products(N, W):
    # independent check of arg-interval membership with long-double boundary rays
    xi1, xi2 = wl.freqs(N)
    pi = np.longdouble(np.pi)
    count = np.zeros(W, int)
    for a, b in zip(xi1.ravel(), xi2.ravel()):
        l = oracle.wedge_of(W, int(a), int(b))
        if a == 0 and b == 0:
            assert l == -1
            continue
        count[l] += 1
        lo = (2 * l - 1) * pi / W
        hi = (2 * l + 1) * pi / W
        A, B = np.longdouble(a), np.longdouble(b)
        assert np.cos(lo) * B - np.sin(lo) * A >= 0
        assert np.cos(hi) * B - np.sin(hi) * A < 0
    assert count.sum() == N * N - 1 and count.min() > 0


# ------------------------------------------------------------------ NUDFT component oracle
def test_nudft_single_coefficient_and_uniform_targets():
    n1, n2 = 6, 10
    c = np.zeros((n1, n2), complex)
    c[1, 7] = 2 - 1j  # k = (1 - 3, 7 - 5) = (-2, 2)
    y = rng.random((50, 2)) * 3 - 1
    np.testing.assert_allclose(oracle.nudft2(c, y), (2 - 1j) * np.exp(2j * np.pi * (-2 * y[:, 0] + 2 * y[:, 1])),
                               atol=1e-13)
    # uniform targets y = j/n reduce to an (un-normalised) inverse FFT
    c = crandn(n1, n2)
    j1, j2 = np.meshgrid(np.arange(n1), np.arange(n2), indexing="ij")
    y = np.stack([j1.ravel() / n1, j2.ravel() / n2], axis=1)
    ref = np.fft.ifft2(np.fft.ifftshift(c)) * n1 * n2
    np.testing.assert_allclose(oracle.nudft2(c, y).reshape(n1, n2), ref, atol=1e-11)


# ------------------------------------------------------------------ workloads
def test_workload_radii_golden():
    g = GOLD["grt_radii"]
    N = 64
    op = wl.grt_operator(N)
    for x1, x2, c1, c2 in g["points"]:
        i, j = int(round(x1 * N)), int(round(x2 * N))
        assert abs(op.c1[i, j] - c1) < 1e-15 and abs(op.c2[i, j] - c2) < 1e-15
    p = wl.paper_ellipse_operator(N)
    assert abs(p.c1[0, 0] - GOLD["paper_radii_at_origin"]["r1"]) < 1e-15
    assert abs(p.c2[0, 0] - GOLD["paper_radii_at_origin"]["r2"]) < 1e-15


def test_workload_inputs_deterministic():
    a = wl.white_noise(32, 0)
    assert np.array_equal(a, wl.white_noise(32, 0)) and np.all(a.imag == 0)
    b = wl.white_noise(32, 0, "c64")
    assert np.array_equal(b.real.astype(np.float32).astype(np.float64), b.real)
    g = wl.gaussian_bumps(64, 0)
    assert g.shape == (64, 64) and np.abs(g).max() > 0.1
    p = wl.sample_points(1024, 4096, 1)
    assert len(np.unique(p)) == 4096 and np.all(np.diff(p) > 0)


# ------------------------------------------------------------------ Bessel amplitude (Appendix)
def circle_average_kernel(rho, nth=256):
    """(1/4 pi^2) int_0^{2 pi} e^{2 pi i rho cos th} d th by the trapezoid rule (spectrally accurate):
    the Appendix kernel (1/2 pi) J0(2 pi rho) obtained WITHOUT a Bessel routine."""
    th = 2 * np.pi * np.arange(nth) / nth
    rho = np.asarray(rho, float)
    return np.exp(2j * np.pi * rho[..., None] * np.cos(th)).mean(-1) * (2 * np.pi) / (4 * np.pi ** 2)


def test_bessel_pair_sums_to_circle_average():
    # Appendix: a_+ e^{2 pi i rho} + a_- e^{-2 pi i rho} = (1/2 pi) J0(2 pi rho), so L_+ + L_- is the
    # circle-average operator for every frequency with rho >= 1/2 (reading R22 clamps below 1/2).
    # catches: wrong Y0 sign, wrong e^{-+2 pi i rho} factor, wrong 1/4 pi, wrong J0 argument
    N = 24
    f = crandn(N, N)
    fh = np.fft.fft2(f) / N
    xi1, xi2 = wl.freqs(N)
    fh[np.hypot(xi1, xi2) < 3] = 0          # r >= 1/4 below: rho >= 3/4 on the support
    lp, lm = wl.bessel_grt_operator(N, +1), wl.bessel_grt_operator(N, -1)
    out = oracle.fio(lp, fhat=fh) + oracle.fio(lm, fhat=fh)
    x1, x2 = wl.grid(N)
    ref = np.zeros((N, N), complex)
    for i in range(N):
        for j in range(N):
            rho = lp.c1[i, j] * np.hypot(xi1, xi2)
            ker = circle_average_kernel(rho) * np.exp(2j * np.pi * (x1[i, j] * xi1 + x2[i, j] * xi2))
            ref[i, j] = (ker * fh).sum() / N
    np.testing.assert_allclose(out, ref, atol=1e-12 * np.abs(ref).max())


def test_bessel_single_mode_asymptotics():
    # f_hat = delta_xi0 with rho = r |xi0| large: a_+(rho) -> (1/4 pi) sqrt(1/(pi^2 rho)) e^{-i pi/4}
    # (H0^(1)(z) ~ sqrt(2/(pi z)) e^{i(z - pi/4)}); checks the sign of Y0 and of
    # the demodulating exponential separately from the pair identity
    N = 64
    op = wl.bessel_grt_operator(N, +1)
    fh = np.zeros((N, N), complex)
    xi0 = (24, -17)
    fh[xi0[0] % N, xi0[1] % N] = 1.0
    out = oracle.fio(op, fhat=fh)
    x1, x2 = wl.grid(N)
    rho = op.c1 * np.hypot(*xi0)
    amp = N * out * np.exp(-2j * np.pi * (x1 * xi0[0] + x2 * xi0[1] + rho))
    asym = np.exp(-1j * np.pi / 4) / (4 * np.pi * np.pi * np.sqrt(rho))
    assert np.max(np.abs(amp / asym - 1)) < 2e-2      # leading term, rho in [7, 30]
    om = wl.bessel_grt_operator(N, -1)
    out_m = oracle.fio(om, fhat=fh)
    amp_m = N * out_m * np.exp(-2j * np.pi * (x1 * xi0[0] + x2 * xi0[1] - rho))
    np.testing.assert_allclose(amp_m, np.conj(amp), rtol=1e-12)   # a_- = conj(a_+) for real rho


def test_bessel_dc_term_uses_clamped_radius():
    # reading R22: rho_e = max(rho, 1/2); at xi = 0 the pair sums to -(1/2 pi) J0(pi) / N
    N = 16
    fh = np.zeros((N, N), complex)
    fh[0, 0] = 1.0
    s = oracle.fio(wl.bessel_grt_operator(N, +1), fhat=fh) + oracle.fio(wl.bessel_grt_operator(N, -1), fhat=fh)
    np.testing.assert_allclose(s, -circle_average_kernel(0.5) / N * np.ones((N, N)), rtol=1e-12)


# ------------------------------------------------------------------ wedge-restricted mode
def wedge_by_cross_products(W, xi1, xi2):
    """The wedge of xi != 0 from the half-open arg interval [(2l-1) pi/W, (2l+1) pi/W),
    decided by the signs of long-double cross products with the two boundary rays -- no atan2."""
    pi = np.longdouble(np.pi)
    A, B = np.longdouble(xi1), np.longdouble(xi2)
    hits = [l for l in range(W)
            if np.cos((2 * l - 1) * pi / W) * B - np.sin((2 * l - 1) * pi / W) * A >= 0
            and np.cos((2 * l + 1) * pi / W) * B - np.sin((2 * l + 1) * pi / W) * A < 0]
    assert len(hits) == 1, (xi1, xi2, hits)
    return hits[0]


@pytest.mark.parametrize("xi0", [(-13, 5), (7, -11), (-16, -16), (3, 0), (-1, 9), (0, -7)])
def test_wedge_restricted_single_mode(xi0):
    # fhat = delta_{xi0}: the partial operator of the wedge that owns xi0 reproduces the single-mode
    # closed form (1/N) e^{2 pi i Phi(x, xi0)}; every other wedge gives exactly 0.
    # catches: a selection that classifies the raw FFT index (k1, k2) instead of the signed frequency
    # (xi1, xi2) -- every xi0 above has a negative component, whose raw index lies in another wedge --
    # a swapped axis in the classification, or an off-by-one wedge
    N, W = 32, 8
    op = wl.grt_operator(N)
    fh = np.zeros((N, N), complex)
    fh[xi0[0] % N, xi0[1] % N] = 1.0
    own = wedge_by_cross_products(W, *xi0)
    raw = wedge_by_cross_products(W, xi0[0] % N if xi0[0] % N else 0, xi0[1] % N if xi0[1] % N else 0) \
        if (xi0[0] % N, xi0[1] % N) != (0, 0) else None
    x1, x2 = wl.grid(N)
    phi = x1 * xi0[0] + x2 * xi0[1] + np.sqrt(op.c1 ** 2 * xi0[0] ** 2 + op.c2 ** 2 * xi0[1] ** 2)
    mode = np.exp(2j * np.pi * phi) / N
    for l in range(W):
        out = oracle.fio(op, fhat=fh, wedges=[l], W=W, include_dc=False)
        if l == own:
            np.testing.assert_allclose(out, mode, atol=1e-13)
        else:
            assert np.array_equal(out, np.zeros_like(out)), (l, own)
    if any(v < 0 for v in xi0):
        assert raw != own  # the case is discriminating: the raw-index wedge differs
    # the DC switch: xi = 0 is in no wedge and only include_dc brings it in
    fdc = np.zeros((N, N), complex)
    fdc[0, 0] = 2.0
    assert np.array_equal(oracle.fio(op, fhat=fdc, wedges=list(range(W)), W=W, include_dc=False),
                          np.zeros((N, N), complex))
    np.testing.assert_allclose(oracle.fio(op, fhat=fdc, wedges=[], W=W, include_dc=True),
                               np.full((N, N), 2.0 / N), atol=1e-15)


# ------------------------------------------------------------------ adjoint branches
def _pairing_ops(N):
    x1, x2 = wl.grid(N)
    grt = wl.grt_operator(N)
    neg = wl.Operator(N, grt.c1, grt.c2, sign=-1, name="grt-")                       # rho_sign = -1
    shifted = wl.Operator(N, grt.c1, grt.c2, b1=0.05 * np.sin(2 * np.pi * x2), b2=0.03 * np.cos(2 * np.pi * x1),
                          sign=-1, name="grt-b")                                       # b != 0
    wave = wl.wave_operator(N)
    px = wave.px.copy()
    px[1] = px[1] * np.exp(0.7j) * (1 + 0.3 * x2)                                     # complex spatial factor
    pxi = wave.pxi.copy()
    pxi[1] = pxi[1] * np.exp(-0.2j)                                                    # complex frequency factor
    amp = wl.Operator(N, wave.c1, wave.c2, b1=shifted.b1, px=px, pxi=pxi, name="wave-amp-b")
    return {"bessel+": wl.bessel_grt_operator(N, 1), "bessel-": wl.bessel_grt_operator(N, -1), "rho_sign-": neg,
            "b": shifted, "amp+b": amp}


@pytest.mark.parametrize("name", ["bessel+", "bessel-", "rho_sign-", "b", "amp+b"])
def test_adjoint_pairing_all_branches(name):
    # <L f, g>_X = <fhat, widehat(L* g)>_Omega for every branch of oracle_fio_adjoint_freq: the Bessel
    # amplitude with both signs, rho_sign = -1, b(x) != 0 and a complex separable amplitude.  The forward
    # branches are pinned by closed forms above (circle average, asymptotics, shifts, the wave amplitude),
    # so this pins the adjoint's conj(a) and e^{-2 pi i Phi} in each branch.  Random complex fhat covers
    # every frequency (DC included).
    N = 12
    op = _pairing_ops(N)[name]
    f, g = crandn(N, N), crandn(N, N)
    lhs = np.vdot(g, oracle.fio(op, f))
    rhs = np.vdot(oracle.fio_adjoint_hat(op, g), oracle.dft2(f))
    assert abs(lhs - rhs) < 1e-11 * abs(lhs), (lhs, rhs)
    # and the adjoint is not trivially consistent: conjugating the amplitude's sign breaks the pairing
    if name.startswith("bessel"):
        other = wl.bessel_grt_operator(N, -op.sign)
        bad = np.vdot(oracle.fio_adjoint_hat(other, g), oracle.dft2(f))
        assert abs(lhs - bad) > 1e-3 * abs(lhs)


# ------------------------------------------------------------------ smooth polar-wedge partition (reading R2)
@pytest.mark.parametrize("N,W,ov", [(64, 8, 0.25), (64, 16, 1.0), (40, 12, 0.5)])
def test_smooth_partition_of_unity(N, W, ov):
    # sum_l chi_l = 1 on Omega \ {0} (PAPER.md:236-238 needs only this), 0 <= chi <= 1, at most two
    # wedges overlap, and away from the tapers chi_l is the paper's indicator wedge
    chi = oracle.smooth_wedge_weights(N, W, ov)
    tot = chi.sum(0)
    tot[0, 0] = 1.0
    assert np.abs(tot - 1).max() < 1e-13  # rounding of the wrapped angle at the 0 / 2 pi seam
    assert chi.min() >= 0 and chi.max() <= 1
    assert (chi > 0).sum(0).max() <= 2
    xi1, xi2 = wl.freqs(N)
    th = np.arctan2(xi2, xi1)
    D = 2 * np.pi / W
    d = np.mod(th + D / 2, D)                  # angle above the last boundary ray
    far = (np.minimum(d, D - d) > 0.5 * ov * D + 1e-9)
    far[0, 0] = False
    for a, b in zip(*np.nonzero(far)):
        l = wedge_by_cross_products(W, int(xi1[a, b]), int(xi2[a, b]))
        assert chi[l, a, b] == 1.0 and chi[:, a, b].sum() == 1.0, (a, b, l)


def test_smooth_partition_boundary_center_and_rotation():
    # chi_l = 1/2 on the paper's boundary rays (2l +- 1) pi / W, 1 at the wedge centre, and
    # chi_l(theta) = chi_0(theta - 2 pi l / W) (rotation covariance)
    W, ov = 16, 0.3
    D = 2 * np.pi / W
    for l in range(W):
        assert abs(oracle.smooth_chi_angle(W, ov, l, (l - 0.5) * D) - 0.5) < 1e-15
        assert abs(oracle.smooth_chi_angle(W, ov, l, (l + 0.5) * D) - 0.5) < 1e-15
        assert oracle.smooth_chi_angle(W, ov, l, l * D) == 1.0
    th = np.linspace(-np.pi, np.pi, 2001)
    for l in (1, 5, 11):
        np.testing.assert_allclose(oracle.smooth_chi_angle(W, ov, l, th), oracle.smooth_chi_angle(W, ov, 0, th - l * D),
                                   atol=1e-14)


def test_smooth_step_is_smooth():
    # S is C-infinity: finite differences of S and S' are continuous across the taper edges and S'
    # vanishes at tau = +-1 (no kink where the taper meets the indicator)
    t = np.linspace(-1.5, 1.5, 30001)
    s = oracle._smooth_step(t)
    d1 = np.gradient(s, t)
    d2 = np.gradient(d1, t)
    assert np.abs(np.diff(d1)).max() < 1e-2 and np.abs(np.diff(d2)).max() < 0.5
    assert abs(d1[np.searchsorted(t, -1.0)]) < 1e-12 and abs(d1[np.searchsorted(t, 1.0)]) < 1e-12
    np.testing.assert_allclose(s + oracle._smooth_step(-t), 1.0, atol=1e-15)
