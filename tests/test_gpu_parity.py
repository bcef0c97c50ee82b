"""Parity of the CUDA path (through the C ABI of include/fio.h) against the CPU oracle.

Every expected value comes from oracle/ (direct summation of eq. dfio)
or from a closed form; the bar is relative l2 <= 10 eps (BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle
import workloads as wl

torch = pytest.importorskip("torch")
fio = pytest.importorskip("paper_math_0610051_b200")

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def make_plan(op, eps=1e-6, dtype="c128", **kw):
    return fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=eps, dtype=dtype, device=0,
                    rho_sign=op.sign, amplitude=op.amp, **kw)


def run(op, f, eps=1e-6, dtype="c128", **kw):
    plan = make_plan(op, eps, dtype, **kw)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    out = plan.apply(torch.from_numpy(f).to(DEV, tdt))
    torch.cuda.synchronize()
    return plan, out.cpu().numpy().astype(np.complex128)


def crandn(N, seed=7):
    r = np.random.default_rng(seed)
    return r.standard_normal((N, N)) + 1j * r.standard_normal((N, N))


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("N", [8, 16, 40, 64])
def test_identity_phase_returns_f(N):
    # Phi = x.xi -> L = inverse DFT, L f = f; separation rank is 1 per wedge
    f = crandn(N)
    plan, out = run(wl.identity_operator(N), f)
    assert np.all(plan.wedges()["q"] == 1)
    assert oracle.rel_l2(out, f) <= 1e-5


def test_integer_shift_is_roll():
    N = 64
    f = crandn(N)
    _, out = run(wl.shift_operator(N, 3, -5), f)
    assert oracle.rel_l2(out, np.roll(f, (-3, 5), axis=(0, 1))) <= 1e-5


def test_constant_radii_multiplier():
    # FFT-multiply-iFFT propagator (constant c1 != c2 pins the axis convention)
    N = 64
    f = crandn(N)
    op = wl.const_ellipse_operator(N, 0.3, 1.7)
    xi1, xi2 = wl.freqs(N)
    m = np.exp(2j * np.pi * np.sqrt(0.09 * xi1 ** 2 + 2.89 * xi2 ** 2))
    ref = N * np.fft.ifft2(m * np.fft.fft2(f) / N)
    _, out = run(op, f)
    assert oracle.rel_l2(out, ref) <= 1e-5


# ------------------------------------------------------------------ configs vs the oracle
def test_config0_full_grid_c128():
    cfg = wl.config("cfg0")
    op, f = wl.make_operator(cfg), wl.make_input(cfg)
    plan, out = run(op, f, eps=cfg["eps"])
    err = oracle.rel_l2(out, oracle.fio(op, f))
    assert err <= 10 * cfg["eps"], err
    sep = plan.wedges()["sep_err"]
    print("config0 sampled separation errors", sep, "end-to-end", err)
    assert plan.info["certified"] == 1, sep


def test_config0_c64():
    cfg = wl.config("cfg0")
    op = wl.make_operator(cfg)
    f = wl.white_noise(cfg["N"], 0, "c64")
    _, out = run(op, f, eps=1e-4, dtype="c64")
    err = oracle.rel_l2(out, oracle.fio(op, f))
    assert err <= 1e-3, err


def test_wave_amplitude_small():
    # config 2's family (variable c(x) and the rank-2 amplitude) at N = 64
    op = wl.wave_operator(64)
    f = wl.white_noise(64, 0)
    _, out = run(op, f)
    err = oracle.rel_l2(out, oracle.fio(op, f))
    assert err <= 1e-5, err


def test_config1_bumps_full_grid():
    cfg = wl.config("cfg1")
    op, f = wl.make_operator(cfg), wl.make_input(cfg)
    _, out = run(op, f, eps=cfg["eps"])
    err = oracle.rel_l2(out, oracle.fio(op, f))
    assert err <= 10 * cfg["eps"], err


def test_config2_wave_sampled():
    cfg = wl.config("cfg2")
    op, f = wl.make_operator(cfg), wl.make_input(cfg)
    _, out = run(op, f, eps=cfg["eps"])
    pts = wl.sample_points(op.N, 4096, 1)
    err = oracle.rel_l2(out.ravel()[pts], oracle.fio(op, f, pts=pts))
    assert err <= 10 * cfg["eps"], err


@pytest.mark.parametrize("name", ["cfg3_c64", "cfg3_c128"])
def test_config3_sampled(name):
    cfg = wl.config(name)
    op, f = wl.make_operator(cfg), wl.make_input(cfg)
    _, out = run(op, f, eps=cfg["eps"], dtype=cfg["dtype"])
    pts = wl.sample_points(op.N, 4096, 1)
    ref = oracle.fio(op, f, pts=pts)
    err, mx = _pointwise(out.ravel()[pts], ref)
    print(f"{name}: rel l2 {err:.3e}, max|err_i|/rms {mx:.3e}")
    assert err <= 10 * cfg["eps"] and mx <= 100 * cfg["eps"], (err, mx)


# ------------------------------------------------------------------ structure
def test_sharded_partials_sum_to_full():
    # L = sum_l L_l: the per-rank partials of a 3-way wedge sharding add up
    # to the 1-rank result, and rank r's partial equals the oracle restricted to its wedges
    N = 64
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 0)
    _, full = run(op, f)
    acc = np.zeros_like(full)
    for r in range(3):
        plan, part = run(op, f, rank=r, nranks=3)
        acc += part
        if r == 1:
            ws = plan.wedges()["l"]
            ref = oracle.fio(op, f, wedges=list(ws), W=plan.info["W"], include_dc=False)
            assert oracle.rel_l2(part, ref) <= 1e-5
    assert oracle.rel_l2(acc, full) <= 1e-12


def test_linearity_and_apply_host():
    N = 64
    op = wl.grt_operator(N)
    plan = fio.Plan(N, op.c1, op.c2, eps=1e-6, device=0)
    f, g = crandn(N, 1), crandn(N, 2)
    a, b = 0.3 - 1.1j, 2.0
    tf = lambda z: torch.from_numpy(z).to(DEV)
    Lf, Lg, Lh = (plan.apply(tf(z)).cpu().numpy() for z in (f, g, a * f + b * g))
    assert oracle.rel_l2(Lh, a * Lf + b * Lg) <= 1e-12
    hin = torch.from_numpy(f).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    plan.apply_host(hin, hout)
    assert np.array_equal(hout.numpy(), Lf)


@pytest.mark.parametrize("dtype,eps", [("c128", 1e-6), ("c64", 1e-4)])
def test_apply_host_stream_equals_apply(dtype, eps):
    # fio_apply_host_stream (pipelined copies, double-buffered staging): every result is fio_apply's,
    # bit for bit, for distinct inputs -- odd count so both staging buffers are reused and one is
    # left half-used; count 0 is a no-op
    N, count = 96, 5
    op = wl.grt_operator(N)
    plan = fio.Plan(N, op.c1, op.c2, eps=eps, dtype=dtype, device=0)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    fs = torch.stack([torch.from_numpy(crandn(N, 10 + i)).to(tdt) for i in range(count)]).pin_memory()
    outs = torch.full((count, N, N), float("nan"), dtype=tdt).pin_memory()
    plan.apply_host_stream(fs, outs)
    for i in range(count):
        assert torch.equal(outs[i], plan.apply(fs[i].to(DEV)).cpu()), i
    plan.apply_host_stream(fs[:0], outs[:0])
    with pytest.raises(fio.FioError):
        plan.apply_host_stream(fs, outs[:2])
    with pytest.raises(fio.FioError):
        plan.apply_host_stream(fs.to(torch.complex64 if dtype == "c128" else torch.complex128), outs)


def test_invalid_arguments():
    op = wl.grt_operator(64)
    with pytest.raises(fio.FioError):
        fio.Plan(64, op.c1, op.c2, eps=0.0, device=0)
    with pytest.raises(fio.FioError):
        fio.Plan(14, np.zeros(196), np.zeros(196), device=0)  # 14 = 2*7 is not 5-smooth
    with pytest.raises(fio.FioError):
        fio.Plan(64, op.c1, op.c2, rank=2, nranks=2, device=0)


@pytest.mark.slow
def test_config4_sampled():
    # N = 2048, complex128, eps = 1e-6: direct sum at 4096 seeded output points (BASELINE configs[4])
    cfg = wl.config("cfg4")
    op, f = wl.make_operator(cfg), wl.make_input(cfg)
    plan, out = run(op, f, eps=cfg["eps"])
    pts = wl.sample_points(op.N, 4096, 1)
    err, mx = _pointwise(out.ravel()[pts], oracle.fio(op, f, pts=pts))
    print("config4: W", plan.info["W"], "sum_q", plan.info["sum_q"], "plan s", plan.info["plan_seconds"], "err", err,
          "max|err_i|/rms", mx)
    assert err <= 10 * cfg["eps"] and mx <= 100 * cfg["eps"], (err, mx)


# ------------------------------------------------------------------ adjoint
def adjoint_ref(op, g):
    """(L* g)(x) = (1/N) sum_xi e^{2 pi i x.xi} widehat(L* g)(xi), the hat from the oracle."""
    return op.N * np.fft.ifft2(oracle.fio_adjoint_hat(op, g))


def run_adj(op, g, eps=1e-6, dtype="c128", **kw):
    plan = make_plan(op, eps, dtype, **kw)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    out = plan.apply_adjoint(torch.from_numpy(g).to(DEV, tdt))
    torch.cuda.synchronize()
    return plan, out.cpu().numpy().astype(np.complex128)


@pytest.mark.parametrize("name", ["grt", "wave"])
def test_adjoint_matches_oracle(name):
    N = 64
    op = wl.grt_operator(N) if name == "grt" else wl.wave_operator(N)
    g = crandn(N, 11)
    _, out = run_adj(op, g)
    err = oracle.rel_l2(out, adjoint_ref(op, g))
    assert err <= 1e-5, err


def test_adjoint_c64_and_identity():
    N = 64
    op = wl.grt_operator(N)
    g = crandn(N, 12).astype(np.complex64).astype(np.complex128)
    _, out = run_adj(op, g, eps=1e-4, dtype="c64")
    assert oracle.rel_l2(out, adjoint_ref(op, g)) <= 1e-3
    _, out = run_adj(wl.identity_operator(32), crandn(32, 13))
    assert oracle.rel_l2(out, crandn(32, 13)) <= 1e-5


def test_adjoint_pairing_is_exact():
    # <L~ f, g> = <f, L~* g>: the GPU adjoint is the conjugate transpose of the GPU forward
    N = 64
    op = wl.wave_operator(N)
    plan = fio.Plan(N, op.c1, op.c2, px=op.px, pxi=op.pxi, eps=1e-6, device=0)
    f, g = crandn(N, 21), crandn(N, 22)
    Lf = plan.apply(torch.from_numpy(f).to(DEV)).cpu().numpy()
    Lsg = plan.apply_adjoint(torch.from_numpy(g).to(DEV)).cpu().numpy()
    lhs, rhs = np.vdot(g, Lf), np.vdot(Lsg, f)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(f) * np.linalg.norm(g) * N, (lhs, rhs)


@pytest.mark.parametrize("N,W,dtype,tol", [(128, 32, "c128", 1e-12), (128, 32, "c64", 1e-5), (512, 0, "c128", 1e-12),
                                           (1024, 0, "c128", 1e-12), (1024, 0, "c64", 1e-5)])
def test_adjoint_pairing_dense_regions(N, W, dtype, tol):
    # the GRT map folds: at N >= 128 with W >= 32 whole warps of K3 groups share one anchor, the case
    # the segmented warp reduction of the spread must sum over all 32 lanes
    op = wl.grt_operator(N)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    plan = fio.Plan(N, op.c1, op.c2, eps=1e-6 if dtype == "c128" else 1e-4, dtype=dtype, device=0, n_wedges=W)
    f, g = crandn(N, 41), crandn(N, 42)
    Lf = plan.apply(torch.from_numpy(f).to(DEV, tdt)).cpu().numpy().astype(np.complex128)
    Lsg = plan.apply_adjoint(torch.from_numpy(g).to(DEV, tdt)).cpu().numpy().astype(np.complex128)
    if dtype == "c64":  # the GPU saw the rounded inputs
        f, g = f.astype(np.complex64).astype(np.complex128), g.astype(np.complex64).astype(np.complex128)
    lhs, rhs = np.vdot(g, Lf), np.vdot(Lsg, f)
    assert abs(lhs - rhs) <= tol * np.linalg.norm(f) * np.linalg.norm(g), (lhs, rhs)


def test_adjoint_sharded_partials():
    N = 64
    op = wl.grt_operator(N)
    g = crandn(N, 31)
    _, full = run_adj(op, g)
    acc = sum(run_adj(op, g, rank=r, nranks=2)[1] for r in range(2))
    assert oracle.rel_l2(acc, full) <= 1e-12


@pytest.mark.parametrize("N,dtype,eps", [(96, "c128", 1e-6), (120, "c64", 1e-4), (8, "c128", 1e-6), (30, "c128", 1e-6)])
def test_ragged_sizes_full_grid(N, dtype, eps):
    # non-power-of-2 grids (5-smooth N, ragged K3 chunks and FFT batches, W = 8 wedges
    # of a few cells at N = 8) against the direct sum
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 3, dtype)
    _, out = run(op, f, eps=eps, dtype=dtype)
    err = oracle.rel_l2(out, oracle.fio(op, f))
    assert err <= 10 * eps, err


# ------------------------------------------------------------------ Bessel-amplitude GRT pair (NEXT-4)
@pytest.mark.parametrize("sign", [1, -1])
def test_bessel_grt_full_grid(sign):
    # L_+- of PAPER.md:1591-1614 (circle radius eq. circlerad, amplitude eq. ellipses_amp)
    N = 64
    op = wl.bessel_grt_operator(N, sign)
    f = wl.white_noise(N, 5)
    plan, out = run(op, f)
    err = oracle.rel_l2(out, oracle.fio(op, f))
    assert err <= 1e-5, err


def test_bessel_grt_c64_and_adjoint():
    N = 128
    op = wl.bessel_grt_operator(N, -1)
    f = wl.white_noise(N, 6, "c64")
    _, out = run(op, f, eps=1e-4, dtype="c64")
    assert oracle.rel_l2(out, oracle.fio(op, f)) <= 1e-3
    g = crandn(64, 41)
    op64 = wl.bessel_grt_operator(64, 1)
    _, out = run_adj(op64, g)
    assert oracle.rel_l2(out, adjoint_ref(op64, g)) <= 1e-5


def test_bessel_grt_paper_table_replay():
    # loose pin against Table tbl:result_b: N = 64, eps = 10 N^-2 = 2.44e-3,
    # white noise -> the paper reports error 7.30e-4; our error must be of the same order (< 10 eps)
    N = 64
    eps = 10.0 / N ** 2
    op = wl.bessel_grt_operator(N, 1)
    f = wl.white_noise(N, 0)
    _, out = run(op, f, eps=eps)
    err = oracle.rel_l2(out, oracle.fio(op, f))
    print("bessel L+ N=64 eps=%.3g err=%.3g (paper 7.30e-4)" % (eps, err))
    assert err <= 2 * eps


# ------------------------------------------------------------------ separation (P3) vs dense SVD
def test_separation_rank_matches_dense_svd():
    # for each wedge the plan's q should be the eps-rank of the
    # residual kernel A_l(x, xi) = e^{2 pi i (rho - grad rho(x, xihat_l).xi)}, computed here by a
    # dense numpy SVD of the full N^2 x |W_l| matrix (no product or oracle code involved)
    N, eps = 32, 1e-6
    op = wl.grt_operator(N)
    plan = make_plan(op, eps)
    wd = plan.wedges()
    W = plan.info["W"]
    geo = fio.geometry(N, W)
    xi1, xi2 = wl.freqs(N)
    C1, C2 = op.c1.ravel(), op.c2.ravel()
    for l, q in zip(wd["l"], wd["q"]):
        m = geo["wedge_of"].ravel() == l
        a1, a2 = xi1.ravel()[m].astype(float), xi2.ravel()[m].astype(float)
        th = 2 * np.pi * l / W
        u1, u2 = np.cos(th), np.sin(th)
        den = np.sqrt(C1 ** 2 * u1 ** 2 + C2 ** 2 * u2 ** 2)
        g1, g2 = C1 ** 2 * u1 / den, C2 ** 2 * u2 / den
        rho = np.sqrt(np.outer(C1 ** 2, a1 ** 2) + np.outer(C2 ** 2, a2 ** 2))
        A = np.exp(2j * np.pi * (rho - np.outer(g1, a1) - np.outer(g2, a2)))
        s = np.linalg.svd(A, compute_uv=False)
        rank = int((s > eps * s[0]).sum())
        assert rank - 1 <= q <= rank + 8, (l, q, rank)
    assert np.all(wd["sep_err"] <= 10 * eps)


# ------------------------------------------------------------------ skeleton storage (NEXT-3)
@pytest.mark.parametrize("dtype,eps", [("c128", 1e-6), ("c64", 1e-4)])
def test_skeleton_storage_matches_stored_alpha(dtype, eps):
    # U = A_[C] V S^{-1} rebuilt per apply equals the stored alpha' (same seed);
    # storage drops from N^2 sum_q to O(r q) per wedge
    N = 64
    op = wl.wave_operator(N)
    f = wl.white_noise(N, 2, dtype)
    p_full, out_full = run(op, f, eps=eps, dtype=dtype)
    p_sk, out_sk = run(op, f, eps=eps, dtype=dtype, skeleton=True)
    tol = 1e-12 if dtype == "c128" else 1e-5
    assert oracle.rel_l2(out_sk, out_full) <= tol
    assert oracle.rel_l2(out_sk, oracle.fio(op, f)) <= 10 * eps
    i_full, i_sk = p_full.info, p_sk.info
    assert i_sk["skeleton_bytes"] > 0 and i_sk["skeleton_bytes"] < i_full["alpha_bytes"] / 20
    g = crandn(N, 51)
    if dtype == "c128":
        Lsg = p_sk.apply_adjoint(torch.from_numpy(g).to(DEV)).cpu().numpy()
        Lf = p_sk.apply(torch.from_numpy(f).to(DEV)).cpu().numpy()
        assert abs(np.vdot(g, Lf) - np.vdot(Lsg, f)) <= 1e-12 * np.linalg.norm(f) * np.linalg.norm(g) * N


# ------------------------------------------------------------------ multi-RHS (NEXT-2)
@pytest.mark.parametrize("skeleton", [False, True])
def test_apply_batch_equals_single_applies(skeleton):
    N = 64
    op = wl.grt_operator(N)
    plan = make_plan(op, 1e-6, skeleton=skeleton)
    fs = np.stack([crandn(N, 60 + b) for b in range(3)])
    out = plan.apply_batch(torch.from_numpy(fs).to(DEV)).cpu().numpy()
    for b in range(3):
        single = plan.apply(torch.from_numpy(fs[b]).to(DEV)).cpu().numpy()
        assert np.array_equal(out[b], single)
    assert oracle.rel_l2(out[1], oracle.fio(op, fs[1])) <= 1e-5
    out5 = plan.apply_batch(torch.from_numpy(np.concatenate([fs, fs[:2]])).to(DEV)).cpu().numpy()  # workspace grows
    assert np.array_equal(out5[4], out[1])


# ------------------------------------------------------------------ options and argument checking
@pytest.mark.parametrize("kw", [dict(n_wedges=16), dict(n_wedges=8, nufft_w=8), dict(r_init=16), dict(seed=7)])
def test_plan_options_keep_parity(kw):
    # L does not depend on W (sum chi_l = 1), the taps, the skeleton size or the seed
    N = 64
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 8)
    plan, out = run(op, f, **kw)
    assert oracle.rel_l2(out, oracle.fio(op, f)) <= 1e-5
    info = plan.info
    if "n_wedges" in kw:
        assert info["W"] == kw["n_wedges"]
    if "nufft_w" in kw:
        assert info["nufft_w"] == kw["nufft_w"]


def test_loose_eps_and_status():
    N = 32
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 9)
    plan, out = run(op, f, eps=0.05)
    assert plan.status in (fio.FIO_OK, fio.FIO_WNOTCERT)
    assert oracle.rel_l2(out, oracle.fio(op, f)) <= 0.5
    assert plan.info["nufft_w"] >= 4


def test_more_invalid_arguments():
    op = wl.grt_operator(64)
    with pytest.raises(fio.FioError):
        fio.Plan(64, op.c1, op.c2, amplitude="bogus", device=0)
    with pytest.raises(fio.FioError):
        fio.Plan(64, op.c1, op.c2, nufft_w=2, device=0)
    with pytest.raises(fio.FioError):
        fio.Plan(64, op.c1[:10], op.c2, device=0)
    plan = fio.Plan(64, op.c1, op.c2, eps=1e-4, device=0)
    with pytest.raises(fio.FioError):
        plan.apply(torch.zeros((64, 64), dtype=torch.complex64, device=DEV))   # wrong dtype
    with pytest.raises(fio.FioError):
        plan.apply(torch.zeros((32, 32), dtype=torch.complex128, device=DEV))  # wrong shape


# ------------------------------------------------------------------ determinism of the two-stream K3 schedule
@pytest.mark.parametrize("dtype,eps", [("c128", 1e-6), ("c64", 1e-4)])
def test_apply_is_deterministic(dtype, eps):
    # K3's wedges alternate between two streams with their own accumulators, each point is written by
    # one thread per wedge and the accumulators are added in a fixed order: repeated applies (and a
    # re-planned operator with the same seed) agree bit for bit (reading R20)
    N = 256
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 9, dtype)
    plan, ref = run(op, f, eps=eps, dtype=dtype)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    t = torch.from_numpy(f).to(DEV, tdt)
    for _ in range(3):
        assert np.array_equal(plan.apply(t).cpu().numpy().astype(np.complex128), ref)
    _, again = run(op, f, eps=eps, dtype=dtype)
    assert np.array_equal(again, ref)


def test_c64_storage_at_1e6():
    # FP32 arithmetic with the 1e-6 plan (w = 7 taps) still meets the 10 eps bar: FP32 rounding
    # (~1e-7 relative) stays below the separation / NUFFT error
    N = 256
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 4, "c64")
    _, out = run(op, f, eps=1e-6, dtype="c64")
    err = oracle.rel_l2(out, oracle.fio(op, f))
    assert err <= 1e-5, err


# ------------------------------------------------------------------ plan save / load (NEXT-3)
@pytest.mark.parametrize("dtype,skeleton", [("c128", False), ("c64", False), ("c128", True)])
def test_plan_save_load_roundtrip(tmp_path, dtype, skeleton):
    N = 128
    op = wl.grt_operator(N)
    eps = 1e-6 if dtype == "c128" else 1e-4
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    p1 = make_plan(op, eps, dtype, skeleton=skeleton)
    path = str(tmp_path / "plan.fio")
    p1.save(path)
    p2 = make_plan(op, eps, dtype, skeleton=skeleton, load=path)
    assert p2.info["sum_q"] == p1.info["sum_q"] and p2.info["W"] == p1.info["W"]
    f = torch.from_numpy(wl.white_noise(N, 5, dtype)).to(DEV, tdt)
    a, b = p1.apply(f), p2.apply(f)
    torch.cuda.synchronize()
    assert torch.equal(a, b)  # same factors, same kernels: bit-identical
    print("plan s", p1.info["plan_seconds"], "load s", p2.info["plan_seconds"])


def test_plan_load_rejects_other_operator(tmp_path):
    N = 64
    op = wl.grt_operator(N)
    p1 = make_plan(op)
    path = str(tmp_path / "plan.fio")
    p1.save(path)
    with pytest.raises(fio.FioError):
        make_plan(op, eps=1e-5, load=path)  # other eps
    with pytest.raises(fio.FioError):
        make_plan(wl.wave_operator(N), load=path)  # other phase (hash)


def test_apply_captures_into_cuda_graph():
    # the whole apply (K0..K3 on the caller's stream plus the plan's side stream, fork/join by events)
    # is capturable: replaying the graph reproduces the eager result bit for bit
    N = 128
    op = wl.grt_operator(N)
    plan = make_plan(op)
    f = torch.from_numpy(wl.white_noise(N, 6)).to(DEV)
    ref = plan.apply(f)
    out = torch.empty_like(f)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.apply(f, out=out)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.apply(f, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


# ------------------------------------------------------------------ argument checking of the binding and the file format
def _fnv1a(b: bytes) -> int:
    h = 1469598103934665603
    for c in b:
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def test_plan_load_rejects_corrupted_body(tmp_path):
    # a flipped byte fails the body checksum; a skeleton column rewritten to xi = 0 (in no wedge) with a
    # recomputed checksum fails the index validation -- FIO_EINVAL, never an out-of-bounds device read
    import struct
    N = 64
    op = wl.grt_operator(N)
    p1 = make_plan(op)
    path = str(tmp_path / "plan.fio")
    p1.save(path)
    raw = bytearray(open(path, "rb").read())
    HDR = 88  # magic[8], 9 x int32, pad, eps, es_beta, seed, input_hash, body_hash
    assert struct.unpack_from("<Q", raw, 80)[0] == _fnv1a(bytes(raw[HDR:]))
    bad = bytearray(raw)
    bad[HDR + 40] ^= 0x5A
    open(path, "wb").write(bad)
    with pytest.raises(fio.FioError):
        make_plan(op, load=path)
    bad = bytearray(raw)
    l, q, r, nc, nr = struct.unpack_from("<5i", bad, HDR)
    assert nc > 0
    struct.pack_into("<i", bad, HDR + 20 + 8, 0)  # first skeleton column -> flat index 0 (xi = 0)
    struct.pack_into("<Q", bad, 80, _fnv1a(bytes(bad[HDR:])))
    open(path, "wb").write(bad)
    with pytest.raises(fio.FioError):
        make_plan(op, load=path)
    open(path, "wb").write(raw)  # the untouched file still loads
    make_plan(op, load=path)


def test_binding_rejects_bad_operands():
    N = 64
    op = wl.grt_operator(N)
    plan = make_plan(op)
    f = torch.zeros((N, N), dtype=torch.complex128, device=DEV)
    with pytest.raises(fio.FioError):
        plan.apply(f, out=torch.empty((N, N), dtype=torch.complex64, device=DEV))      # out dtype
    with pytest.raises(fio.FioError):
        plan.apply(f, out=torch.empty((N, N // 2), dtype=torch.complex128, device=DEV))  # out shape
    with pytest.raises(fio.FioError):
        plan.apply(f, out=torch.empty((N, N), dtype=torch.complex128, device=DEV).t())   # non-contiguous out
    with pytest.raises(fio.FioError):
        plan.apply_adjoint(f, out=torch.empty((N, N), dtype=torch.complex64, device=DEV))
    with pytest.raises(fio.FioError):
        plan.apply_host(torch.zeros((N, N), dtype=torch.complex64), torch.zeros((N, N), dtype=torch.complex128))
    with pytest.raises(fio.FioError):
        plan.apply_host(torch.zeros((N, N - 1), dtype=torch.complex128), torch.zeros((N, N), dtype=torch.complex128))
    with pytest.raises(fio.FioError):  # overlapping f / out inside the library (one buffer, shifted view)
        buf = torch.zeros((2 * N, N), dtype=torch.complex128, device=DEV)
        plan.apply(buf[N // 2:N // 2 + N], out=buf[:N])
    # the caller's current device is left as it was
    before = torch.cuda.current_device()
    plan.apply(f)
    assert torch.cuda.current_device() == before


# ------------------------------------------------------------------ full-grid element-wise parity at the headline sizes
def _pointwise(out, ref):
    """(rel l2, max_i |err_i| / rms(ref)) over every output point."""
    rms = np.sqrt(np.mean(np.abs(ref) ** 2))
    return oracle.rel_l2(out, ref), float(np.abs(out - ref).max() / rms)


@pytest.mark.parametrize("N,dtype,eps", [(1024, "c128", 1e-6), (1024, "c64", 1e-4), (2048, "c128", 1e-6),
                                         (2048, "c64", 1e-4)])
def test_full_grid_pointwise_shift_field(N, dtype, eps):
    # Phi = (x + k(x)/N).xi with an integer field k(x): Lf[n] = f[n + k(n)] exactly (reading R12,
    # pinned on the oracle by test_pointwise_shift_pins_spatial_indexing) -- checked at EVERY output point
    # of the headline grids, so a fault confined to one K3 chunk or one wedge cannot hide
    n1, n2 = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    k1 = (n1 // 97 + 2 * (n2 // 131)) % 5 - 2
    k2 = ((n1 // 61) * (n2 // 83)) % 7 - 3
    op = wl.shift_operator(N, k1, k2)
    f = wl.white_noise(N, 11, dtype)
    plan, out = run(op, f, eps=eps, dtype=dtype)
    ref = f[(n1 + k1) % N, (n2 + k2) % N]
    rel, mx = _pointwise(out, ref)
    print(f"shift field N={N} {dtype}: rel l2 {rel:.3e}, max|err|/rms {mx:.3e}, sum_q {plan.info['sum_q']}")
    assert rel <= 10 * eps and mx <= 100 * eps, (rel, mx)


@pytest.mark.parametrize("N,dtype,eps", [(1024, "c128", 1e-6), (1024, "c64", 1e-4), (2048, "c128", 1e-6),
                                         (2048, "c64", 1e-4)])
def test_full_grid_pointwise_piecewise_radii(N, dtype, eps):
    # c1, c2 piecewise constant over x (4 regions): at every x, Lf(x) is the constant-radius Fourier
    # multiplier of that x's radii (pinned on the oracle by
    # test_piecewise_radii_pins_c1_c2_indexing).  The warped points x + grad rho(xihat_l) are genuinely
    # off-grid, so this exercises the whole NUFFT (K1, K2, K3) at every output point of the grid.
    n1, n2 = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    ma = ((n1 * 7) // N + (n2 * 5) // N) % 2 == 0
    mb = (n1 + 3 * n2) % 4 == 0
    A1, B1, A2, B2 = 0.3, 1.1, 0.9, 0.45
    c1 = np.where(ma, A1, B1)
    c2 = np.where(mb, A2, B2)
    op = wl.Operator(N, c1, c2)
    f = wl.white_noise(N, 12, dtype)
    plan, out = run(op, f, eps=eps, dtype=dtype)
    fh = np.fft.fft2(f) / N
    xi1, xi2 = wl.freqs(N)
    ref = np.zeros((N, N), complex)
    for v1 in (A1, B1):
        for v2 in (A2, B2):
            m = np.exp(2j * np.pi * np.sqrt(v1 ** 2 * xi1 ** 2 + v2 ** 2 * xi2 ** 2))
            sel = (c1 == v1) & (c2 == v2)
            ref[sel] = (N * np.fft.ifft2(m * fh))[sel]
    rel, mx = _pointwise(out, ref)
    print(f"piecewise radii N={N} {dtype}: rel l2 {rel:.3e}, max|err|/rms {mx:.3e}, sum_q {plan.info['sum_q']}")
    assert rel <= 10 * eps and mx <= 100 * eps, (rel, mx)


# ------------------------------------------------------------------ high-accuracy complex128
@pytest.mark.parametrize("N", [64, 256])
def test_high_accuracy_c128(N):
    # eps = 1e-8 and 1e-10: FP64 throughout (row and column weights, alpha', grids, accumulation), the
    # shifted-CholeskyQR3 separation below 1e-7 and up to 12 taps; full grid against the direct sum
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 21)
    ref = oracle.fio(op, f)
    for eps in (1e-8, 1e-10):
        plan, out = run(op, f, eps=eps)
        rel, mx = _pointwise(out, ref)
        info = plan.info
        print(f"N={N} eps={eps:g}: rel l2 {rel:.3e} max|err|/rms {mx:.3e} taps {info['nufft_w']} "
              f"sum_q {info['sum_q']} sep {info['max_sep_err']:.2e}")
        assert rel <= 10 * eps, (eps, rel)
        if eps >= 1e-8:  # at 1e-10 the sampled Frobenius error is ~10 eps: report only
            assert info["certified"] == 1


def test_eps_floors_are_rejected():
    op = wl.grt_operator(64)
    with pytest.raises(fio.FioError, match="floor"):
        make_plan(op, eps=1e-7, dtype="c64")
    with pytest.raises(fio.FioError, match="floor"):
        make_plan(op, eps=1e-12, dtype="c128")
    make_plan(op, eps=1e-6, dtype="c64")  # at the floors: accepted
    make_plan(op, eps=1e-11, dtype="c128")


# ------------------------------------------------------------------ smooth polar-wedge partition (reading R2)
@pytest.mark.parametrize("name,full", [("cfg0", True), ("cfg1", True), ("cfg2", False), ("cfg3_c64", False),
                                       ("cfg3_c128", False)])
def test_smooth_partition_configs(name, full):
    # sum_l chi_l = 1: the smooth taper changes the wedges, not L
    cfg = wl.config(name)
    op, f = wl.make_operator(cfg), wl.make_input(cfg)
    plan, out = run(op, f, eps=cfg["eps"], dtype=cfg["dtype"], wedge_overlap=0.25)
    assert plan.info["wedge_overlap"] == 0.25 and plan.info["members"] > op.N ** 2 - 1
    if full:
        ref, got = oracle.fio(op, f), out
    else:
        pts = wl.sample_points(op.N, 4096, 1)
        ref, got = oracle.fio(op, f, pts=pts), out.ravel()[pts]
    err, mx = _pointwise(got, ref)
    print(f"smooth {name}: rel l2 {err:.3e} max/rms {mx:.3e} sum_q {plan.info['sum_q']} "
          f"members {plan.info['members']} fine {plan.info['fine_elems']}")
    assert err <= 10 * cfg["eps"] and mx <= 100 * cfg["eps"], (err, mx)


def test_smooth_partition_partials_and_adjoint():
    # rank r's partial is L applied to (sum of its chi_l) fhat -- the oracle with its own chi -- and the
    # adjoint (whose K1* now accumulates the two wedges sharing a frequency) stays the exact transpose
    N, ov = 64, 0.5
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 0)
    fh = oracle.dft2(f)
    chi = oracle.smooth_wedge_weights(N, 16, ov)
    plan, part = run(op, f, rank=1, nranks=3, n_wedges=16, wedge_overlap=ov)
    ws = plan.wedges()["l"]
    ref = oracle.fio(op, fhat=fh * chi[list(ws)].sum(0))
    assert oracle.rel_l2(part, ref) <= 1e-5
    full = make_plan(op, n_wedges=16, wedge_overlap=ov)
    a, b = crandn(N, 71), crandn(N, 72)
    La = full.apply(torch.from_numpy(a).to(DEV)).cpu().numpy()
    Lsb = full.apply_adjoint(torch.from_numpy(b).to(DEV)).cpu().numpy()
    assert abs(np.vdot(b, La) - np.vdot(Lsb, a)) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(b) * N
    assert oracle.rel_l2(Lsb, adjoint_ref(op, b)) <= 1e-5


# ------------------------------------------------------------------ the paper's own experiment (Table tbl:result_a)
@pytest.mark.parametrize("N", [64, 128])
def test_paper_table_result_a_replay(N):
    # PAPER.md:1440-1458 (eq. nrphase: ellipse radii r1, r2), white noise, eps = 10 N^-2, error measured on
    # the full grid against the direct sum; the paper prints (Table tbl:result_a) the
    # errors 2.08e-3 (N = 64) and 8.02e-4 (N = 128) for its own Matlab run -- a loose pin: ours must be
    # of the same order and inside the 10 eps bar
    import json
    import os
    rows = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))[
        "paper_table_result_a"]["rows"]
    paper = {int(r[0]): (r[1], r[2]) for r in rows}
    eps, printed = paper[N]
    assert abs(eps - 10.0 / N ** 2) < 1e-3 * eps
    op = wl.paper_ellipse_operator(N)
    f = wl.white_noise(N, 0)
    plan, out = run(op, f, eps=eps)
    err = oracle.rel_l2(out, oracle.fio(op, f))
    print(f"Table tbl:result_a replay N={N}: eps {eps:.3g}, error {err:.3g} (paper {printed:.3g}), "
          f"W {plan.info['W']} sum_q {plan.info['sum_q']}")
    assert err <= 10 * eps and printed / 20 <= err <= 5 * printed, (err, printed)


# ------------------------------------------------------------------ the NUFFT alone (K1 -> K2 -> K3) against the direct NUDFT
@pytest.mark.parametrize("N,dtype,eps,npts", [(128, "c128", 1e-6, None), (128, "c64", 1e-4, None),
                                              (1024, "c128", 1e-6, 2048), (1024, "c64", 1e-4, 2048)])
def test_nufft_component_vs_direct_nudft(N, dtype, eps, npts):
    # "The only step that requires attention" (section 3.4): the nonuniform Fourier
    # series of evaluation step 3 at the warped points.  A phase linear in xi, Phi = (x + b(x)).xi with a
    # real, non-integer displacement b, has a residual identically 1 (separation rank 1 in every wedge,
    # PAPER.md:1283-1302), so the apply IS the wedge-split NUFFT: Lf(x) = (1/N) sum_xi fhat(xi)
    # e^{2 pi i (x + b(x)).xi}, compared here with oracle.nudft2 (direct sum, pinned in
    # test_oracle_pins.py) at arbitrary off-grid targets y = x + b(x) -- every tap of K3's window, the
    # box maps M and the deconvolution folded into beta' are exercised without the separation.
    n1, n2 = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    r = np.random.default_rng(5)
    b1 = 0.2 * np.sin(2 * np.pi * n2 / N) + r.uniform(-2.5, 2.5, (N, N)) / N
    b2 = 0.15 * np.cos(2 * np.pi * n1 / N) + r.uniform(-2.5, 2.5, (N, N)) / N
    z = np.zeros((N, N))
    op = wl.Operator(N, z, z.copy(), b1, b2, name="warp-only")
    f = wl.white_noise(N, 13, dtype)
    plan, out = run(op, f, eps=eps, dtype=dtype)
    assert np.all(plan.wedges()["q"] == 1)
    idx = np.arange(N * N) if npts is None else wl.sample_points(N, npts, seed=3)
    p1, p2 = idx // N, idx % N
    y = np.stack([p1 / N + b1[p1, p2], p2 / N + b2[p1, p2]], axis=1)
    fh = np.fft.fftshift(oracle.dft2(f))   # box [-N/2, N/2)^2 in nudft2's centred layout
    ref = oracle.nudft2(fh, y) / N
    rel, mx = _pointwise(out.ravel()[idx], ref)
    print(f"NUFFT component N={N} {dtype}: rel l2 {rel:.3e}, max|err|/rms {mx:.3e}, w {plan.info['nufft_w']}")
    assert rel <= 10 * eps and mx <= 100 * eps, (rel, mx)


# ------------------------------------------------------------------ the paper's acceptance rule
@pytest.mark.parametrize("name", ["cfg0"])
def test_paper_acceptance_rule(name):
    # opts.paper_accept = 1: r uniform columns, r doubled until q <= r/3 (the paper's column step and test,
    # PAPER.md:1136-1143, 1213-1221) instead of pivoted columns accepted at q <= 3r/4 (reading R8).  The
    # operator is the same and parity must hold; the measured difference (printed, R8) is that
    # uniform columns find a smaller numerical rank q for the same eps -- a uniform sample misses
    # directions the pivoting picks up -- at many times the plan time.  (Config 1, measured once and
    # recorded in profiles/r02_paper_accept.txt: sum_q 325 vs 420, sampled separation error 2e-3, rel l2
    # 1.3e-5 > 10 eps after 223 s of planning -- why the default departs from the paper, reading R8.)
    cfg = wl.config(name)
    op, f = wl.make_operator(cfg), wl.make_input(cfg)
    base = make_plan(op, cfg["eps"])
    plan, out = run(op, f, eps=cfg["eps"], paper_accept=True)
    wd, wb = plan.wedges(), base.wedges()
    err = oracle.rel_l2(out, oracle.fio(op, f))
    print(f"{name} paper rule: sum_q {plan.info['sum_q']} (default {base.info['sum_q']}), mean r "
          f"{wd['r'].mean():.1f} (default {wb['r'].mean():.1f}), plan {plan.info['plan_seconds']:.2f} s "
          f"(default {base.info['plan_seconds']:.2f} s), rel l2 {err:.3e}, max sep err {wd['sep_err'].max():.2e}")
    assert err <= 10 * cfg["eps"], err
    nmem = np.bincount(fio.geometry(op.N, plan.info["W"])["wedge_of"].ravel() + 1,
                       minlength=plan.info["W"] + 1)[1:][wd["l"]]
    assert np.all((3 * wd["q"] <= wd["r"]) | (wd["r"] >= np.minimum(512, nmem))), (wd["q"], wd["r"])


# ------------------------------------------------------------------ the maximum size (reading R21: N <= 4096)
@pytest.mark.parametrize("dtype,eps", [("c64", 1e-4), ("c128", 1e-6)])
def test_max_size_shift_field_pointwise(dtype, eps):
    # N = 4096, the largest grid the library accepts: the pointwise integer-shift field (exact reference
    # Lf[n] = f[n + k(n)], reading R12) compared at all 16.8 M output points, W = 128 wedges
    N = 4096
    n1, n2 = np.meshgrid(np.arange(N, dtype=np.int64), np.arange(N, dtype=np.int64), indexing="ij")
    k1 = (n1 // 389 + 2 * (n2 // 523)) % 5 - 2
    k2 = ((n1 // 241) * (n2 // 331)) % 7 - 3
    op = wl.shift_operator(N, k1, k2)
    f = wl.white_noise(N, 17, dtype)
    plan, out = run(op, f, eps=eps, dtype=dtype)
    ref = f[(n1 + k1) % N, (n2 + k2) % N]
    rel, mx = _pointwise(out, ref)
    print(f"max size N={N} {dtype}: W {plan.info['W']}, rel l2 {rel:.3e}, max|err|/rms {mx:.3e}")
    assert rel <= 10 * eps and mx <= 100 * eps, (rel, mx)


@pytest.mark.slow
def test_max_size_grt_c64_sampled():
    # N = 4096 generalized-Radon phase (BASELINE configs[0] family), complex64 at eps = 1e-4: the largest
    # plan that fits one B200 (alpha' ~123 GB resident), checked against the direct sum at 256 seeded points
    N, eps = 4096, 1e-4
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 0, "c64")
    plan, out = run(op, f, eps=eps, dtype="c64")
    pts = wl.sample_points(N, 256, 1)
    ref = oracle.fio(op, f, pts=pts)
    rel, mx = _pointwise(out.ravel()[pts], ref)
    print(f"max size GRT N={N} c64: W {plan.info['W']}, sum_q {plan.info['sum_q']}, alpha "
          f"{plan.info['alpha_bytes'] / 1e9:.1f} GB, plan {plan.info['plan_seconds']:.1f} s, rel l2 {rel:.3e}, "
          f"max|err|/rms {mx:.3e}")
    assert rel <= 10 * eps and mx <= 100 * eps, (rel, mx)


# ------------------------------------------------------------------ distinct handles are independent (include/fio.h)
def test_concurrent_handles_on_threads():
    # two plans (different operators and dtypes) applied concurrently from two host threads, each on its
    # own CUDA stream: every result equals the same plan's serial apply bit for bit (no process-wide
    # launch state, per-handle workspaces; DESIGN.md section 2 "Device state")
    import threading
    N = 256
    jobs = [(wl.grt_operator(N), wl.white_noise(N, 21, "c128"), "c128", 1e-6),
            (wl.wave_operator(N), wl.white_noise(N, 22, "c64"), "c64", 1e-4)]
    plans, refs, ins = [], [], []
    for op, f, dt, eps in jobs:
        p, r = run(op, f, eps=eps, dtype=dt)
        plans.append(p)
        refs.append(r)
        ins.append(torch.from_numpy(f).to(DEV, torch.complex64 if dt == "c64" else torch.complex128))
    results = [[], []]
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream(device=DEV)
            with torch.cuda.stream(s):
                for _ in range(8):
                    out = plans[i].apply(ins[i], stream=s)
                    s.synchronize()
                    results[i].append(out.cpu().numpy().astype(np.complex128))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for i in range(2):
        assert len(results[i]) == 8
        for r in results[i]:
            assert np.array_equal(r, refs[i])


# ------------------------------------------------------------------ randomized operators (seeded fuzz over the plan's parameter space)
def _random_operator(seed):
    """A seeded random member of the phase/amplitude family of include/fio.h: smooth random radii fields
    c1, c2 (trigonometric polynomials of degree <= 2, values in [0.15, 1.4]), a smooth displacement b,
    the sign of rho, and a random separable amplitude of rank 0-2 (pxi_k: 1, xi1/|xi| or xi2/|xi|)."""
    r = np.random.default_rng(1000 + seed)
    N = int(r.choice([8, 10, 12, 16, 18, 20, 24, 30, 32, 40, 48, 50, 60, 64, 72, 80, 90, 96, 100, 120, 128]))
    x1, x2 = wl.grid(N)

    def smooth(lo, hi):
        v = np.zeros((N, N))
        for m in range(3):
            for n in range(3):
                v += r.normal() * np.cos(2 * np.pi * (m * x1 + n * x2) + r.uniform(0, 2 * np.pi)) / (1 + m + n)
        v = (v - v.min()) / max(v.max() - v.min(), 1e-12)
        return lo + (hi - lo) * v

    c1 = smooth(r.uniform(0.15, 0.6), r.uniform(0.7, 1.4))
    c2 = smooth(r.uniform(0.15, 0.6), r.uniform(0.7, 1.4))
    b1 = b2 = None
    if r.random() < 0.5:
        b1, b2 = smooth(-0.05, 0.05), smooth(-0.05, 0.05)
    K = int(r.integers(0, 3))
    px = pxi = None
    if K:
        xi1, xi2 = wl.freqs(N)
        rad = np.sqrt(xi1.astype(float) ** 2 + xi2.astype(float) ** 2)
        choices = [np.ones((N, N)), np.where(rad > 0, xi1 / np.where(rad > 0, rad, 1), 0.0),
                   np.where(rad > 0, xi2 / np.where(rad > 0, rad, 1), 0.0)]
        px = np.stack([smooth(0.2, 1.0) * np.exp(1j * smooth(0, 1)) for _ in range(K)]).astype(np.complex128)
        pxi = np.stack([choices[int(r.integers(0, 3))] for _ in range(K)]).astype(np.complex128)
    sign = int(r.choice([1, -1]))
    op = wl.Operator(N, c1, c2, b1, b2, px, pxi, name=f"random{seed}", sign=sign)
    dtype = "c64" if r.random() < 0.35 else "c128"
    eps = float(r.choice([1e-4, 1e-5])) if dtype == "c64" else float(r.choice([1e-5, 1e-6, 1e-7, 1e-8]))
    kw = {}
    if r.random() < 0.4:
        kw["n_wedges"] = int(8 * r.integers(1, 5))
    if r.random() < 0.3:
        kw["wedge_overlap"] = 0.25
    return op, dtype, eps, kw, int(r.integers(0, 1 << 30))


@pytest.mark.parametrize("seed", range(16))
def test_randomized_operators_full_grid(seed):
    # every output point against the direct sum (eq. dfio) for a seeded random operator: grid size (even,
    # 5-smooth, 8..128), radii fields, displacement, rho sign, separable amplitude rank, dtype, eps,
    # wedge count and partition all drawn from the seed -- parity must not depend on a lucky configuration
    op, dtype, eps, kw, fseed = _random_operator(seed)
    f = wl.white_noise(op.N, fseed % 997, dtype)
    plan, out = run(op, f, eps=eps, dtype=dtype, **kw)
    ref = oracle.fio(op, f)
    rel, mx = _pointwise(out, ref)
    print(f"random{seed}: N={op.N} {dtype} eps={eps:g} sign={op.sign} K={op.K} b={'yes' if op.b1 is not None else 'no'} "
          f"{kw} W={plan.info['W']} sum_q={plan.info['sum_q']}: rel l2 {rel:.3e}, max|err|/rms {mx:.3e}")
    assert rel <= 10 * eps and mx <= _pointwise_bar(op.N, eps, kw), (rel, mx)


def _pointwise_bar(N, eps, kw):
    # the l2 bar (10 eps, BASELINE north_star) always holds; the pointwise bar 100 eps is asserted at the
    # default wedge count (reading R1).  A user-forced count below it widens the wedges past the aperture
    # the separation-rank bound assumes: measured, l2 stays < 10 eps while the worst
    # point reaches ~200 eps (N = 160, W = 8 instead of 24) -- there only gross faults (1000 eps) fail
    default_w = max(8, 8 * int(np.floor(2 * np.sqrt(N) / 8 + 0.5)))
    return (1000 if kw.get("n_wedges", default_w) < default_w else 100) * eps


@pytest.mark.parametrize("seed", range(8))
def test_randomized_operators_large_sampled(seed):
    # the same seeded family at N in {160 .. 512} (W up to 48), plus the Bessel GRT amplitude on random radii;
    # 2048 sampled output points against the direct sum
    r = np.random.default_rng(5000 + seed)
    op, dtype, eps, kw, fseed = _random_operator(100 + seed)
    N = int(r.choice([160, 192, 200, 240, 250, 256, 288, 300, 320, 360, 384, 400, 432, 450, 480, 500, 512]))
    x1, x2 = wl.grid(N)
    # resample the small operator's smooth fields on the larger grid (same trigonometric family)
    rr = np.random.default_rng(7000 + seed)
    def smooth(lo, hi):
        v = np.zeros((N, N))
        for m in range(3):
            for n in range(3):
                v += rr.normal() * np.cos(2 * np.pi * (m * x1 + n * x2) + rr.uniform(0, 2 * np.pi)) / (1 + m + n)
        v = (v - v.min()) / max(v.max() - v.min(), 1e-12)
        return lo + (hi - lo) * v
    c1, c2 = smooth(0.2, 1.2), smooth(0.2, 1.2)
    amp = "bessel" if seed % 4 == 3 else "separable"
    if amp == "bessel":
        c2 = c1.copy()  # the circle GRT pair has equal radii
    opL = wl.Operator(N, c1, c2, name=f"random_large{seed}", sign=op.sign, amp=amp)
    f = wl.white_noise(N, fseed % 997, dtype)
    plan, out = run(opL, f, eps=eps, dtype=dtype, **kw)
    pts = wl.sample_points(N, 2048, 2 + seed)
    ref = oracle.fio(opL, f, pts=pts)
    rel, mx = _pointwise(out.ravel()[pts], ref)
    print(f"random_large{seed}: N={N} {dtype} eps={eps:g} sign={opL.sign} amp={amp} {kw} W={plan.info['W']} "
          f"sum_q={plan.info['sum_q']}: rel l2 {rel:.3e}, max|err|/rms {mx:.3e}")
    assert rel <= 10 * eps and mx <= _pointwise_bar(N, eps, kw), (rel, mx)


@pytest.mark.parametrize("seed", range(16))
def test_randomized_operators_adjoint(seed):
    # NEXT-1 on the seeded random family: the GPU adjoint against the oracle's L* on
    # the full grid, and exact pairing <L~f, g> = <f, L~* g> with the GPU forward of the same plan
    op, dtype, eps, kw, fseed = _random_operator(seed)
    N = op.N
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    g = wl.white_noise(N, (fseed + 1) % 997, dtype)
    f = wl.white_noise(N, (fseed + 2) % 997, dtype)
    plan = make_plan(op, eps, dtype, **kw)
    Lsg = plan.apply_adjoint(torch.from_numpy(g).to(DEV, tdt)).cpu().numpy().astype(np.complex128)
    Lf = plan.apply(torch.from_numpy(f).to(DEV, tdt)).cpu().numpy().astype(np.complex128)
    rel = oracle.rel_l2(Lsg, adjoint_ref(op, g))
    lhs, rhs = np.vdot(g, Lf), np.vdot(Lsg, f)
    pair = abs(lhs - rhs) / (np.linalg.norm(f) * np.linalg.norm(g))
    ptol = 1e-5 if dtype == "c64" else 1e-12
    print(f"random adjoint {seed}: N={N} {dtype} eps={eps:g} {kw}: rel l2 vs oracle {rel:.3e}, pairing {pair:.2e}")
    assert rel <= 10 * eps, rel
    assert pair <= ptol * N, pair


@pytest.mark.parametrize("seed", range(8))
def test_randomized_operators_api_consistency(seed, tmp_path):
    # every entry point of include/fio.h on the seeded random family agrees with fio_apply: fio_apply_batch
    # (3 inputs) and fio_apply_host_stream bit for bit, a saved-and-loaded plan bit for bit, and a 3-way
    # wedge sharding (per-rank N x N partials, no communicator) summing to the 1-rank result (L = sum_l L_l,
    # PAPER.md:236-241) to rounding
    op, dtype, eps, kw, fseed = _random_operator(seed)
    N = op.N
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    fs = torch.stack([torch.from_numpy(wl.white_noise(N, (fseed + i) % 997, dtype)).to(tdt) for i in range(3)])
    plan = make_plan(op, eps, dtype, **kw)
    single = [plan.apply(fs[i].to(DEV)).cpu() for i in range(3)]
    batch = plan.apply_batch(fs.to(DEV)).cpu()
    hin, hout = fs.clone().pin_memory(), torch.empty_like(fs).pin_memory()
    plan.apply_host_stream(hin, hout)
    for i in range(3):
        assert torch.equal(batch[i], single[i]), ("batch", i)
        assert torch.equal(hout[i], single[i]), ("host_stream", i)
    path = str(tmp_path / "plan.fio")
    plan.save(path)
    loaded = make_plan(op, eps, dtype, load=path, **kw)
    assert torch.equal(loaded.apply(fs[0].to(DEV)).cpu(), single[0])
    acc = torch.zeros_like(single[0], dtype=torch.complex128)
    for r in range(3):
        acc += make_plan(op, eps, dtype, rank=r, nranks=3, **kw).apply(fs[0].to(DEV)).cpu().to(torch.complex128)
    rel = oracle.rel_l2(acc.numpy(), single[0].numpy())
    print(f"random api {seed}: N={N} {dtype} eps={eps:g} {kw}: sharded-sum vs 1 rank {rel:.2e}")
    assert rel <= (1e-5 if dtype == "c64" else 1e-12), rel


@pytest.mark.parametrize("N,dtype,eps", [(1000, "c128", 1e-6), (1080, "c64", 1e-4), (1250, "c128", 1e-6),
                                         (1536, "c64", 1e-5)])
def test_non_power_of_two_headline_sizes(N, dtype, eps):
    # 5-smooth, non-power-of-two grids near the headline size (K0's mixed radices 3 and 5, K1's general
    # f-hat index wrap instead of the power-of-two mask): GRT phase, 1024 sampled points vs the direct sum
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 31, dtype)
    plan, out = run(op, f, eps=eps, dtype=dtype)
    pts = wl.sample_points(N, 1024, 5)
    rel, mx = _pointwise(out.ravel()[pts], oracle.fio(op, f, pts=pts))
    print(f"N={N} {dtype} eps={eps:g}: W {plan.info['W']} sum_q {plan.info['sum_q']}: rel l2 {rel:.3e}, max {mx:.3e}")
    assert rel <= 10 * eps and mx <= 100 * eps, (rel, mx)
