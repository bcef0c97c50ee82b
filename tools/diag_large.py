"""Diagnose two seeded large random operators (tests/test_gpu_parity.py test_randomized_operators_large_sampled):
which stage (separation, NUFFT taps, precision) sets the error.  Measurement script (uses oracle/ as the checker)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch  # noqa: E401,E402
import oracle, workloads as wl  # noqa: E401,E402
import paper_math_0610051_b200 as fio  # noqa: E402

src = open(os.path.join(ROOT, "tests", "test_gpu_parity.py")).read()
exec(src[src.index("def _random_operator"):src.index('@pytest.mark.parametrize("seed", range(16))')])


def large(seed):
    r = np.random.default_rng(5000 + seed)
    op, dtype, eps, kw, fseed = _random_operator(100 + seed)  # noqa: F821
    N = int(r.choice([160, 192, 200, 240, 250, 256, 288, 300, 320, 360, 384, 400, 432, 450, 480, 500, 512]))
    x1, x2 = wl.grid(N)
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
        c2 = c1.copy()
    return wl.Operator(N, c1, c2, sign=op.sign, amp=amp), dtype, eps, kw, fseed


for seed, variants in ((4, [{}, {"r_init": 256}, {"n_wedges": 24}, {"nufft_w": 10}]),
                       (7, [{}, {"dtype": "c128"}, {"nufft_w": 8}, {"eps": 1e-4}, {"n_wedges": 24}])):
    op, dtype, eps, kw, fseed = large(seed)
    pts = wl.sample_points(op.N, 2048, 2 + seed)
    for v in variants:
        dt = v.get("dtype", dtype)
        e = v.get("eps", eps)
        f = wl.white_noise(op.N, fseed % 997, dt)
        ref = oracle.fio(op, f, pts=pts)
        args = {**kw, **{k: x for k, x in v.items() if k not in ("dtype", "eps")}}
        p = fio.Plan(op.N, op.c1, op.c2, eps=e, dtype=dt, device=0, rho_sign=op.sign, amplitude=op.amp, **args)
        t = torch.from_numpy(f).to("cuda:0", torch.complex64 if dt == "c64" else torch.complex128)
        out = p.apply(t).cpu().numpy().astype(np.complex128).ravel()[pts]
        rms = np.sqrt(np.mean(np.abs(ref) ** 2))
        print(f"seed {seed} N={op.N} amp={op.amp} {dt} eps={e:g} {args}: rel {np.linalg.norm(out - ref) / np.linalg.norm(ref):.3e} "
              f"max {np.abs(out - ref).max() / rms:.3e} sum_q {p.info['sum_q']} W {p.info['W']} w {p.info['nufft_w']} "
              f"sep {p.info['max_sep_err']:.2e} cert {p.info['certified']}", flush=True)
        p.close()
