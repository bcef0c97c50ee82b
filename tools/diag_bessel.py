"""Where does the error of the random Bessel-amplitude operator (large seed 7) come from?  Split the input
into its lowest frequencies (|xi| <= 3) and the rest and measure each part's output error; compare with the
same phase and a == 1.  Measurement script (uses oracle/ as the checker)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv = [sys.argv[0]]
import numpy as np, torch  # noqa: E401,E402
import oracle, workloads as wl  # noqa: E401,E402
import paper_math_0610051_b200 as fio  # noqa: E402
exec(open(os.path.join(ROOT, "tools", "diag_large.py")).read().split("for seed, variants in")[0])
op, dtype, eps, kw, fseed = large(7)  # noqa: F821
N = op.N
pts = wl.sample_points(N, 2048, 9)
f = wl.white_noise(N, fseed % 997, "c128")
fh = np.fft.fft2(f)
xi1, xi2 = wl.freqs(N)
low = (xi1.astype(float) ** 2 + xi2.astype(float) ** 2) <= 9
parts = {"all": f, "low |xi|<=3": np.fft.ifft2(np.where(low, fh, 0)), "high": np.fft.ifft2(np.where(low, 0, fh))}
for amp in ("bessel", "separable"):
    o = wl.Operator(N, op.c1, op.c2, sign=op.sign, amp=amp)
    p = fio.Plan(N, o.c1, o.c2, eps=eps, dtype="c128", device=0, rho_sign=o.sign, amplitude=amp, **kw)
    for name, g in parts.items():
        ref = oracle.fio(o, g, pts=pts)
        out = p.apply(torch.from_numpy(np.ascontiguousarray(g)).to("cuda:0")).cpu().numpy().ravel()[pts]
        print(f"amp={amp} eps={eps:g} input {name}: rel {np.linalg.norm(out - ref) / np.linalg.norm(ref):.3e} "
              f"|ref| {np.linalg.norm(ref):.3e} |err| {np.linalg.norm(out - ref):.3e}", flush=True)
    p.close()
