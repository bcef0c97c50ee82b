"""Separation row-sample sweep (reading R8): for FIO_SEP_ROWS = k (rows sampled for the column pivoting =
k x r), report the worst pointwise and the l2 error over the seeded random operators of
tests/test_gpu_parity.py (full grid vs the direct sum) and the plan rank / apply time at N = 1024.
    FIO_SEP_ROWS=k python tools/sep_rows_sweep.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: this is a measurement script, not the product path)
import paper_math_0610051_b200 as fio  # noqa: E402
import workloads as wl  # noqa: E402

src = open(os.path.join(ROOT, "tests", "test_gpu_parity.py")).read()
exec(src[src.index("def _random_operator"):src.index('@pytest.mark.parametrize("seed"')])
res = {"FIO_SEP_ROWS": os.environ.get("FIO_SEP_ROWS", "default"), "random": {}}
worst = 0.0
for seed in range(16):
    op, dt, eps, kw, fs = _random_operator(seed)  # noqa: F821
    f = wl.white_noise(op.N, fs % 997, dt)
    ref = oracle.fio(op, f)
    p = fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=eps, dtype=dt, device=0, rho_sign=op.sign, **kw)
    tdt = torch.complex64 if dt == "c64" else torch.complex128
    out = p.apply(torch.from_numpy(f).to("cuda:0", tdt)).cpu().numpy().astype(np.complex128)
    rms = np.sqrt(np.mean(np.abs(ref) ** 2))
    rel = float(np.linalg.norm(out - ref) / np.linalg.norm(ref))
    mx = float(np.abs(out - ref).max() / rms)
    res["random"][seed] = {"rel_over_eps": rel / eps, "max_over_eps": mx / eps, "sum_q": p.info["sum_q"]}
    worst = max(worst, mx / eps)
    p.close()
res["worst_max_over_eps"] = worst
for name in ("cfg3_c128", "cfg3_c64"):
    cfg = wl.config(name)
    op, fnp = wl.make_operator(cfg), wl.make_input(cfg)
    t0 = time.time()
    p = fio.Plan(op.N, op.c1, op.c2, eps=cfg["eps"], dtype=cfg["dtype"], device=0)
    tp = time.time() - t0
    f = torch.from_numpy(fnp).to("cuda:0", torch.complex64 if cfg["dtype"] == "c64" else torch.complex128)
    out = torch.empty_like(f)
    for _ in range(3):
        p.apply(f, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        p.apply(f, out=out)
    e1.record()
    torch.cuda.synchronize()
    pts = wl.sample_points(op.N, 1024, 1)
    r = oracle.fio(op, fnp, pts=pts)
    got = out.cpu().numpy().astype(np.complex128).ravel()[pts]
    res[name] = {"sum_q": p.info["sum_q"], "plan_s": tp, "ms": e0.elapsed_time(e1) / 10,
                 "rel_l2_1024pts": float(np.linalg.norm(got - r) / np.linalg.norm(r))}
    p.close()
print("RESULT " + json.dumps(res))
