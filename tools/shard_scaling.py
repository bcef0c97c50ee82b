"""Estimate wedge-sharded strong scaling on ONE GPU: time rank r's partial apply (its wedges only:
the compute every rank does at R GPUs) for r = 0..R-1 and report T1 / (R * max_r T_r).  The NCCL
reduce-scatter is not measured (one GPU): `rs_ms_model` is its modelled time, (R-1)/R N^2 s bytes per rank at
the guide's measured 8-rank NCCL bus bandwidth (725 GB/s, B200_PROFILING.md) plus 20 us, and
`est_efficiency_with_rs` = T1 / (R (max_r T_r + rs_ms_model)) -- an estimate, not a multi-GPU measurement."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_math_0610051_b200 as fio  # noqa: E402
import workloads as wl  # noqa: E402


def time_apply(plan, f, steps=5):
    out = torch.empty_like(f)
    for _ in range(2):
        plan.apply(f, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        plan.apply(f, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


res = {}
for name in sys.argv[1:] or ["cfg3_c128"]:
    cfg = wl.config(name)
    op = wl.make_operator(cfg)
    f = torch.from_numpy(wl.make_input(cfg)).to("cuda:0", torch.complex64 if cfg["dtype"] == "c64" else torch.complex128)
    t1 = None
    for R in (1, 2, 4, 8):
        ts = []
        for r in range(R):
            p = fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=cfg["eps"], dtype=cfg["dtype"],
                         device=0, rank=r, nranks=R)
            ts.append(time_apply(p, f))
            p.close()
            torch.cuda.empty_cache()
        tmax = max(ts)
        if R == 1:
            t1 = tmax
        eff = t1 / (R * tmax)
        cs = 8 if cfg["dtype"] == "c64" else 16
        rs = 0.0 if R == 1 else ((R - 1) / R * op.N * op.N * cs / 725e9 + 20e-6) * 1e3
        eff_rs = t1 / (R * (tmax + rs))
        res[f"{name}_R{R}"] = {"max_rank_ms": tmax, "min_rank_ms": min(ts), "est_efficiency": eff,
                               "rs_ms_model": rs, "est_efficiency_with_rs": eff_rs}
        print(f"{name} R={R}: per-rank ms max {tmax:.3f} min {min(ts):.3f} -> est. efficiency {eff:.3f}, "
              f"with the modelled reduce-scatter ({rs:.3f} ms) {eff_rs:.3f}", flush=True)
print(json.dumps(res))
