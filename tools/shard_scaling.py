"""Estimate wedge-sharded strong scaling on ONE GPU: time rank r's partial apply (its wedges only:
the compute every rank does at R GPUs) for r = 0..R-1 and report T1 / (R * max_r T_r).  The NCCL
reduce-scatter (N*N complex, over NVLink) is not included."""
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
        res[f"{name}_R{R}"] = {"max_rank_ms": tmax, "min_rank_ms": min(ts), "est_efficiency": eff}
        print(f"{name} R={R}: per-rank ms max {tmax:.3f} min {min(ts):.3f} -> est. efficiency {eff:.3f}", flush=True)
print(json.dumps(res))
