"""Wedge-count sweep on one GPU (reading R1: the aperture constant is free):
    python tools/w_sweep.py [--configs=cfg3_c64,cfg3_c128] [--wedges=32,48,64,80] [--steps=10]
Per config and W: apply ms (CUDA events), per-stage ms (library profile), sum_q, fine-grid volume, and
"dev" = relative l2 difference of the output from the output at the default W (the first listed W
that equals the default, else the first W).  Parity against the oracle is the tests' job (this tool
does not use oracle/)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_math_0610051_b200 as fio  # noqa: E402
import workloads as wl  # noqa: E402

opts = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("--"))
configs = opts.get("configs", "cfg3_c64,cfg3_c128").split(",")
wedges = [int(w) for w in opts.get("wedges", "32,48,64,80").split(",")]
steps = int(opts.get("steps", "10"))
res = {}
for name in configs:
    cfg = wl.config(name)
    op = wl.make_operator(cfg)
    f = wl.make_input(cfg)
    c64 = cfg["dtype"] == "c64"
    t = torch.from_numpy(f).to("cuda:0", torch.complex64 if c64 else torch.complex128)
    ref = None
    for W in wedges:
        plan = fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=cfg["eps"], dtype=cfg["dtype"],
                        device=0, n_wedges=W)
        out = torch.empty_like(t)
        for _ in range(3):
            plan.apply(t, out=out)
        torch.cuda.synchronize()
        plan.profile_begin(steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            plan.apply(t, out=out)
        e1.record()
        torch.cuda.synchronize()
        st = plan.profile_end()
        got = out.cpu().numpy().astype(np.complex128)
        if ref is None:
            ref = got
        info = plan.info
        r = {"W": info["W"], "ms": e0.elapsed_time(e1) / steps,
             "stages": {k: st[k] / max(st["n"], 1) for k in fio.STAGES}, "sum_q": info["sum_q"],
             "fine_elems": info["fine_elems"], "slot_terms": info["slot_terms"],
             "alpha_GB": info["alpha_bytes"] / 1e9, "plan_s": info["plan_seconds"],
             "dev": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)), "max_sep_err": info["max_sep_err"]}
        res.setdefault(name, []).append(r)
        print(name, json.dumps(r), flush=True)
        plan.close()
print("ALL " + json.dumps(res))
