"""Multi-RHS timing (NEXT-2): per-input ms of fio_apply_batch at batch B against single applies.
    python tools/batch_bench.py [--configs=cfg3_c64,cfg3_c128] [--batches=2,4,8] [--steps=5]
(FIO_K3_RHS=1 in the environment makes K3 serve one right-hand side per launch, for comparison.)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_math_0610051_b200 as fio  # noqa: E402
import workloads as wl  # noqa: E402

opts = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("--"))
steps = int(opts.get("steps", "5"))
res = {}
for name in opts.get("configs", "cfg3_c64,cfg3_c128").split(","):
    cfg = wl.config(name)
    op = wl.make_operator(cfg)
    c64 = cfg["dtype"] == "c64"
    tdt = torch.complex64 if c64 else torch.complex128
    plan = fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=cfg["eps"], dtype=cfg["dtype"], device=0)
    f = torch.from_numpy(wl.make_input(cfg)).to("cuda:0", tdt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        plan.apply(f)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        plan.apply(f)
    e1.record()
    torch.cuda.synchronize()
    r = {"single_ms": e0.elapsed_time(e1) / steps}
    for B in [int(b) for b in opts.get("batches", "2,4,8").split(",")]:
        fb = torch.stack([f * (1 + 0.1 * i) for i in range(B)])
        out = plan.apply_batch(fb)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            plan.apply_batch(fb, out=out)
        e1.record()
        torch.cuda.synchronize()
        r[f"batch{B}_ms_per_input"] = e0.elapsed_time(e1) / steps / B
        r[f"batch{B}_equal_single"] = bool(torch.equal(out[B - 1], plan.apply(fb[B - 1])))
    res[name] = r
    print(name, json.dumps(r), flush=True)
    plan.close()
print("ALL " + json.dumps({"k3_rhs": os.environ.get("FIO_K3_RHS", "default"), **res}))
