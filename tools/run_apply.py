"""Plan + a few applies of one BASELINE config (the command profiled under ncu):
    python tools/run_apply.py cfg3_c64 [applies]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_math_0610051_b200 as fio  # noqa: E402
import workloads as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3_c64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = wl.config(name)
op = wl.make_operator(cfg)
plan = fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=cfg["eps"], dtype=cfg["dtype"], device=0)
f = torch.from_numpy(wl.make_input(cfg)).to("cuda:0", torch.complex64 if cfg["dtype"] == "c64" else torch.complex128)
for _ in range(n):
    out = plan.apply(f)
torch.cuda.synchronize()
print(name, plan.info["sum_q"], plan.info["max_tile_cap"], float(out.abs().mean()))
