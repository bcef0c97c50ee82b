"""Run a few applies of one BASELINE config (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_math_0610051_b200 as fio  # noqa: E402
import workloads as wl  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="cfg3_c64")
p.add_argument("--iters", type=int, default=3)
a = p.parse_args()
cfg = wl.config(a.config)
op = wl.make_operator(cfg)
f = torch.from_numpy(wl.make_input(cfg)).to("cuda:0", torch.complex64 if cfg["dtype"] == "c64" else torch.complex128)
plan = fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=cfg["eps"], dtype=cfg["dtype"], device=0)
for _ in range(a.iters):
    out = plan.apply(f)
torch.cuda.synchronize()
print(a.config, plan.info["sum_q"], plan.info["slots"], float(out.abs().mean()))
