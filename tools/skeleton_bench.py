"""Apply time and plan memory, stored alpha' vs skeleton storage."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_math_0610051_b200 as fio  # noqa: E402
import workloads as wl  # noqa: E402

for name in sys.argv[1:] or ["cfg3_c64", "cfg3_c128"]:
    cfg = wl.config(name)
    op = wl.make_operator(cfg)
    f = torch.from_numpy(wl.make_input(cfg)).to("cuda:0", torch.complex64 if cfg["dtype"] == "c64" else torch.complex128)
    for sk in (False, True):
        p = fio.Plan(op.N, op.c1, op.c2, eps=cfg["eps"], dtype=cfg["dtype"], device=0, skeleton=sk)
        out = p.apply(f)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            p.apply(f, out=out)
        e1.record()
        torch.cuda.synchronize()
        i = p.info
        print(f"{name} skeleton={sk}: {e0.elapsed_time(e1) / 5:.2f} ms/apply, alpha' storage {i['alpha_bytes'] / 1e9:.3f} GB"
              f" (+ skeleton {i['skeleton_bytes'] / 1e6:.2f} MB), workspace {i['workspace_bytes'] / 1e9:.2f} GB", flush=True)
        p.close()
        torch.cuda.empty_cache()

# multi-RHS batch (NEXT-2): one alpha' rebuild per wedge serves all inputs
for name in sys.argv[1:] or ["cfg3_c64", "cfg3_c128"]:
    cfg = wl.config(name)
    op = wl.make_operator(cfg)
    tdt = torch.complex64 if cfg["dtype"] == "c64" else torch.complex128
    for sk in (False, True):
        p = fio.Plan(op.N, op.c1, op.c2, eps=cfg["eps"], dtype=cfg["dtype"], device=0, skeleton=sk)
        for B in (1, 4, 8):
            f = torch.from_numpy(wl.make_input(cfg)).to("cuda:0", tdt).unsqueeze(0).repeat(B, 1, 1).contiguous()
            out = p.apply_batch(f)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                p.apply_batch(f, out=out)
            e1.record()
            torch.cuda.synchronize()
            print(f"{name} skeleton={sk} batch={B}: {e0.elapsed_time(e1) / 3 / B:.2f} ms per input", flush=True)
        p.close()
        torch.cuda.empty_cache()
