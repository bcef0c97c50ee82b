"""Predicted per-rank balance of the wedge-sharded plan (rank 0's plan of R ranks, one GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_math_0610051_b200 as fio  # noqa: E402
import workloads as wl  # noqa: E402

for name in sys.argv[1:] or ["cfg3_c128", "cfg4"]:
    cfg = wl.config(name)
    op = wl.make_operator(cfg)
    for R in (2, 4, 8):
        p = fio.Plan(op.N, op.c1, op.c2, eps=cfg["eps"], dtype=cfg["dtype"], device=0, rank=0, nranks=R)
        i = p.info
        print(f"{name} R={R} W={i['W']} rank0 wedges={i['n_owned']} sum_q={i['sum_q']} "
              f"predicted max/mean load={i['rank_balance']:.3f} plan_s={i['plan_seconds']:.1f}", flush=True)
        p.close()
