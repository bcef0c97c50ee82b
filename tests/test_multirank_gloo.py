"""World-size-2 tests of the wedge-sharded path's host logic on CPU (gloo).

Each rank takes the wedges fio.assign_wedges gives it, computes its partial operator
L_S = sum_{l in S} L_l with the CPU oracle (the CUDA partial is
checked against exactly this on the GPU in test_gpu_parity), and the partials go
through the product's reduce_scatter_rows.  The slabs must tile the full-operator
oracle result."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import oracle
    import workloads as wl
    import paper_math_0610051_b200 as fio
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, W = 32, 8
        op = wl.grt_operator(N)
        f = wl.white_noise(N, 0)
        g = fio.geometry(N, W)
        cost = np.array([(g["wedge_of"] == l).sum() for l in range(W)], float)
        owner = fio.assign_wedges(cost, world)
        mine = [l for l in range(W) if owner[l] == rank]
        part = oracle.fio(op, f, wedges=mine, W=W, include_dc=(rank == 0))
        slab = fio.reduce_scatter_rows(torch.from_numpy(part), world)
        full = oracle.fio(op, f)
        rows = N // world
        err = float(np.abs(slab.numpy() - full[rank * rows:(rank + 1) * rows]).max())
        q.put((rank, len(mine), err))
    finally:
        dist.destroy_process_group()


def test_two_rank_wedge_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert sum(r[1] for r in res) == 8 and all(r[1] > 0 for r in res)
    assert max(r[2] for r in res) < 1e-12
