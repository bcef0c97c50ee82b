"""World-size-2 tests of the wedge-sharded path's host logic on CPU (gloo).

The cross-GPU sum itself is an NCCL reduce-scatter inside the library (fio_apply with a
communicator; its GPU tests are in test_gpu_multirank.py).  What runs on the host, and is tested
here with two gloo ranks:
  - the NCCL unique id: rank 0 draws it through the library (fio_nccl_unique_id) and the binding's
    only collective, broadcast_nccl_id, hands every rank the same 128 bytes;
  - the wedge -> rank assignment (fio_assign_wedges, LPT) and the row-slab bookkeeping (row_slab):
    each rank's partial operator L_S = sum_{l in S} L_l, evaluated here by the
    CPU oracle, summed over the ranks (a test-side all_reduce standing in for the reduce-scatter)
    and cut to the rank's slab, must equal the slab of the full-operator oracle result."""
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
        nid = fio.broadcast_nccl_id()
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        same_id = len(nid) == fio.NCCL_ID_BYTES and all(i == nid for i in ids) and any(nid)
        N, W = 32, 8
        op = wl.grt_operator(N)
        f = wl.white_noise(N, 0)
        g = fio.geometry(N, W)
        cost = np.array([(g["wedge_of"] == l).sum() for l in range(W)], float)
        owner = fio.assign_wedges(cost, world)
        mine = [l for l in range(W) if owner[l] == rank]
        part = torch.from_numpy(oracle.fio(op, f, wedges=mine, W=W, include_dc=(rank == 0)))
        full_sum = torch.view_as_real(part).clone()
        dist.all_reduce(full_sum, op=dist.ReduceOp.SUM)
        r0, r1 = fio.row_slab(N, world, rank)
        slab = torch.view_as_complex(full_sum)[r0:r1].numpy()
        full = oracle.fio(op, f)
        err = float(np.abs(slab - full[r0:r1]).max())
        q.put((rank, len(mine), err, same_id, r1 - r0))
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
    assert all(r[3] for r in res)          # one id, identical on both ranks
    assert [r[4] for r in res] == [16, 16]  # N / R rows each
