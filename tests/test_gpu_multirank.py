"""GPU tests of the wedge-sharded apply with the library's own NCCL communicator (SURVEY.md 8(a) A6,
8(b); BASELINE north_star (3)): L = sum_l L_l, every rank holds the partial sum
over its wedges and fio_apply ends with an NCCL reduce-scatter that leaves rank r its row slab.

- one GPU: a one-rank communicator runs the same NCCL code path (the reduce-scatter is a copy)
  and must reproduce the communicator-free apply bit for bit (forward, adjoint, batch, host);
- >= 2 GPUs: one process per GPU (and, separately, one thread per GPU in a single process)
  compare every rank's slab with the direct-sum oracle.  These skip on a one-GPU box."""
import os
import sys
import threading

import numpy as np
import pytest

import oracle
import workloads as wl

torch = pytest.importorskip("torch")
fio = pytest.importorskip("paper_math_0610051_b200")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _plan(op, eps=1e-6, dtype="c128", **kw):
    return fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=eps, dtype=dtype, rho_sign=op.sign,
                    amplitude=op.amp, **kw)


@pytest.mark.parametrize("dtype,eps", [("c128", 1e-6), ("c64", 1e-4)])
def test_one_rank_communicator_matches_plain_apply(dtype, eps):
    N = 128
    op = wl.grt_operator(N)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    plain = _plan(op, eps, dtype, device=0)
    comm = _plan(op, eps, dtype, device=0, nccl_id=fio.nccl_unique_id())
    assert comm.info["has_comm"] == 1 and comm.info["out_rows"] == N and plain.info["has_comm"] == 0
    f = torch.from_numpy(wl.white_noise(N, 3, dtype)).to("cuda:0", tdt)
    a, b = plain.apply(f), comm.apply(f)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert oracle.rel_l2(b.cpu().numpy(), oracle.fio(op, f.cpu().numpy().astype(np.complex128))) <= 10 * eps
    fb = torch.stack([f, 2 * f])
    assert torch.equal(comm.apply_batch(fb)[1], plain.apply(2 * f))
    hin = f.cpu().pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    comm.apply_host(hin, hout)
    assert torch.equal(hout, a.cpu())
    hs = torch.stack([f.cpu(), (2 * f).cpu(), f.cpu()]).pin_memory()
    ho = torch.empty_like(hs).pin_memory()
    comm.apply_host_stream(hs, ho)
    assert torch.equal(ho[0], a.cpu()) and torch.equal(ho[2], a.cpu())
    ga, gb = plain.apply_adjoint(f), comm.apply_adjoint(f)
    assert oracle.rel_l2(gb.cpu().numpy(), ga.cpu().numpy()) <= 1e-5  # atomics: last bits may differ


@pytest.mark.parametrize("dtype,eps", [("c128", 1e-6), ("c64", 1e-4)])
def test_one_rank_communicator_allgather_matches_plain_apply(dtype, eps):
    # opts.allgather (include/fio.h): reduce-scatter into this rank's rows, then an in-place NCCL
    # all-gather; with one rank both collectives are copies and the result is the plain apply's
    N = 96
    op = wl.grt_operator(N)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    plain = _plan(op, eps, dtype, device=0)
    comm = _plan(op, eps, dtype, device=0, nccl_id=fio.nccl_unique_id(), allgather=True)
    assert comm.info["has_comm"] == 1 and comm.out_rows == N
    f = torch.from_numpy(wl.white_noise(N, 4, dtype)).to("cuda:0", tdt)
    a = plain.apply(f)
    b = torch.full_like(a, float("nan"))
    comm.apply(f, out=b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert oracle.rel_l2(b.cpu().numpy(), oracle.fio(op, f.cpu().numpy().astype(np.complex128))) <= 10 * eps
    fb = torch.stack([f, 2 * f, f])
    ob = comm.apply_batch(fb)
    assert torch.equal(ob[0], a) and torch.equal(ob[1], plain.apply(2 * f)) and torch.equal(ob[2], a)
    hin = f.cpu().pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    comm.apply_host(hin, hout)
    assert torch.equal(hout, a.cpu())
    ga, gb = plain.apply_adjoint(f), comm.apply_adjoint(f)
    assert oracle.rel_l2(gb.cpu().numpy(), ga.cpu().numpy()) <= 1e-5


# ---------------------------------------------------------------- >= 2 GPUs
def _check_slab(op, f, slab, rank, world, pts_all):
    N = op.N
    r0, r1 = fio.row_slab(N, world, rank)
    assert slab.shape == (r1 - r0, N)
    if N <= 256:
        ref = oracle.fio(op, f)[r0:r1]
        return oracle.rel_l2(slab, ref)
    pts = pts_all[(pts_all >= r0 * N) & (pts_all < r1 * N)]
    ref = oracle.fio(op, f, pts=pts)
    return oracle.rel_l2(slab.ravel()[pts - r0 * N], ref)


def _proc(rank, world, port, N, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # only for the id broadcast
    try:
        op = wl.grt_operator(N)
        f = wl.white_noise(N, 0)
        plan = _plan(op, device=rank, rank=rank, nranks=world, group=dist.group.WORLD)
        slab = plan.apply(torch.from_numpy(f).to(f"cuda:{rank}")).cpu().numpy()
        err = _check_slab(op, f, slab, rank, world, wl.sample_points(N, 4096, 1))
        if N <= 256:  # the all-gather option: every rank holds the full Lf
            full = _plan(op, device=rank, rank=rank, nranks=world, group=dist.group.WORLD, allgather=True)
            Lf = full.apply(torch.from_numpy(f).to(f"cuda:{rank}")).cpu().numpy()
            r0, r1 = fio.row_slab(N, world, rank)
            assert Lf.shape == (N, N) and np.array_equal(Lf[r0:r1], slab)
            err = max(err, oracle.rel_l2(Lf, oracle.fio(op, f)))
        q.put((rank, err, plan.info["n_owned"]))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (one process per GPU)")
@pytest.mark.parametrize("N", [256, 2048])
def test_one_process_per_gpu(N):
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_proc, args=(r, world, port, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for rank, err, owned in res:
        assert owned > 0 and isinstance(err, float) and err <= 1e-5, (rank, err)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_two_devices_one_process():
    # one thread per device (fio_plan's communicator init and fio_apply's collective are entered by
    # every rank; ctypes releases the GIL during the library calls)
    N, world = 128, 2
    op = wl.grt_operator(N)
    f = wl.white_noise(N, 1)
    nid = fio.nccl_unique_id()
    out, errs = [None] * world, []

    def run(rank):
        try:
            plan = _plan(op, device=rank, rank=rank, nranks=world, nccl_id=nid)
            with torch.cuda.device(rank):
                out[rank] = plan.apply(torch.from_numpy(f).to(f"cuda:{rank}")).cpu().numpy()
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert oracle.rel_l2(np.concatenate(out), oracle.fio(op, f)) <= 1e-5
