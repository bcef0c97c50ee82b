"""bench.py -- FIO applies/s at N=1024 on 1..8 B200s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3_c128] [--impl fio|reference]

A step is one full fio_apply (K0 input FFT, K1 window x beta + row FFT, K2 column
FFT, K3 interpolation + alpha epilogue; + the reduce-scatter over NCCL when the
wedges are sharded over N ranks) of one synthetic N x N input already resident
in HBM.  Default workload: BASELINE config 3 (N=1024 generalized-Radon FIO) in
complex128 at eps = 1e-6; the complex64 / eps = 1e-4 variant of the same config
is timed in the same run and reported under "variants".  Rank 0 prints ONE
JSON line.  `--impl reference` times the CPU oracle (direct summation, eq. dfio)
on a bounded sample of the same workload -- the only other place bench.py runs
oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402  (input generators only)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="cfg3_c128")
    p.add_argument("--variant", default="cfg3_c64", help="second config timed in the same run ('' = none)")
    p.add_argument("--impl", default="fio", choices=["fio", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-points", type=int, default=8192, help="oracle sample size (output points)")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p is None:
            return
        time.sleep(0.25)
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- roofline model
def k3_algorithmic_bytes(info, N, c64):
    """Algorithmic HBM bytes of the K3 launches of one apply:
    alpha' = N^2 sum_q s (every output point x each owned wedge's terms, no padding), one read of
    every fine grid G_lt, and the Lf write."""
    cs = 8 if c64 else 16
    return N * N * info["sum_q"] * cs + info["fine_elems"] * cs + N * N * cs


def apply_algorithmic_bytes(info, N, c64):
    """Whole apply: K0 (read f, write+read tmp, write fhat), K1 (beta', fhat gather, write P1),
    K2 (read P1, write G) and K3."""
    cs = 8 if c64 else 16
    k0 = 4 * N * N * cs
    k12 = info["beta_bytes"] + N * N * cs + 2 * info["p1_elems"] * cs + info["fine_elems"] * cs
    return k0 + k12 + k3_algorithmic_bytes(info, N, c64)


def k3_resource_model(info, c64, ms, sm_mhz):
    """What binds K3 on chip: per group-term the thread reads its window
    (k3_window_rows x k3_window_cols, plan dtype) -- plus the P row weights (FP32 c64 / FP64 c128) where
    they do not stay in registers -- from shared memory and alpha'(t) from the ring, and issues 2 real FMAs per (point, window cell), 2 per
    (point, row) and 4 for the alpha product.  Fractions of the shared -> register path
    (measured: 126 B/clk/SM for conflict-free 16-byte loads) and of the FMA pipe (measured: 126 FP32 /
    63 FP64 FMA/clk/SM), profiles/r02_microbench.json, at the sampled SM clock."""
    P = info["group_p"]
    win, winr = info["k3_window_cols"], info["k3_window_rows"]
    cs, rs = (8, 4) if c64 else (16, 8)
    gt = info["slot_terms"] / P
    # row weights come from shared memory only where K3 keeps them out of registers (fio_kernels.cu
    # k3_p1reg: complex64 w <= 5 or 9..11, complex128 w <= 9 keep them in registers)
    taps = info["nufft_w"]
    preg = (taps <= 5 or 9 <= taps <= 11) if c64 else taps <= 9
    lsu_bytes = gt * (winr * win * cs + (0 if preg else winr * P * rs) + P * cs)
    fmas = gt * P * (winr * (win * 2 + 2) + 4)
    clk = (sm_mhz or 1965.0) * 1e6
    t = ms * 1e-3
    sms = 148
    lds, f32, f64 = 128.0, 126.4, 63.3  # fallback: the guide's shared-memory path, measured FMA rates
    try:
        with open(os.path.join(ROOT, "profiles", "r02_microbench.json")) as fh:
            mb = json.load(fh)
        lds, f32, f64 = (float(mb["lds128_contiguous_B_per_clk_sm"]), float(mb["ffma2_fma_per_clk_sm"]),
                         float(mb["dfma_per_clk_sm"]))
    except Exception:
        pass
    return {"lsu_bytes": lsu_bytes, "lsu_frac": lsu_bytes / t / (sms * lds * clk),
            "fma": fmas, "fma_frac": fmas / t / (sms * (f32 if c64 else f64) * clk),
            "flops_per_s": 2 * fmas / t, "sm_mhz": sm_mhz, "model": "DESIGN.md section 7"}


def alu_roofline(info, c64, k3_ms):
    """K3 against its arithmetic roofline: the FMAs it issues per apply (k3_resource_model, padding
    slots included) as FLOP/s over the measured FMA peak of its precision (FP64 pipe for complex128,
    FP32 packed FFMA2 for complex64)."""
    fp64, fp32, src = alu_peaks()
    m = k3_resource_model(info, c64, k3_ms, None)
    ach = m["flops_per_s"] / 1e12
    peak = fp32 if c64 else fp64
    return {"bound": "alu", "pipe": "fp32 (FFMA2)" if c64 else "fp64 (DFMA)", "achieved": ach, "peak": peak,
            "unit": "TFLOP/s", "frac": ach / peak, "peak_source": src,
            "flops": 2 * m["fma"], "flops_model": "2 x slot_terms x (rows (2 cols + 2) + 4)"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def alu_peaks():
    """FP64 / FP32 FMA peaks of this pool's B200s, measured by tools/microbench.cu (profiles/
    r02_microbench.json): DFMA and packed FFMA2 over all 148 SMs; fallback = the guide's unit counts
    (64 DFMA / 128 FFMA per clk per SM at 1965 MHz)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_microbench.json")) as fh:
            mb = json.load(fh)
        return float(mb["dfma_tflops"]), float(mb["ffma2_tflops"]), "measured (profiles/r02_microbench.json)"
    except Exception:
        return 2 * 64 * 148 * 1.965e9 / 1e12, 2 * 128 * 148 * 1.965e9 / 1e12, "unit counts x 1965 MHz"


# ---------------------------------------------------------------- CPU oracle baseline
def cpu_oracle_rate(cfg, npts, seed=1):
    import oracle
    op = wl.make_operator(cfg)
    f = wl.make_input(cfg)
    N = cfg["N"]
    fh = oracle.dft2(f)
    pts = wl.sample_points(N, npts, seed)
    t0 = time.perf_counter()
    ref = oracle.fio(op, fhat=fh, pts=pts)
    dt = time.perf_counter() - t0
    pps = len(pts) / dt
    return {"ref": ref, "pts": pts, "seconds": dt, "value": pps / (N * N), "unit": "applies/s", "points_per_s": pps,
            "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"{len(pts)} seeded output points of the N={N} grid (direct sum over all N^2 frequencies, "
                      f"fhat precomputed), {dt:.1f} s; applies/s = points/s / N^2"}


def bench_config(name, world):
    """The `config` object of the JSON line -- identical for the CUDA arm and the oracle arm."""
    cfg = wl.config(name)
    return {"workload": name, "N": cfg["N"], "eps": cfg["eps"],
            "parallelism": f"wedge-sharded x{world}" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (the separated factors alpha' are streamed from HBM every step)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = wl.config(args.config)
    N = cfg["N"]
    times = []
    npts = max(64, args.cpu_points // 4)
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_rate(cfg, npts, seed=1 + i)
        r.pop("ref"), r.pop("pts")  # (r["seconds"]: this step's measured time)
        if i >= args.warmup:
            times.append(r)
    pps = statistics.median([t["points_per_s"] for t in times])
    val = pps / (N * N)
    # ms_per_step is the measured wall time of one timed step (one bounded sample, so the timed region
    # is the one this process actually ran); `value` scales the sample's points/s to whole applies
    step_ms = statistics.median([t["seconds"] for t in times]) * 1e3
    line = {"metric": "fio_applies_per_s", "value": val, "unit": "applies/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "ms_per_full_apply_extrapolated": 1e3 / val, "devices": "host CPU cores only (the oracle)",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic", "impl": "reference",
            "config": bench_config(args.config, world),
            "points_per_s": pps,
            "cpu_baseline": {"value": val, "unit": "applies/s", "cores": times[0]["cores"], "kind": "oracle",
                             "sample": f"each step: {npts} seeded output points (direct sum), median over steps"},
            "e2e": {"value": val, "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def time_config(name, args, rank, world, local, group):
    import torch
    import torch.distributed as dist
    import paper_math_0610051_b200 as fio

    cfg = wl.config(name)
    N = cfg["N"]
    c64 = cfg["dtype"] == "c64"
    op = wl.make_operator(cfg)
    f_np = wl.make_input(cfg)
    dev = torch.device("cuda", local)
    # N > 1: the plan owns an NCCL communicator (id broadcast over `group`); fio_apply then ends with
    # the library's reduce-scatter and returns this rank's (N/R) x N row slab
    plan = fio.Plan(N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=cfg["eps"], dtype=cfg["dtype"],
                    device=local, rank=rank, nranks=world, group=group if world > 1 else None)
    info = plan.info
    tdt = torch.complex64 if c64 else torch.complex128
    f = torch.from_numpy(f_np).to(dev, tdt)
    stream = torch.cuda.current_stream(dev)

    def step():
        return plan.apply(f, out=out)

    out = torch.empty((plan.out_rows, N), dtype=tdt, device=dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier(group=group)
    plan.profile_begin(args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(group=group)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(group=group)
    ms = e0.elapsed_time(e1)
    stages = plan.profile_end()
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        ms = float(t.item())
    ms_step = ms / args.steps
    applies_per_s = 1e3 / ms_step
    # adjoint (NEXT-1), same input, device-timed
    adj_ms = None
    if world == 1:
        g = torch.empty_like(f)
        for _ in range(2):
            plan.apply_adjoint(f, out=g)
        a0e, a1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a0e.record(stream)
        for _ in range(args.steps):
            plan.apply_adjoint(f, out=g)
        a1e.record(stream)
        torch.cuda.synchronize(dev)
        adj_ms = a0e.elapsed_time(a1e) / args.steps
        del g
    # e2e through the public API with host buffers (pinned), copies inside the timed region,
    # device-timed with CUDA events on the launching stream (max over ranks): one
    # fio_apply_host_stream call serves the K steps' inputs (one pinned N x N host buffer per step)
    # and reads every result back, the copies pipelined with the applies
    # (at most 32 steps per call: bounded pinned memory for long runs)
    per_call = min(args.steps, 32)
    hin1 = torch.from_numpy(f_np.astype(np.complex64 if c64 else np.complex128))
    hin = hin1.unsqueeze(0).repeat(per_call, 1, 1).pin_memory()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hout = torch.empty((per_call, plan.out_rows, N), dtype=hin.dtype).pin_memory()
    d2h = hout[0].numel() * hout.element_size()
    plan.apply_host_stream(hin[:2], hout[:2])  # warm-up (allocates the staging buffers)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier(group=group)
    ev0.record(stream)
    done = 0
    while done < args.steps:
        k = min(per_call, args.steps - done)
        plan.apply_host_stream(hin[:k], hout[:k])
        done += k
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = ev0.elapsed_time(ev1) / args.steps
    e2e_equal = bool(torch.equal(hout[k - 1], out.cpu()))  # the streamed results are fio_apply's, bit for bit
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        e2e_ms = float(t.item())
    e2e = {"value": 1e3 / e2e_ms, "unit": "applies/s", "h2d_bytes_per_step": hin[0].numel() * hin.element_size(),
           "d2h_bytes_per_step": d2h, "api": "fio_apply_host_stream (copies pipelined with the applies)",
           "equals_device_output": e2e_equal}
    n = max(stages["n"], 1)
    k3_ms = stages["K3_interp"] / n
    hbm, src = peaks()
    k3_bytes = k3_algorithmic_bytes(info, N, c64)
    traffic = None  # DRAM bytes of all K3 launches of one apply, from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "r02_k3_traffic.json")) as fh:
            tr = json.load(fh).get(name)
        if (tr and world == 1 and tr.get("sum_q") == info["sum_q"]
                and tr.get("max_tile_cap") == info["max_tile_cap"]):
            traffic = tr["dram_bytes"]
    except Exception:
        traffic = None
    ach = k3_bytes / (k3_ms * 1e-3) / 1e9
    total_stage = sum(stages[k] for k in fio.STAGES) / n
    res = {
        "name": name, "N": N, "eps": cfg["eps"], "dtype": "c64" if c64 else "c128",
        "ms_per_step": ms_step, "applies_per_s": applies_per_s, "points_per_s": applies_per_s * N * N,
        "stage_ms": {k: stages[k] / n for k in fio.STAGES},
        "k3_share": k3_ms / total_stage if total_stage > 0 else None,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                     "traffic": traffic, "kernel": "k_interp_groups (K3, all wedge launches of one apply)",
                     "peak_source": src, "traffic_source": "profiles/r02_k3_traffic.json (ncu, cold cache)",
                     "algorithmic_bytes": k3_bytes,
                     "bytes_model": "N^2 sum_q s (alpha') + fine_elems s (G read once) + N^2 s (Lf write)"},
        "alu_roofline": dict(alu_roofline(info, c64, k3_ms), traffic=traffic,
                             kernel="k_interp_groups (K3, all wedge launches of one apply)"),
        "apply_hbm_gbs": apply_algorithmic_bytes(info, N, c64) / (ms_step * 1e-3) / 1e9,
        "k3_resources": k3_resource_model(info, c64, k3_ms, clk.summary().get("sm_mhz")),
        "plan": {"W": info["W"], "sum_q": info["sum_q"], "nufft_w": info["nufft_w"],
                 "plan_seconds": info["plan_seconds"], "max_sep_err": info["max_sep_err"],
                 "alpha_GB": info["alpha_bytes"] / 1e9, "fine_elems": info["fine_elems"],
                 "slots": info["slots"], "max_tile_cap": info["max_tile_cap"],
                 "k3_group_fill": N * N * info["n_owned"] / max(info["slots"], 1),
                 "group_p": info["group_p"],
                 "rank_balance": info["rank_balance"]},
        "launches_per_step": info["launches_per_apply"],
        "adjoint_ms_per_step": adj_ms,
        "clocks": clk.summary(), "e2e": e2e,
        "out": out.cpu().numpy().astype(np.complex128) if world == 1 else None,
    }
    plan.close()
    del f, out
    torch.cuda.empty_cache()
    return res


def run_gpu(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    group = None
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    else:
        torch.cuda.set_device(local)
    main = time_config(args.config, args, rank, world, local, group)
    variants = {}
    if args.variant:
        v = time_config(args.variant, args, rank, world, local, group)
        variants[args.variant] = {k: v[k] for k in ("dtype", "eps", "applies_per_s", "points_per_s", "ms_per_step",
                                                    "roofline", "stage_ms", "k3_share", "plan", "e2e",
                                                    "adjoint_ms_per_step", "k3_resources", "alu_roofline")}
    if rank == 0:
        cpu = None
        check = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_oracle_rate(wl.config(args.config), args.cpu_points)
            # the TIMED output against the oracle values the cpu_baseline leg just computed
            ref, pts = cpu.pop("ref"), cpu.pop("pts")
            got = main["out"].ravel()[pts]
            rms = float(np.sqrt(np.mean(np.abs(ref) ** 2)))
            check = {"rel_l2": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
                     "max_abs_err_over_rms": float(np.abs(got - ref).max() / rms), "points": int(len(pts)),
                     "bar": f"rel_l2 <= 10 eps = {10 * main['eps']:g}"}
        line = {
            "metric": "fio_applies_per_s", "value": main["applies_per_s"], "unit": "applies/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": main["dtype"], "data": "synthetic",
            "config": bench_config(args.config, world),
            "alpha_GB_per_step": main["plan"]["alpha_GB"],
            "points_per_s": main["points_per_s"],
            # the roofline that binds the dominant kernel: FP64 pipe for complex128 K3,
            # HBM for complex64; the other one is reported beside it
            "roofline": main["alu_roofline"] if main["dtype"] == "c128" else main["roofline"],
            "hbm_roofline": main["roofline"], "alu_roofline": main["alu_roofline"],
            "apply_hbm_gbs": main["apply_hbm_gbs"], "stage_ms": main["stage_ms"],
            "k3_resources": main["k3_resources"],
            "k3_share": main["k3_share"], "plan": main["plan"], "adjoint_ms_per_step": main["adjoint_ms_per_step"],
            "clocks": main["clocks"], "e2e": main["e2e"],
            "gpu_launches": main["launches_per_step"] * args.steps,
            "cpu_baseline": cpu, "check": check, "variants": variants,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
