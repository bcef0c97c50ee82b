"""Build K3 variants (compile-time switches) in scratch copies of the repo and time them on the GPU.

    python tools/k3_variants.py NAME=FLAGS[@ENV=V,...] [NAME=FLAGS ...] [--configs=cfg3_c64,cfg3_c128] [--steps=10]
                                [--overlap=0.25]

Each variant: copy the repo to /tmp/fio_var_NAME, build libfio_b200.so with FIO_NVCC_FLAGS=FLAGS,
then (in a fresh process) plan + apply the configs, report per-stage ms (CUDA events, library
profile) and "dev": the relative l2 difference of the variant's output from the FIRST variant's output
on the same config (parity against the oracle is the tests' job; this tool does not use oracle/).
--wedges=W overrides the wedge count (opts.n_wedges)."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, time
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import os
import paper_math_0610051_b200 as fio, workloads as wl
res = {}
for name in sys.argv[2].split(","):
    cfg = wl.config(name); op = wl.make_operator(cfg); f = wl.make_input(cfg)
    c64 = cfg["dtype"] == "c64"
    kw = {"n_wedges": int(sys.argv[5])} if len(sys.argv) > 5 and int(sys.argv[5]) > 0 else {}
    plan = fio.Plan(op.N, op.c1, op.c2, eps=cfg["eps"], dtype=cfg["dtype"], device=0,
                    wedge_overlap=float(sys.argv[4]) if len(sys.argv) > 4 else 0.0, **kw)
    t = torch.from_numpy(f).to("cuda:0", torch.complex64 if c64 else torch.complex128)
    out = torch.empty_like(t)
    for _ in range(3): plan.apply(t, out=out)
    torch.cuda.synchronize()
    steps = int(sys.argv[3])
    plan.profile_begin(steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): plan.apply(t, out=out)
    e1.record(); torch.cuda.synchronize()
    st = plan.profile_end()
    g = torch.empty_like(t)
    plan.apply_adjoint(t, out=g); torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(3): plan.apply_adjoint(t, out=g)
    a1.record(); torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.complex128)
    refp = f"/tmp/fio_var_first_{name}.npy"  # written by the first variant of this tool invocation
    if sys.argv[6] == "1":
        np.save(refp, got)
    ref = np.load(refp)
    dev = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    info = plan.info
    res[name] = {"ms": e0.elapsed_time(e1) / steps, "stages": {k: st[k] / max(st["n"], 1) for k in fio.STAGES},
                 "adj_ms": a0.elapsed_time(a1) / 3, "dev": dev,
                 "sum_q": info["sum_q"], "slots": info["slots"], "slot_terms": info["slot_terms"],
                 "alpha_GB": info["alpha_bytes"] / 1e9, "group_p": info["group_p"],
                 "k3_thread_slots": info["k3_thread_slots"], "max_tile_cap": info["max_tile_cap"],
                 "fine_elems": info["fine_elems"], "wedge_overlap": info["wedge_overlap"]}
    plan.close()
print("RESULT " + json.dumps(res))
'''


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    opts = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("--"))
    configs = opts.get("configs", "cfg3_c64,cfg3_c128")
    steps = opts.get("steps", "10")
    out = {}
    for vi, spec in enumerate(args):
        name, flags = spec.split("=", 1) if "=" in spec else (spec, "")
        d = f"/tmp/fio_var_{name}"
        if os.path.exists(d):
            shutil.rmtree(d)
        shutil.copytree(ROOT, d, ignore=shutil.ignore_patterns(".git", "gpurun_out", "profiles", "*.ncu-rep"))
        if spec.split("=", 1)[-1].split("@")[0] == "" :
            pass  # product build: the in-tree .so is rebuilt below with no extra flags
        runenv = {}
        if "@" in flags:  # NAME=FLAGS@ENV=V,ENV2=V2: run-time environment of the variant
            flags, e = flags.split("@", 1)
            runenv = dict(kv.split("=", 1) for kv in e.split(",") if kv)
        env = dict(os.environ, FIO_NVCC_FLAGS=flags)
        subprocess.check_call([sys.executable, "-c", "from paper_math_0610051_b200 import build; build.build(force=True)"],
                              cwd=d, env=env)
        r = subprocess.run([sys.executable, "-c", CHILD, d, configs, steps, opts.get("overlap", "0"),
                            opts.get("wedges", "0"), "1" if vi == 0 else "0"], cwd=d,
                           capture_output=True, text=True,
                           env=dict(os.environ, **runenv))
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        out[name] = {"flags": flags, **(json.loads(line[0][7:]) if line else {"error": r.stderr[-2000:]})}
        print(name, json.dumps(out[name]), flush=True)
    print("ALL " + json.dumps(out))


if __name__ == "__main__":
    main()
