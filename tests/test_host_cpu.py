"""CPU tests of the product's host logic and of the C ABI (no GPU: no compute calls).

- the library builds, loads and exports every entry point include/fio.h declares;
- the wedge partition agrees with the oracle's independent
  classification, covers Omega \\ {0} exactly once, and every lattice relabeling
   is unimodular and injective into its box;
- the wedge -> rank assignment covers every wedge once and is deterministic;
- the product refuses to run without CUDA (no CPU fallback).
"""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import workloads as wl
import paper_math_0610051_b200 as fio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fio.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fio_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = fio.load_library()
    decl = declared_symbols()
    assert len(decl) >= 10
    nm = subprocess.run(["nm", "-D", "--defined-only", fio.library_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(fio_\w+)", nm))
    for name in decl:
        assert name in exported, name
        getattr(lib, name)
    assert set(fio.SYMBOLS) == set(decl)
    assert b"sm_100a" in lib.fio_version()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", fio.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


@pytest.mark.parametrize("N,W", [(64, 8), (40, 16), (256, 16), (96, 24)])
def test_partition_matches_oracle_and_is_exact(N, W):
    g = fio.geometry(N, W)
    wo = g["wedge_of"]
    xi1, xi2 = wl.freqs(N)
    ref = np.vectorize(lambda a, b: oracle.wedge_of(W, int(a), int(b)))(xi1, xi2)
    assert np.array_equal(wo, ref)
    assert wo[0, 0] == -1 and (wo >= 0).sum() == N * N - 1
    assert set(np.unique(wo[wo >= 0])) == set(range(W))


@pytest.mark.parametrize("N,W", [(64, 8), (256, 16), (1024, 32)])
def test_lattice_boxes_are_exact_relabelings(N, W):
    g = fio.geometry(N, W)
    xi1, xi2 = wl.freqs(N)
    total_fine = 0
    for l in range(W):
        M = g["M"][l]
        assert round(np.linalg.det(M)) == 1 and np.all(np.abs(M) <= 3)
        m = g["wedge_of"] == l
        z = np.stack([xi1[m], xi2[m]], 1) @ M.T - g["xc"][l]
        n1, n2 = g["box"][l]
        i1, i2 = z[:, 0] + n1 // 2, z[:, 1] + n2 // 2
        assert i1.min() >= 0 and i1.max() < n1 and i2.min() >= 0 and i2.max() < n2
        assert len(np.unique(i1 * n2 + i2)) == m.sum()          # injective
        n1f, n2f = g["fine"][l]
        assert n1f == 2 * n1 and n2f == 2 * n2                   # oversampling sigma = 2
        for n in (n1f, n2f):
            k = n
            for p in (2, 3, 5):
                while k % p == 0:
                    k //= p
            assert k == 1                                        # 5-smooth FFT lengths
        total_fine += n1f * n2f
    if N == 1024:
        assert total_fine < 9.0 * N * N  # sheared boxes keep the fine volume near 8.8 N^2


def test_wedge_assignment_lpt():
    rng = np.random.default_rng(3)
    cost = rng.uniform(1, 2, 32)
    for R in (1, 2, 3, 8):
        owner = fio.assign_wedges(cost, R)
        assert owner.min() >= 0 and owner.max() < R and len(owner) == 32
        loads = np.bincount(owner, weights=cost, minlength=R)
        assert loads.max() - loads.min() <= cost.max() + 1e-12   # LPT bound
        assert np.array_equal(owner, fio.assign_wedges(cost, R))


def test_no_cpu_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    op = wl.grt_operator(64)
    with pytest.raises(fio.FioError):
        fio.Plan(64, op.c1, op.c2)


def test_plan_load_rejects_missing_and_malformed_files(tmp_path):
    # fio_plan_load validates the file before touching the GPU (include/fio.h)
    import ctypes
    lib = fio.load_library()
    N = 16
    c = np.full(N * N, 0.5)
    ph = fio._Phase(c.ctypes.data, c.ctypes.data, None, None, 1)
    amp = fio._Amp(0, None, None, 0)
    h = ctypes.c_void_p()
    st = lib.fio_plan_load(ctypes.byref(h), str(tmp_path / "missing.fio").encode(), N, ctypes.byref(ph),
                           ctypes.byref(amp), 1e-6, None)
    assert st == -1 and b"cannot open" in lib.fio_last_error()
    bad = tmp_path / "bad.fio"
    bad.write_bytes(b"not a plan file at all" * 8)
    st = lib.fio_plan_load(ctypes.byref(h), str(bad).encode(), N, ctypes.byref(ph), ctypes.byref(amp), 1e-6, None)
    assert st == -1 and b"not a valid plan file" in lib.fio_last_error()


@pytest.mark.parametrize("W,ov", [(16, 0.25), (8, 1.0), (24, 0.6), (16, 0.0)])
def test_product_partition_weights_match_oracle(W, ov):
    # the product's chi_l (C++, fio_partition_weights) against the oracle's independent numpy version
    # of the same definition (reading R2); overlap 0 is the paper's indicator
    N = 48
    xi1, xi2 = wl.freqs(N)
    ref = oracle.smooth_wedge_weights(N, W, ov) if ov > 0 else None
    for a in range(N):
        for b in range(N):
            got = fio.partition_weights(W, ov, int(xi1[a, b]), int(xi2[a, b]))
            if ov > 0:
                np.testing.assert_allclose(got, ref[:, a, b], atol=1e-13)
            else:
                exp_ = np.zeros(W)
                l = oracle.wedge_of(W, int(xi1[a, b]), int(xi2[a, b]))
                if l >= 0:
                    exp_[l] = 1.0
                assert np.array_equal(got, exp_)


def test_ctypes_structs_match_the_c_abi(tmp_path):
    # the binding's ctypes mirrors of fio_opts / fio_phase / fio_amplitude / fio_info must have the C
    # layout (fio_plan copies the whole fio_opts: a missing trailing field would be read as garbage)
    import ctypes
    structs = {"fio_opts": fio._Opts, "fio_phase": fio._Phase, "fio_amplitude": fio._Amp,
               "fio_info": fio._Info}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "fio.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                          check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_allgather_option_is_validated_before_any_device_work():
    # fio_opts.allgather (include/fio.h): only with a communicator, only 0 or 1 -- FIO_EINVAL otherwise
    import ctypes
    lib = fio.load_library()
    N = 16
    c = np.full(N * N, 0.5)
    ph = fio._Phase(c.ctypes.data, c.ctypes.data, None, None, 1)
    amp = fio._Amp(0, None, None, 0)
    for val, msg in [(1, b"needs a communicator"), (2, b"must be 0 or 1")]:
        o = fio._Opts()
        lib.fio_default_opts(ctypes.byref(o))
        assert o.allgather == 0
        o.allgather = val
        h = ctypes.c_void_p()
        st = lib.fio_plan(ctypes.byref(h), N, ctypes.byref(ph), ctypes.byref(amp), 1e-6, ctypes.byref(o))
        assert st == -1 and msg in lib.fio_last_error() and not h.value
