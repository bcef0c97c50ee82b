"""Per-kernel SASS instruction mix of the built library (cuobjdump -sass), for the hot kernels.

    python tools/sass_summary.py [path/to/libfio_b200.so] > profiles/r02_sass_summary.txt

Counts static instructions by mnemonic family -- the evidence that K3 uses TMA (UTMALDG: tensor-map
tile loads; UBLKCP: cp.async.bulk), mbarriers (SYNCS), cp.async (LDGSTS), and which FMA pipe it feeds
(DFMA for complex128, FFMA2 packed FP32 for complex64)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAMILIES = ["UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "DFMA", "DMUL", "DADD", "FFMA2", "FMUL2", "FADD2", "FFMA",
            "LDS", "STS", "LDG", "STG", "RED", "ATOMG", "SHFL", "BAR", "MUFU", "HMMA", "UTCMMA", "UTCHMMA"]
HOT = [
    ("K3 c128 w7 (headline)", r"k_interp_groupsI7double2Li7ELi4ELi1E"),
    ("K3 c64 w5", r"k_interp_groupsI6float2Li5ELi4ELi1E"),
    ("K3 c128 w7, 2 RHS", r"k_interp_groupsI7double2Li7ELi4ELi2E"),
    ("K1 rowpass c128", r"k_rowpassI7double2"),
    ("K2 colpass c128", r"k_colpassI7double2"),
    ("K0 rows c128", r"k_fft_rowsI7double2"),
    ("adjoint spread c128 w7", r"k_spread_groupsI7double2Li7ELi4E"),
]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_math_0610051_b200", "libfio_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            funcs[cur].append(m.group(1))
    print(f"# static SASS instruction counts per kernel ({os.path.basename(lib)}, sm_100a; cuobjdump -sass)")
    print("# family: " + ", ".join(FAMILIES))
    for label, pat in HOT:
        names = [n for n in funcs if re.search(pat, n)]
        if not names:
            print(f"{label}: not found")
            continue
        c = collections.Counter(funcs[names[0]])
        fam = {f: sum(v for k, v in c.items() if k == f) for f in FAMILIES}
        tot = sum(c.values())
        print(f"\n{label}  [{names[0][:90]}]  total {tot}")
        print("  " + "  ".join(f"{f} {fam[f]}" for f in FAMILIES if fam[f]))


if __name__ == "__main__":
    main()
