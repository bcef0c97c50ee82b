"""Top SASS instructions of one kernel by warp-stall samples (ncu --page source, SASS view).

usage: python tools/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import subprocess
import sys


def main(path, kregex, n=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kregex}"], capture_output=True, text=True).stdout
    import re
    lines = out.splitlines()
    # one section per kernel: '"Kernel Name","<name>"' then the table
    sec, keep = [], False
    for l in lines:
        if l.startswith('"Kernel Name"'):
            keep = re.search(kregex, l) is not None and not sec
            continue
        if keep:
            sec.append(l)
    rows = list(csv.reader(sec))
    h = rows[0]
    ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[1:] if len(r) == len(h)]
    tot = sum(float(r[iss] or 0) for r in body)
    body.sort(key=lambda r: -float(r[iss] or 0))
    print(f"total samples {tot:.0f}")
    for r in body[:n]:
        print(f"{float(r[iss]) / tot * 100:5.1f}%  {r[ia][-5:]}  {r[isrc].strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
