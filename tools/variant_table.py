"""Format tools/k3_variants.py logs as the rows of profiles/r02_k3_variants.txt.

    python tools/variant_table.py [--k12] gpurun_out/var17.log [...] >> profiles/r02_k3_variants.txt
(--k12: also the K1 / K2 stage times)"""
import json
import sys


def rows(path, with_k12=False):
    out = [f"\n== {path.rsplit('/', 1)[-1]}"]
    for line in open(path):
        if line.startswith("ALL") or "{" not in line:
            continue
        name, js = line.split(" ", 1)
        try:
            d = json.loads(js)
        except json.JSONDecodeError:
            continue
        for cfg, r in d.items():
            if cfg == "flags" or not isinstance(r, dict):
                continue
            st = r["stages"]
            k12 = f"K1 {st['K1_rowpass']:6.3f} K2 {st['K2_colpass']:6.3f}  " if with_k12 else ""
            out.append(f"  {name:8s} {d['flags'][:70]:70s} {cfg:10s} {k12}K3 {st['K3_interp']:7.3f}  apply "
                       f"{r['ms']:7.3f}  " + (f"err {r['err']:.2e}" if "err" in r else f"dev {r['dev']:.1e}") +
                       f"  P {r.get('group_p')}")
    return out


if __name__ == "__main__":
    k12 = "--k12" in sys.argv
    for p in sys.argv[1:]:
        if p != "--k12":
            print("\n".join(rows(p, k12)))
