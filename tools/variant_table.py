"""Format tools/k3_variants.py logs as the rows of profiles/r02_k3_variants.txt.

    python tools/variant_table.py gpurun_out/var17.log [...] >> profiles/r02_k3_variants.txt"""
import json
import sys


def rows(path):
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
            out.append(f"  {name:8s} {d['flags'][:70]:70s} {cfg:10s} K3 {r['stages']['K3_interp']:7.3f}  apply "
                       f"{r['ms']:7.3f}  err {r['err']:.2e}  P {r.get('group_p')}")
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("\n".join(rows(p)))
