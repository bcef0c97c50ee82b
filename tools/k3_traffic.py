"""Sum the DRAM bytes of all K3 launches of one apply from ncu --csv metric dumps.

usage: python tools/k3_traffic.py OUT.json cfg=path.csv:SUM_Q:MAX_TILE_CAP [...]
Each csv comes from
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k_interp_groups --csv python tools/run_apply.py CFG 1
(every K3 launch of one apply, cold cache per launch); SUM_Q and MAX_TILE_CAP are the plan's sum of
separation ranks and largest K3 chunk footprint (printed by run_apply.py), so bench.py uses the capture
only for the plan (and K3 chunking) it was taken on.
"""
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}


def parse(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iid, iname, iunit, ival = (h.index(k) for k in ("ID", "Metric Name", "Metric Unit", "Metric Value"))
    acc = {}
    ids = set()
    for r in rows[1:]:
        ids.add(r[iid])
        v = float(r[ival].replace(",", "")) * SCALE.get(r[iunit], 1.0)
        acc[r[iname]] = acc.get(r[iname], 0.0) + v
    return len(ids), acc


def main():
    out = {}
    for arg in sys.argv[2:]:
        cfg, rest = arg.split("=", 1)
        path, sum_q, cap = rest.rsplit(":", 2)
        n, acc = parse(path)
        rd, wr = acc.get("dram__bytes_read.sum", 0.0), acc.get("dram__bytes_write.sum", 0.0)
        out[cfg] = {"launches": n, "sum_q": int(sum_q), "max_tile_cap": int(cap), "dram_read_bytes": rd, "dram_write_bytes": wr,
                    "dram_bytes": rd + wr,
                    "ncu_time_s": acc.get("gpu__time_duration.sum", 0.0),
                    "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                           f"--clock-control none -k regex:k_interp_groups, python tools/run_apply.py {cfg} 1 "
                           "(all K3 launches of one apply; cold cache per launch)"}
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
