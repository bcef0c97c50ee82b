"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel.

usage: python tools/launch_summary.py launches.csv
Apply kernels (K0-K3, the K3 accumulator) get their share of the summed apply time; plan kernels
are listed without a share.  ncu serialises launches with a cold cache, so the shares (not the
absolute times) are what compare with bench.py's stage_ms.
"""
import csv
import sys

APPLY = {"k_fft_rows", "k_fft_cols", "k_rowpass", "k_colpass", "k_interp_groups", "k_accum", "k_dc_only"}
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ik, iu, iv = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
    agg = {}
    order = []
    for r in rows[1:]:
        name = r[ik].split("(")[0].split("<")[0].replace("void ", "").replace("fio::", "").strip()
        ms = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1e-6)
        if name not in agg:
            agg[name] = [0, 0.0]
            order.append(name)
        agg[name][0] += 1
        agg[name][1] += ms
    tot_apply = sum(v[1] for k, v in agg.items() if k in APPLY)
    for k in order:
        n, ms = agg[k]
        share = f"  share_of_apply={ms / tot_apply:.3f}" if k in APPLY and tot_apply > 0 else ""
        print(f"{k:32s} launches={n:5d} total_ms={ms:10.3f}{share}")


if __name__ == "__main__":
    main(sys.argv[1])
