"""Summarise one ncu report of K3: occupancy, pipes, shared-memory wavefronts/conflicts, stall mix,
and the share of stall samples per kernel region (prologue vs term loop vs epilogue).
    python tools/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]
for k in want:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
print("stalls (per issue):")
for k, x in zip(h, v):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            if float(x) > 0.05:
                print(f"   {k[34:-23]:28s} {float(x):.2f}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ia, isrc, iss = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
data = [(int(x[ia], 16), x[isrc], float(x[iss] or 0)) for x in rows[2:]]
tot = sum(d[2] for d in data) or 1
bars = [a for a, s, _ in data if "BAR.SYNC" in s]
if len(bars) >= 2:
    b1 = bars[1]
    pro = sum(x for a, s, x in data if a < b1)
    print(f"samples before the term loop barrier: {pro / tot:.2%}")
top = sorted(data, key=lambda t: -t[2])[:12]
for a, s, x in top:
    print(f"   {x / tot:6.2%}  {s[:80]}")
