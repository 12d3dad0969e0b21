"""Markdown summary of ncu --set full reports (one launch each): time, DRAM
bytes, throughputs, occupancy, FP64 pipe, top stall reasons.
  python scripts/ncu_summary.py a.ncu-rep [b.ncu-rep ...] > summary.md"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % (active cycles)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_active.avg", "SM active cycles"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2]


for rep in sys.argv[1:]:
    h, u, v = raw(rep)
    d = dict(zip(h, zip(v, u)))
    name = d.get("Kernel Name", ("?", ""))[0]
    print(f"## {rep.split('/')[-1]}: `{name[:110]}`\n")
    print("| metric | value |\n|---|---|")
    for k, label in KEYS:
        if k in d:
            print(f"| {label} | {d[k][0]} {d[k][1]} |")
    stalls = []
    for k, (val, unit) in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls.append((float(val.replace(",", "")), k.split("stalled_")[1]))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    top = ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:6])
    print(f"\nwarp-state samples: {top}\n")
