"""Summarise ncu captures for profiles/ (run here, on the CPU box).

    python profiles/summarize.py gpurun_out/prof.ncu-rep > profiles/rNN_<name>.txt
    python profiles/summarize.py --launches gpurun_out/launches.csv > profiles/rNN_launches.txt

For every profiled kernel: duration, DRAM bytes, instruction count, issue /
occupancy, FP64 pipe use, top stall reasons and the SASS opcode mix per
executed warp instruction (from the source page).
"""

import csv
import io
import re
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def summarize(rep):
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    h, units = raw[0], raw[1]
    for r in raw[2:]:
        print(f"== {r[h.index('Kernel Name')]}")
        for key, label in KEYS:
            if key in h:
                print(f"   {label:22s} {r[h.index(key)]} {units[h.index(key)]}")
        stalls = []
        for i, col in enumerate(h):
            if col.startswith("smsp__average_warps_issue_stalled") and \
                    col.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), col.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        print("   stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls)[::-1][:6]))
    src = ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"])
    kern, hdr = None, None
    mix = defaultdict(Counter)
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "Kernel Name":
            kern = r[1]
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        try:
            e = int(r[hdr.index("Instructions Executed")])
        except (TypeError, ValueError, IndexError):
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[hdr.index("Source")].strip())
        if m:
            mix[kern][m.group(2)] += e
    for k, c in mix.items():
        tot = sum(c.values())
        print(f"-- SASS mix {k[:60]} (executed warp instructions, share)")
        print("   " + ", ".join(f"{op} {v / tot:.1%}" for op, v in c.most_common(24)))


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(j for j, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    per = defaultdict(list)
    for r in rows[i + 1:]:
        if len(r) > h.index("Metric Value") and r[h.index("Metric Name")] == "gpu__time_duration.sum":
            per[r[h.index("Kernel Name")]].append(float(r[h.index("Metric Value")]))
    tot = sum(sum(v) for v in per.values())
    print(f"{'kernel':70s} {'n':>4s} {'mean ns':>12s} {'share':>7s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:70]:70s} {len(v):4d} {sum(v) / len(v):12.0f} {sum(v) / tot:7.1%}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summarize(sys.argv[1])
