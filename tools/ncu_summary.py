"""Summarise an ncu --set full report per kernel (the profiles/*_ncu.txt
format): time, DRAM bytes, warp instructions, issue / occupancy, pipes, hit
rates, the top stall reasons per issue and the SASS opcode mix.
usage: ncu_summary.py REPORT [KERNEL_REGEX]"""
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

ROWS = [("duration", "gpu__time_duration.sum"), ("dram read", "dram__bytes_read.sum"),
        ("dram write", "dram__bytes_write.sum"), ("warp instructions", "smsp__inst_executed.sum"),
        ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("registers/thread", "launch__registers_per_thread"), ("grid", "launch__grid_size"),
        ("block", "launch__block_size"),
        ("fp64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("fma pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("L1 hit %", "l1tex__t_sector_hit_rate.pct"), ("L2 hit %", "lts__t_sector_hit_rate.pct"),
        ("L1 LSU wavefronts %", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed")]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kre:
        cmd += ["-k", "regex:" + kre]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"]
        print(f"== {name}")
        for label, key in ROWS:
            if key in d:
                print(f"   {label:22s} {d[key]} {u.get(key, '')}".rstrip())
        st = {k[len(STALL):].replace("_per_issue_active.ratio", ""): float(v)
              for k, v in d.items() if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")
              and v not in ("", "n/a")}
        top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
        print("   stalls/issue: " + ", ".join(f"{k}={v:.2f}" for k, v in top))
        short = name.split("(")[0].split("::")[-1].split("<")[0]
        mix = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "sass_mix.py"),
                              rep, short], capture_output=True, text=True).stdout.splitlines()
        ops = []
        for ln in mix[1:25]:
            p = ln.split()
            if len(p) >= 3:
                ops.append(f"{p[0]} {p[2]}")
        print(f"-- SASS mix {short} (executed warp instructions, share)")
        print("   " + ", ".join(ops))


if __name__ == "__main__":
    main()
