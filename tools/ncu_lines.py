"""Per-source-line executed warp instructions and stall samples from an ncu
report (source page, CUDA+SASS correlated).  usage: ncu_lines.py REP KERNEL [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
path = ""
agg = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            agg.append((int(r[7]), int(r[4]), f"{path}:{r[0]}", r[1].strip()[:70]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1
tots = sum(a[1] for a in agg) or 1
print(f"total {tot:,} warp instructions, {tots:,} samples")
for n, smp, loc, src in sorted(agg, reverse=True)[:top]:
    print(f"{100*n/tot:5.1f}% {100*smp/tots:5.1f}%s {loc:24s} {src}")
