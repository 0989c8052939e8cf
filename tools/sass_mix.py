"""Aggregate an ncu report's SASS source page by opcode: executed warp
instructions and stall samples.  usage: sass_mix.py REPORT KERNEL_REGEX"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      "regex:" + kre, "--print-source=sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rd = csv.DictReader(io.StringIO("\n".join(lines[start:])))
ins, smp = Counter(), Counter()
tot_i = tot_s = 0
for r in rd:
    try:
        n = int(r["Instructions Executed"] or 0)
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    except (ValueError, KeyError):
        continue
    op = r["Source"].split()
    op = [t for t in op if not t.startswith("@")]
    op = op[0] if op else "?"
    ins[op] += n
    smp[op] += s
    tot_i += n
    tot_s += s
print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
for op, n in ins.most_common(40):
    print(f"{op:28s} {n:14,d} {100*n/tot_i:6.2f}%   samples {100*smp[op]/max(tot_s,1):6.2f}%")
