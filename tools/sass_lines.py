"""Join an ncu SASS source page (--page source --csv --print-source sass)
with nvdisasm line info (-g) of the same cubin: warp instructions executed
per CUDA source line (file:line), top N.

    python tools/sass_lines.py <sass.csv> <cubin> <mangled-kernel-substring> [N]
"""
import csv
import re
import subprocess
import sys
from collections import Counter


def line_map(cubin, fun):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur = None
    loc = None
    res = {}
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur and fun in cur:
            res[int(m.group(1), 16)] = loc
    return res


def main():
    csvf, cubin, fun = sys.argv[1:4]
    N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lm = line_map(cubin, fun)
    rows = list(csv.reader(open(csvf)))
    hdr = rows[1]
    ai, ei, si = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
    base = None
    by = Counter()
    tot = 0
    ops = Counter()
    for r in rows[2:]:
        if len(r) <= ei or not r[ai].startswith("0x"):
            continue
        a = int(r[ai], 16)
        base = a if base is None else base
        n = int(r[ei] or 0)
        tot += n
        by[lm.get(a - base, ("?", 0))] += n
        op = r[si].split()[0] if r[si].split() else "?"
        if op.startswith("@"):
            op = r[si].split()[1]
        ops[op.split(".")[0]] += n
    print("total warp instructions", tot)
    for (f, l), n in by.most_common(N):
        print(f"{n:12d} {100 * n / tot:5.1f}%  {f}:{l}")
    print("ops:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in ops.most_common(25)))


if __name__ == "__main__":
    main()
