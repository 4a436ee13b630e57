"""Executed-instruction mix by SASS opcode from an ncu report's source page:
python tools/sass_mix.py REPORT.ncu-rep [top] [kernel-regex]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 24
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3], "-c", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si, ei = h.index("Source"), h.index("Instructions Executed")
smp = h.index("Warp Stall Sampling (All Samples)")
c, s = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= ei or not r[si].strip():
        continue
    try:
        n = float(r[ei])
        m = float(r[smp] or 0)
    except ValueError:
        continue
    op = r[si].strip().split()
    o = op[1] if op[0].startswith("@") else op[0]
    c[o.split(".")[0]] += n
    s[o.split(".")[0]] += m
tot, tots = sum(c.values()), sum(s.values())
print(f"{'opcode':10s} {'executed':>9s} {'%':>5s} {'stall smp %':>11s}")
for o, n in c.most_common(top):
    print(f"{o:10s} {n / 1e6:8.2f}M {100 * n / tot:5.1f} {100 * s[o] / max(tots, 1):10.1f}")
print(f"total {tot / 1e6:.2f}M warp instructions")
