"""Executed instructions and stall samples per CUDA source line of one kernel in an
ncu report (captured with --import-source on, built with -lineinfo):
python tools/line_mix.py REPORT.ncu-rep KERNEL_REGEX [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "-c", "1", "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, data, hdr = "?", [], None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    ei, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    try:
        n, m = float(r[ei]), float(r[si])
    except ValueError:
        continue
    if n > 0 or m > 0:
        data.append((n, m, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot, tots = sum(d[0] for d in data), sum(d[1] for d in data)
print(f"total {tot / 1e6:.2f}M warp instructions, {tots:.0f} stall samples")
for n, m, loc, src in sorted(data, reverse=True)[:top]:
    print(f"{n / 1e6:7.2f}M {100 * n / tot:5.1f}%  smp {100 * m / max(tots, 1):5.1f}%  {loc:18s} {src}")
