#!/usr/bin/env python
"""Top CUDA source lines by warp-stall samples from an ncu report (needs -lineinfo builds).

    python profiles/srcstall.py REPORT.ncu-rep [kernel-regex] [launch-index] [top]
"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kre}", "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True,
                     text=True).stdout


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


fname, hdr, lines = "?", None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
    elif r[0] == "Function Name":
        func = r[1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        lines.append((f(r[4]), fname, r[0], r[1].strip()))
tot = sum(x[0] for x in lines) or 1.0
print(func[:120], "| stall samples", int(tot))
for s, fn, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
    print("%6.1f%%  %s:%-5s %s" % (100 * s / tot, fn, ln, src[:100]))
