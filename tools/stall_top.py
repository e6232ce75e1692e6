"""Top SASS lines by warp-stall samples of an ncu report: python tools/stall_top.py rep [n] [context]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = r[2:]
ai, si, st, ie = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"))
tot = sum(float(x[st] or 0) for x in rows)
print("total samples", tot, "instructions", sum(float(x[ie] or 0) for x in rows))
for x in sorted(rows, key=lambda x: -float(x[st] or 0))[:n]:
    print(x[ai][-5:], x[si][:80].ljust(80), x[st], x[ie])
