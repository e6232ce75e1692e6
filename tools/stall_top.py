"""Top SASS lines by warp-stall samples of an ncu report: python tools/stall_top.py rep [n] [context]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
hi = [i for i, x in enumerate(r) if "Address" in x][0]
h = r[hi]
rows = [x for x in r[hi + 1:] if len(x) == len(h) and x[0] != "Address"]
ai, si, st, ie = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"))
def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


tot = sum(f(x[st]) for x in rows)
print("total samples", tot, "instructions", sum(f(x[ie]) for x in rows))
for x in sorted(rows, key=lambda x: -f(x[st]))[:n]:
    print(x[ai][-5:], x[si][:80].ljust(80), x[st], x[ie])
