"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) into a markdown table:
launches, total device time, share, DRAM bytes per kernel.
    python tools/launch_summary.py launches.csv "title" > profiles/x.md"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
agg = defaultdict(lambda: {"n": set(), "t": 0.0, "dram": 0.0})
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", ""))
    a = agg[name]
    a["n"].add(r[ii])
    if r[mi] == "gpu__time_duration.sum":
        a["t"] += v / 1e3 if "nsecond" in "".join(r) else v / 1e3
    else:
        a["dram"] += v
tot = sum(a["t"] for a in agg.values())
title = sys.argv[2] if len(sys.argv) > 2 else "launch list"
print(f"# {title}\n")
print("ncu `--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` "
      "(every launch; cold cache, serialised: compare shares, not absolutes).\n")
print("| kernel | launches | total us | share | DRAM MB per launch |")
print("|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda x: -x[1]["t"]):
    n = len(a["n"])
    print(f"| `{k[:90]}` | {n} | {a['t']:.1f} | {100 * a['t'] / tot:.1f}% | {a['dram'] / max(n, 1) / 1e6:.2f} |")
print(f"| **total** | {sum(len(a['n']) for a in agg.values())} | {tot:.1f} | 100% | |")
