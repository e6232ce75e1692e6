"""Print the kernel launch list (last rep) of gpurun_out/sb_launches.csv."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sb_launches.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
d = rows[hi + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
ks = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", "")) / 1e3) for r in d]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = len(ks) // reps
tot = 0
for k, t in ks[(reps - 1) * n:]:
    tot += t
    print(f"{k[:70]:70s} {t:8.1f}")
print("total", round(tot, 1), "launches", n)
