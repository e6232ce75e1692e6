"""Group an ncu source-page (SASS) export by execution count: which code
regions (per-iteration overhead, member sweeps, per-group work) take the
instructions and the stall samples.
    ncu -i REP --page source --csv --print-source sass > src.csv
    python tools/src_profile.py src.csv [--dump out.txt]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 1 and r[0].startswith("0x")]
iA, iS = hdr.index("Address"), hdr.index("Source")
iW, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = int(data[0][iA], 16)
out = [(int(r[iA], 16) - base, r[iS].strip(), int(r[iW]), int(r[iE])) for r in data]
tot_w = sum(o[2] for o in out)
tot_e = sum(o[3] for o in out)
print(f"instructions {tot_e / 1e6:.2f} M warp-instr, {tot_w} stall samples, {len(out)} SASS lines")
by = defaultdict(lambda: [0, 0, 0])
for off, s, w, e in out:
    by[e][0] += 1
    by[e][1] += w
    by[e][2] += e
for k, (n, w, e) in sorted(by.items(), key=lambda x: -x[1][1])[:14]:
    print(f"exec={k:8d} n_instr={n:4d} samples={w:5d} ({100 * w / tot_w:4.1f}%) warp-instr={e / 1e6:6.2f}M")
if "--dump" in sys.argv:
    with open(sys.argv[sys.argv.index("--dump") + 1], "w") as f:
        for off, s, w, e in out:
            f.write(f"{off:05x} {e:9d} {w:6d}  {s}\n")
