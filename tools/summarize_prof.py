"""Summarise gpurun_out/ ncu outputs into profiles/<round>_*.

    python tools/summarize_prof.py r01

Writes profiles/<round>_launches.md (per-kernel device time of one bench run,
cold-cache and serialised: compare SHARES), profiles/<round>_force_kernel.md
(key metrics of one full k_force capture) and profiles/force_kernel_ncu.json
(DRAM traffic per launch, read by bench.py for roofline.traffic).
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
OUT = REPO / "gpurun_out"
PROF = REPO / "profiles"


def launches(tag):
    rows = list(csv.reader(open(OUT / "launches.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) / 1e3
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"# {tag}: kernel launch list of `python bench.py --steps 20 --warmup 5 --no-cpu-baseline`",
             "", "ncu `--metrics gpu__time_duration.sum --clock-control none` (every launch; cold cache,",
             "serialised: compare shares, not absolutes).  Whole run incl. warm-up and the e2e phase.", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% |")
    lines.append(f"| **total** | {sum(cnt.values())} | {T:.1f} | 100% |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")


def ncu_csv(page, rep):
    r = subprocess.run(["ncu", "-i", str(rep), "--page", page, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def force(tag):
    rep = OUT / "force_prof.ncu-rep"
    det = ncu_csv("details", rep)
    hdr = det[0]
    want = ["Duration", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
            "Theoretical Occupancy", "Achieved Occupancy", "No Eligible", "Executed Instructions",
            "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Memory Throughput"]
    name = ""
    vals = {}
    for row in det[1:]:
        d = dict(zip(hdr, row))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in want and d["Metric Name"] not in vals:
            vals[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    raw = ncu_csv("raw", rep)
    rh, rv = raw[0], raw[2]
    R = dict(zip(rh, rv))
    rd = float(R.get("dram__bytes_read.sum", "0").replace(",", ""))
    wr = float(R.get("dram__bytes_write.sum", "0").replace(",", ""))
    unit = raw[1][rh.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in rh else ""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    traffic = (rd + wr) * scale
    pipes = {k: R[k] for k in rh if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active")
             and any(p in k for p in ("fma.", "alu.", "lsu.", "fp64.", "xu."))}
    stalls = {k.split("stalled_")[1]: R[k] for k in rh if k.startswith("smsp__pcsamp_warps_issue_stalled")
              and not k.endswith("not_issued") and float(R[k] or 0) > 100}
    lines = [f"# {tag}: one full ncu capture of `{name[:80]}`", "",
             "`ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1` on the bench command",
             "(96k SPC water, Ewald, m = 4, G = 4 groups).", "", "| metric | value |", "|---|---|"]
    lines += [f"| {k} | {v} |" for k, v in vals.items()]
    lines += [f"| DRAM read + write per launch | {traffic / 1e6:.1f} MB |"]
    lines += ["", "Pipe utilisation (% of peak, active cycles):", ""]
    lines += [f"- `{k}`: {v}" for k, v in pipes.items()]
    lines += ["", "Warp stall samples (> 100):", ""]
    lines += [f"- {k}: {v}" for k, v in sorted(stalls.items(), key=lambda x: -float(x[1]))]
    (PROF / f"{tag}_force_kernel.md").write_text("\n".join(lines) + "\n")
    (PROF / "force_kernel_ncu.json").write_text(json.dumps(
        {"kernel": name, "dram_bytes_per_launch": traffic, "round": tag, "source": f"profiles/{tag}_force_kernel.md"},
        indent=1) + "\n")


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    PROF.mkdir(exist_ok=True)
    launches(tag)
    force(tag)
    print((PROF / f"{tag}_force_kernel.md").read_text())
