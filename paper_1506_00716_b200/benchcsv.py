"""The reference's benchmark table (`clustermd bench`, cli.py:424-516) on the
GPU path: for every (layout, workers, rebuild interval) the median MD step
rate over repeats of run_md, ns/day, the pair and useful-flop ratios of a
fresh list, the step-time shares of forces / lifecycle / integration and the
step-0 total energy, written in the same versioned CSV schema
(`# clustermd-bench-csv-v1`, sixteen columns).  The command-line front end is
out of scope; this is the function behind it."""

from __future__ import annotations

import statistics

from .engine import ListPolicy, run_md
from .gridder import build_cluster_grid
from .kernels import KernelLayout, flop_count
from .model import NonbondedParams, ParameterError, ParticleSystem
from .pairlist import build_pair_list, interaction_stats, prune_pair_list

BENCH_CSV_HEADER = "# clustermd-bench-csv-v1"
BENCH_COLUMNS = ("m", "n_lane", "supercluster", "workers", "rebuild_interval", "steps", "repeats",
                 "steps_per_s_median", "steps_per_s_spread", "ns_per_day", "pair_ratio", "useful_flop_ratio",
                 "share_forces", "share_lifecycle", "share_integrate", "e_total_step0")


def bench_rows(system: ParticleSystem, params: NonbondedParams, *, layouts=((4, 4),), workers_list=(1,),
               rebuild_intervals=(10,), steps: int = 100, repeats: int = 3, dt: float = 2e-3,
               supercluster: int = 1, prune: bool = True, target_occupancy=None) -> list[list]:
    """One row per (layout, workers, rebuild interval), the reference's
    columns and value rules (rates from the TimingReport "step" section,
    spread = (max - min) / median, ns/day = rate * dt * 86.4)."""
    if steps < 1 or repeats < 1:
        raise ParameterError(f"steps and repeats must be >= 1, got {steps}, {repeats}")
    rows = []
    for m, n_lane in layouts:
        layout = KernelLayout(m=m, n_lane=n_lane)
        for workers in workers_list:
            for interval in rebuild_intervals:
                policy = ListPolicy(rebuild_interval=interval, prune_on_build=prune)
                rates, last = [], None
                for _ in range(repeats):
                    res = run_md(system, params, layout, dt, steps, supercluster_size=supercluster, policy=policy,
                                 workers=workers, report_interval=max(steps, 1), target_occupancy=target_occupancy)
                    wall = res.timing.total("step")
                    rates.append(steps / wall if wall > 0 else 0.0)
                    last = res
                med = statistics.median(rates)
                spread = (max(rates) - min(rates)) / med if med else 0.0
                grid = build_cluster_grid(system, m, target_occupancy)
                plist = build_pair_list(grid, system.box, params.r_list, supercluster_size=supercluster,
                                        n_lane=n_lane)
                if prune:
                    plist = prune_pair_list(plist, grid.clustered_positions, system.box)
                stats = interaction_stats(plist, grid, grid.clustered_positions, system.box, params.r_cut)
                flops = flop_count(plist, grid, layout, system.box, params.r_cut)
                secs = last.timing.sections
                step_total = last.timing.total("step") or 1.0
                share = {k: (secs[k][1] / step_total if k in secs else 0.0)
                         for k in ("forces", "lifecycle", "integrate")}
                rows.append([m, n_lane, supercluster, workers, interval, steps, repeats, repr(med), repr(spread),
                             repr(med * dt * 86.4), repr(stats.ratio), repr(flops.ratio),
                             repr(share["forces"]), repr(share["lifecycle"]), repr(share["integrate"]),
                             repr(float(last.e_total[0]))])
    return rows


def bench_csv(system: ParticleSystem, params: NonbondedParams, path=None, **kw) -> str:
    """The CSV text (header line, column line, one line per row); written to
    ``path`` when given."""
    lines = [BENCH_CSV_HEADER, ",".join(BENCH_COLUMNS)]
    lines += [",".join(str(v) for v in row) for row in bench_rows(system, params, **kw)]
    text = "\n".join(lines) + "\n"
    if path is not None:
        with open(path, "w") as fh:
            fh.write(text)
    return text
