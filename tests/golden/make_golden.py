"""Generate golden vectors by running the REAL reference (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--large]

Imports clustermd read-only from /root/reference/pkg/src, runs its public API
(build_cluster_grid, build_pair_list, prune_pair_list, interaction_stats,
compute_nonbonded, compute_nonbonded_original, brute_force_nonbonded,
pair_interaction) on seeded inputs and stores inputs + outputs as compressed
npz files next to this script.  The GPU box never runs this script; tests
there only read the committed .npz files.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import clustermd as cm  # noqa: E402
from clustermd.cli import generate_system  # noqa: E402

from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402


def pack_bits(masks: np.ndarray) -> np.ndarray:
    rows, m, _ = masks.shape
    flat = masks.reshape(rows, m * m).astype(np.uint64)
    w = np.uint64(1) << np.arange(m * m, dtype=np.uint64)
    return (flat * w).sum(axis=1, dtype=np.uint64)


def uniform_system(n, box_lengths, seed, charged=False, n_types=1):
    """Same construction as the reference tests' helpers.uniform_system."""
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, 1.0, (n, 3)) * np.asarray(box_lengths)
    charges = np.zeros(n)
    if charged:
        charges = 0.1 * np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    return cm.ParticleSystem(positions=pos, velocities=np.zeros((n, 3)), masses=np.full(n, 39.948),
                             charges=charges, lj_type=(np.arange(n) % n_types).astype(np.int64),
                             box=cm.SimBox(box_lengths))


def type_table(n_types, base_eps=0.996, base_sig=0.34):
    eps = base_eps * (1.0 + 0.1 * np.arange(n_types))
    sig = base_sig * (1.0 - 0.05 * np.arange(n_types))
    t = np.empty((n_types, n_types, 2))
    for a in range(n_types):
        for b in range(n_types):
            t[a, b, 0] = np.sqrt(eps[a] * eps[b])
            t[a, b, 1] = 0.5 * (sig[a] + sig[b])
    return t


def dump_case(name, system, lj_table, *, m, r_cut, r_list, shift, occupancy=None,
              supercluster=1, brute=True):
    params = cm.NonbondedParams(r_cut=r_cut, r_list=r_list, lj_table=lj_table, shift_potential=shift)
    box = system.box
    grid = cm.build_cluster_grid(system, m, target_occupancy=occupancy)
    built = cm.build_pair_list(grid, box, r_list, supercluster_size=supercluster, n_lane=m)
    pruned = cm.prune_pair_list(built, grid.clustered_positions, box)
    layout = cm.KernelLayout(m=m, n_lane=m)
    res_c = cm.compute_nonbonded(pruned, grid, system.positions, system.charges, system.lj_type,
                                 params, box, layout)
    res_o = cm.compute_nonbonded_original(pruned, grid, system.positions, system.charges,
                                          system.lj_type, params, box, layout)
    stats = cm.interaction_stats(pruned, grid, grid.clustered_positions, box, r_cut)
    out = dict(
        positions=system.positions, charges=system.charges, lj_type=system.lj_type,
        masses=system.masses, box=box.lengths, lj_table=np.asarray(lj_table),
        m=m, r_cut=r_cut, r_list=r_list, shift=int(shift),
        occupancy=np.nan if occupancy is None else occupancy, supercluster=supercluster,
        # grid
        perm=grid.perm, inverse_perm=grid.inverse_perm, fill_mask=grid.fill_mask,
        cell_counts=np.asarray(grid.cell_counts), cell_of_cluster=grid.cell_of_cluster,
        clustered_positions=grid.clustered_positions, bboxes=grid.bboxes,
        # lists
        built_offsets=built.offsets, built_j=built.j_idx.astype(np.int32), built_masks=pack_bits(built.masks),
        pruned_offsets=pruned.offsets, pruned_j=pruned.j_idx.astype(np.int32),
        pruned_masks=pack_bits(pruned.masks),
        # forces
        f_clustered=res_c.forces, f_original=res_o.forces, e_lj=res_o.e_lj, e_coulomb=res_o.e_coulomb,
        n_admitted=stats.n_admitted, n_within=stats.n_within_cutoff,
    )
    if supercluster > 1:
        out.update(super_offsets=pruned.super_offsets, super_j=pruned.super_j_idx.astype(np.int32),
                   super_pair_idx=pruned.super_pair_idx.astype(np.int32),
                   built_super_offsets=built.super_offsets, built_super_j=built.super_j_idx.astype(np.int32),
                   built_super_pair_idx=built.super_pair_idx.astype(np.int32))
    if brute:
        bf = cm.brute_force_nonbonded(system, params)
        out.update(bf_forces=bf.forces, bf_e_lj=bf.e_lj, bf_e_coulomb=bf.e_coulomb)
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: n={system.n} clusters={grid.n_clusters} built={built.n_pairs} "
          f"pruned={pruned.n_pairs} admitted={stats.n_admitted} within={stats.n_within_cutoff}")


def spc(n, seed):
    s, table = spc_water(n, seed=seed)
    return cm.ParticleSystem(positions=s.positions, velocities=s.velocities, masses=s.masses,
                             charges=s.charges, lj_type=s.lj_type, box=cm.SimBox(s.box.lengths)), table


def main():
    # SPC water 3k (config 1): reference default grid and the tuned grid
    sys3k, tab = spc(3000, seed=2024)
    L = float(sys3k.box.lengths[0])
    dump_case("spc3k_default", sys3k, tab, m=4, r_cut=1.0, r_list=1.1, shift=True)
    dump_case("spc3k_tuned", sys3k, tab, m=4, r_cut=1.0, r_list=1.1, shift=True,
              occupancy=tuned_occupancy(3000, L, 4))
    dump_case("spc3k_tuned_m8", sys3k, tab, m=8, r_cut=1.0, r_list=1.1, shift=True,
              occupancy=tuned_occupancy(3000, L, 8))
    # reference-test style uniform systems: every cluster size, 2 types, charges
    for m, seed in ((1, 101), (2, 102), (4, 103), (8, 104)):
        s = uniform_system(300, [4.0, 3.6, 3.3], seed=seed, charged=True, n_types=2)
        dump_case(f"uniform_m{m}", s, type_table(2), m=m, r_cut=0.9, r_list=1.0, shift=(m % 2 == 0))
    s = uniform_system(500, [5.0, 5.0, 5.0], seed=46, charged=True, n_types=2)
    dump_case("uniform_super8", s, type_table(2), m=4, r_cut=0.9, r_list=1.0, shift=True, supercluster=8)
    # the reference's own fluid generators (cli.generate_system)
    s, table = generate_system("lj_fluid", 400, 20.0, 120.0, 44)
    dump_case("lj_fluid400", s, table, m=4, r_cut=0.9, r_list=1.0, shift=True)
    s, table = generate_system("charged_fluid", 600, 20.0, 120.0, 7)
    dump_case("charged_fluid600", s, table, m=4, r_cut=0.9, r_list=1.0, shift=False)

    # known-answer scalars (test_kernels.py:27-61, test_gridder.py:81-94)
    params = cm.NonbondedParams(r_cut=0.9, r_list=1.0, lj_table=np.array([[[0.0, 0.3]]]))
    e, fr = cm.pair_interaction(0.25, 0, 0, 1.0, -1.0, params)
    pos = np.zeros((6, 3))
    pos[:, 2] = [0.5, 0.5, 0.5, 0.2, 0.2, 0.9]
    tie = cm.ParticleSystem(positions=pos, velocities=np.zeros((6, 3)), masses=np.ones(6),
                            charges=np.zeros(6), lj_type=np.zeros(6, dtype=int), box=cm.SimBox([2.0, 2.0, 2.0]))
    g = cm.build_cluster_grid(tie, 2, target_occupancy=1000)
    np.savez_compressed(HERE / "scalars.npz", coulomb_e=e, coulomb_fr=fr, tie_perm=g.perm)
    print("scalars:", e, fr, g.perm.tolist())


def digest(*arrays) -> str:
    """SHA-256 over the arrays' bytes in a fixed dtype per array (see callers)."""
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def list_digest(plist) -> str:
    return digest(np.asarray(plist.offsets, dtype=np.int64), np.asarray(plist.j_idx, dtype=np.int64),
                  pack_bits(plist.masks))


def dump_large(name, n, *, m, tuned, r_cut=1.0, r_list=1.1, seed=2024, f64=False):
    """BASELINE-size case (24k / 96k SPC water): the reference's grid, built
    and pruned lists and counts as SHA-256 digests (the arrays are tens of MB),
    its forces in original order and its energies.  Positions are regenerated
    by systems.spc_water(n, seed) on the test side and pinned by their digest."""
    import time

    system, tab = spc(n, seed)
    L = float(system.box.lengths[0])
    occ = tuned_occupancy(n, L, m) if tuned else None
    params = cm.NonbondedParams(r_cut=r_cut, r_list=r_list, lj_table=tab, shift_potential=True)
    box = system.box
    t0 = time.time()
    grid = cm.build_cluster_grid(system, m, target_occupancy=occ)
    built = cm.build_pair_list(grid, box, r_list, n_lane=m)
    pruned = cm.prune_pair_list(built, grid.clustered_positions, box)
    layout = cm.KernelLayout(m=m, n_lane=m)
    res = cm.compute_nonbonded_original(pruned, grid, system.positions, system.charges, system.lj_type,
                                        params, box, layout)
    stats = cm.interaction_stats(pruned, grid, grid.clustered_positions, box, r_cut)
    out = dict(
        n=n, seed=seed, m=m, r_cut=r_cut, r_list=r_list, shift=1,
        occupancy=np.nan if occ is None else occ, box=box.lengths,
        positions_digest=digest(np.asarray(system.positions, dtype=np.float64)),
        n_clusters=grid.n_clusters, n_slots=grid.perm.shape[0],
        grid_digest=digest(np.asarray(grid.perm, dtype=np.int64), np.asarray(grid.fill_mask, dtype=np.bool_),
                           np.asarray(grid.cell_of_cluster, dtype=np.int64),
                           np.asarray(grid.bboxes, dtype=np.float64)),
        perm_digest=digest(np.asarray(grid.perm, dtype=np.int64)),
        bbox_digest=digest(np.asarray(grid.bboxes, dtype=np.float64)),
        built_rows=built.n_pairs, built_digest=list_digest(built),
        pruned_rows=pruned.n_pairs, pruned_digest=list_digest(pruned),
        pruned_offsets_digest=digest(np.asarray(pruned.offsets, dtype=np.int64)),
        n_admitted=stats.n_admitted, n_within=stats.n_within_cutoff,
        f_original=res.forces if f64 else res.forces.astype(np.float32),
        e_lj=res.e_lj, e_coulomb=res.e_coulomb,
    )
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: n={n} clusters={grid.n_clusters} built={built.n_pairs} pruned={pruned.n_pairs} "
          f"admitted={stats.n_admitted} within={stats.n_within_cutoff} ({time.time() - t0:.1f} s)", flush=True)


def main_large():
    """24k (config 2 geometry) with both grid rules, 96k (config 3) tuned and
    default (the needle-cluster multi-image case) and 96k m = 8."""
    dump_large("spc24k_default", 24000, m=4, tuned=False, f64=True)
    dump_large("spc24k_tuned", 24000, m=4, tuned=True, f64=True)
    dump_large("spc96k_tuned", 96000, m=4, tuned=True)
    dump_large("spc96k_tuned_m8", 96000, m=8, tuned=True)
    dump_large("spc96k_default", 96000, m=4, tuned=False)


def dump_diagnostics():
    """Reference outputs of the diagnostics row: the
    write_pairs_csv file (SHA-256 of its bytes), flop_count for several
    kernel layouts, and scatter_to_original of a seeded per-slot array."""
    import hashlib
    import tempfile

    out = {}
    cases = [("spc3k_tuned", 4), ("spc3k_default", 4), ("uniform_m8", 8), ("uniform_m2", 2), ("uniform_super8", 4)]
    for name, m in cases:
        with np.load(HERE / f"{name}.npz") as z:
            g = {k: z[k] for k in z.files}
        n = g["positions"].shape[0]
        system = cm.ParticleSystem(positions=g["positions"], velocities=np.zeros((n, 3)), masses=g["masses"],
                                   charges=g["charges"], lj_type=g["lj_type"], box=cm.SimBox(g["box"]))
        occ = None if np.isnan(g["occupancy"]) else float(g["occupancy"])
        grid = cm.build_cluster_grid(system, m, target_occupancy=occ)
        built = cm.build_pair_list(grid, system.box, float(g["r_list"]), supercluster_size=int(g["supercluster"]))
        pruned = cm.prune_pair_list(built, grid.clustered_positions, system.box)
        for tag, pl in (("built", built), ("pruned", pruned)):
            with tempfile.TemporaryDirectory() as d:
                path = Path(d) / "pairs.csv"
                cm.write_pairs_csv(pl, grid, system.box, path)
                out[f"{name}_{tag}_csv_sha256"] = hashlib.sha256(path.read_bytes()).hexdigest()
        layouts = [(m, nl) for nl in (1, 2, 4, 8)]
        fl = np.array([[nl, cm.flop_count(pruned, grid, cm.KernelLayout(m=m, n_lane=nl), system.box,
                                          float(g["r_cut"])).total_flops,
                        cm.flop_count(pruned, grid, cm.KernelLayout(m=m, n_lane=nl), system.box,
                                      float(g["r_cut"])).useful_flops] for _, nl in layouts], dtype=np.int64)
        out[f"{name}_flops"] = fl
        rng = np.random.default_rng(99)
        vals = rng.normal(size=(grid.n_slots, 3))
        out[f"{name}_scatter_in"] = vals
        out[f"{name}_scatter_out"] = cm.scatter_to_original(grid, vals)
        print(name, "csv", out[f"{name}_pruned_csv_sha256"][:12], "flops", fl.tolist())
    np.savez_compressed(HERE / "diagnostics.npz", **out)


if __name__ == "__main__":
    if "--large" in sys.argv:
        main_large()
    elif "--diagnostics" in sys.argv:
        dump_diagnostics()
    else:
        main()
