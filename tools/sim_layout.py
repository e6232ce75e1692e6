"""CPU model of the force kernel's slot-pair work for a grouped layout.

    python tools/sim_layout.py [atoms]

Builds the pruned list with the oracle (C port), forms groups of G
consecutive clusters of a column, entries (group, cj) with member patterns,
and counts the slot pairs a warp evaluates (R = 32/m entries per iteration,
member k skipped when absent from all R entries) against admitted pairs.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import native, search  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96000
m = 4
s, _ = spc_water(n, seed=2024)
L = np.asarray(s.box.lengths)
occ = tuned_occupancy(n, float(L[0]), m)
g = search.build_grid(np.asarray(s.positions), L, m, occ)
lst = native.search_list(g, L, 1.1)
pl = native.prune_list(lst, g["clustered_positions"], L)
nc = g["n_clusters"]
ci = search.row_ci(pl)
cj = pl["j_idx"]
adm = pl["masks"].reshape(len(cj), -1).sum(1)
print(f"atoms {n} clusters {nc} rows {len(cj)} admitted {adm.sum()}")
coc = g["cell_of_cluster"]
col_first = np.searchsorted(coc, np.arange(g["cells"] ** 2 + 1))


def simulate(G, R, order="pattern"):
    k_in = (np.arange(nc) - col_first[coc]) % G
    grp_first = np.arange(nc) - k_in
    gid = np.unique(grp_first, return_inverse=True)[1]
    key = gid[ci].astype(np.int64) * (nc + 1) + cj
    ukey, inv = np.unique(key, return_inverse=True)
    pat = np.zeros(len(ukey), dtype=np.int64)
    np.bitwise_or.at(pat, inv, 1 << k_in[ci])
    eg = ukey // (nc + 1)
    if order == "pattern":
        o = np.lexsort((ukey % (nc + 1), pat, eg))
    else:
        o = np.arange(len(ukey))
    eg, pat = eg[o], pat[o]
    bounds = np.searchsorted(eg, np.arange(eg.max() + 2))
    comp = 0
    per_member = 16 * m * m // (m * m) * m // m  # placeholder
    for gi in range(len(bounds) - 1):
        p = pat[bounds[gi]:bounds[gi + 1]]
        pad = (-len(p)) % R
        p = np.concatenate([p, np.zeros(pad, dtype=np.int64)]).reshape(-1, R)
        orp = np.bitwise_or.reduce(p, axis=1)
        comp += int(sum(bin(int(x)).count("1") for x in orp)) * R * m * m
    print(f"G={G} R={R} order={order}: entries {len(ukey)} computed slot pairs {comp} "
          f"eff {adm.sum() / comp:.3f}  mean members/entry {np.mean([bin(int(x)).count('1') for x in pat]):.2f}")


for G, R in ((4, 8), (4, 1), (2, 8), (8, 8), (4, 4)):
    simulate(G, R)
simulate(4, 8, order="j")
