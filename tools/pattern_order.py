"""Search the force order of member patterns (csrc/search.cu pattern_rank).

    python tools/pattern_order.py [atoms] [steps]

Builds the inner list (r_inner = r_c + 0.02) of the SPC box with the oracle,
forms the force kernel's groups (G = 4 consecutive clusters of a column) and
entries (group, j-cluster) with their member patterns, and counts the member
sweeps k_force_h runs when each group's entries are laid out in a given
pattern order and processed R = 8 at a time (a member's sweep runs when any
of the R entries holds it).  A random-swap local search over the order
minimises the evaluated slot pairs; prints admitted / evaluated for ascending
pattern values, and the best order found."""
import random
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import native, search  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
m, G, R = 4, 4, 8
s, _ = spc_water(n, seed=2024)
L = np.asarray(s.box.lengths)
g = search.build_grid(np.asarray(s.positions), L, m, tuned_occupancy(n, float(L[0]), m))
pl = native.prune_list(native.search_list(g, L, 1.1), g["clustered_positions"], L)
ci_all = search.row_ci(pl)
inner = (search.row_min_dist_sq(pl, g["clustered_positions"], L) <= 1.02 ** 2) | (ci_all == pl["j_idx"])
ci, cj = ci_all[inner], pl["j_idx"][inner]
adm = int(pl["masks"].reshape(len(ci_all), -1)[inner].sum())
nc, coc = g["n_clusters"], g["cell_of_cluster"]
col_first = np.searchsorted(coc, np.arange(g["cells"] ** 2 + 1))
k_in = (np.arange(nc) - col_first[coc]) % G
gid = np.unique(np.arange(nc) - k_in, return_inverse=True)[1]
ukey, inv = np.unique(gid[ci].astype(np.int64) * (nc + 1) + cj, return_inverse=True)
pat = np.zeros(len(ukey), dtype=np.int64)
np.bitwise_or.at(pat, inv, 1 << k_in[ci])
eg = ukey // (nc + 1)
popc = np.array([bin(x).count("1") for x in range(16)])
cnt = np.zeros((eg.max() + 1, 16), dtype=np.int64)
np.add.at(cnt, (eg, pat), 1)


def evaluated(order):
    c = cnt[:, order]
    cum = np.cumsum(c, axis=1)
    start = cum - c
    nit = (cum[:, -1] + R - 1) // R
    tot = 0
    for it in range(int(nit.max())):
        ov = (np.minimum(cum, it * R + R) - np.maximum(start, it * R)) > 0
        u = np.zeros(len(c), dtype=np.int64)
        for k, p in enumerate(order):
            u |= np.where(ov[:, k], p, 0)
        tot += int(popc[u][it < nit].sum())
    return tot * R * m * m


print(f"atoms {n}: entries {len(ukey)}, admitted {adm}; ascending patterns: {adm / evaluated(list(range(16))):.3f}")
best = list(range(16))
bc = evaluated(best)
random.seed(1)
for _ in range(steps):
    i, j = random.sample(range(15), 2)
    cand = best[:]
    cand[i], cand[j] = cand[j], cand[i]
    c = evaluated(cand)
    if c < bc:
        best, bc = cand, c
rank = [0] * 16
for i, p in enumerate(best):
    rank[p] = i
print(f"best order {best}: {adm / bc:.3f}; pattern_rank table {rank}")
