"""Grid + cluster-pair search restated in numpy (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/clustermd/gridder.py and pairlist.py.  All
decisions (column binning, z order, bounding-box gap, prune distance) are the
same FP64 operations in the same order as the reference, so results are
bit-identical; tests/test_oracle.py pins this against golden vectors made by
the reference itself (tests/golden/make_golden.py).

Outputs are plain dicts of numpy arrays so that nothing here depends on the
product package.
"""

from __future__ import annotations

import math

import numpy as np

from .geometry import min_image, wrap

_CHUNK = 4096  # pairlist.py:24 -- rows per vectorized distance batch


def grid_cells(n: int, m: int, target_occupancy=None) -> int:
    """gridder.py:82-91: cells per side = max(1, round(sqrt(n / occ)))."""
    occ = 2.0 * m if target_occupancy is None else float(target_occupancy)
    return max(1, int(round(math.sqrt(n / occ))))


def build_grid(positions, lengths, m: int, target_occupancy=None) -> dict:
    """gridder.py:69-146 restated without the per-column Python loop.

    Column binning (:92-94) -> stable (cell, z, index) order (:97) -> pad
    each column to a multiple of m with copies of its last particle
    (:104-117) -> inverse permutation (:127-130) -> AABBs (:132-134).
    """
    lengths = np.asarray(lengths, dtype=np.float64)
    n = int(np.asarray(positions).reshape(-1, 3).shape[0])
    pos = wrap(np.asarray(positions, dtype=np.float64).reshape(-1, 3), lengths)
    cells = grid_cells(n, m, target_occupancy)
    ix = np.minimum((pos[:, 0] / lengths[0] * cells).astype(np.int64), cells - 1)
    iy = np.minimum((pos[:, 1] / lengths[1] * cells).astype(np.int64), cells - 1)
    cell = ix * cells + iy
    order = np.lexsort((np.arange(n), pos[:, 2], cell))

    counts = np.bincount(cell, minlength=cells * cells).astype(np.int64)
    padded = -(-counts // m) * m
    first_sorted = np.cumsum(counts) - counts
    first_slot = np.cumsum(padded) - padded
    n_slots = int(padded.sum())
    slot_col = np.repeat(np.arange(cells * cells, dtype=np.int64), padded)
    k = np.arange(n_slots, dtype=np.int64) - first_slot[slot_col]
    src = first_sorted[slot_col] + np.minimum(k, counts[slot_col] - 1)
    perm = order[src] if n_slots else np.empty(0, dtype=np.int64)
    fill = k >= counts[slot_col]
    n_clusters = n_slots // m

    inverse = np.empty(n, dtype=np.int64)
    inverse[perm[~fill]] = np.nonzero(~fill)[0]
    cpos = pos[perm] if n_slots else np.empty((0, 3))
    grouped = cpos.reshape(n_clusters, m, 3)
    if n_clusters:
        bboxes = np.stack([grouped.min(axis=1), grouped.max(axis=1)], axis=1)
    else:
        bboxes = np.empty((0, 2, 3))
    return dict(
        m=m,
        n=n,
        n_clusters=n_clusters,
        cells=cells,
        perm=perm,
        inverse_perm=inverse,
        fill_mask=fill,
        cell_of_cluster=slot_col[::m].copy(),
        clustered_positions=cpos,
        bboxes=bboxes,
    )


def scatter_to_original(grid: dict, values) -> np.ndarray:
    """gridder.py:149-162: drop filler slots, out[perm[real]] = v[real]."""
    values = np.asarray(values)
    out = np.zeros((grid["n"],) + values.shape[1:], dtype=values.dtype)
    real = ~grid["fill_mask"]
    out[grid["perm"][real]] = values[real]
    return out


def bbox_gap_sq(lo_i, hi_i, lo_j, hi_j, lengths) -> np.ndarray:
    """gridder.py:165-185: periodic AABB gap, images {-L, 0, +L} per dim,
    summed ((0 + gx^2) + gy^2) + gz^2."""
    lo_j = np.asarray(lo_j, dtype=np.float64)
    hi_j = np.asarray(hi_j, dtype=np.float64)
    total = np.zeros(lo_j.shape[:-1], dtype=np.float64)
    for d in range(3):
        span = lengths[d]
        a = lo_j[..., d] - hi_i[d]
        b = lo_i[d] - hi_j[..., d]
        g_here = np.maximum(0.0, np.maximum(a, b))
        g_minus = np.maximum(0.0, np.maximum(a - span, b + span))
        g_plus = np.maximum(0.0, np.maximum(a + span, b - span))
        g = np.minimum(g_here, np.minimum(g_minus, g_plus))
        total = total + g * g
    return total


def masks_for_rows(ci, cj, fill_mask, m) -> np.ndarray:
    """pairlist.py:106-112: real_i x real_j, strict upper triangle on the
    diagonal row.  Returns (rows, m, m) bool."""
    real = ~np.asarray(fill_mask).reshape(-1, m)
    masks = real[ci][:, :, None] & real[cj][:, None, :]
    diag = ci == cj
    if np.any(diag):
        masks[diag] &= np.triu(np.ones((m, m), dtype=bool), k=1)
    return masks


def pack_masks(masks) -> np.ndarray:
    """(rows, m, m) bool -> uint64 with bit a*m + b (the GPU list format)."""
    rows, m, _ = masks.shape
    flat = masks.reshape(rows, m * m).astype(np.uint64)
    weights = (np.uint64(1) << np.arange(m * m, dtype=np.uint64))
    return (flat * weights).sum(axis=1, dtype=np.uint64)


def unpack_masks(bits, m) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.uint64)
    shifts = np.arange(m * m, dtype=np.uint64)
    return ((bits[:, None] >> shifts) & np.uint64(1)).astype(bool).reshape(-1, m, m)


def build_pairs_bruteforce(grid: dict, lengths, r_list: float) -> dict:
    """pairlist.py:177-201: for every ci, all cj >= ci with AABB gap^2 <=
    r_list^2 (O(n_c^2), the reference's own search), CSR + masks."""
    lengths = np.asarray(lengths, dtype=np.float64)
    nc = grid["n_clusters"]
    lows = grid["bboxes"][:, 0] if nc else np.empty((0, 3))
    highs = grid["bboxes"][:, 1] if nc else np.empty((0, 3))
    r2 = r_list * r_list
    counts = np.zeros(nc, dtype=np.int64)
    parts = []
    for ci in range(nc):
        gap = bbox_gap_sq(lows[ci], highs[ci], lows[ci:], highs[ci:], lengths)
        js = np.nonzero(gap <= r2)[0].astype(np.int64) + ci
        counts[ci] = js.shape[0]
        parts.append(js)
    return _finish_list(grid, counts, parts, r_list)


def _finish_list(grid, counts, parts, r_list) -> dict:
    nc = grid["n_clusters"]
    m = grid["m"]
    offsets = np.zeros(nc + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    j_idx = np.concatenate(parts) if parts else np.empty(0, dtype=np.int64)
    ci = np.repeat(np.arange(nc, dtype=np.int64), counts)
    masks = masks_for_rows(ci, j_idx, grid["fill_mask"], m) if j_idx.size else np.empty((0, m, m), bool)
    return dict(m=m, offsets=offsets, j_idx=j_idx, masks=masks, r_list=float(r_list))


def list_from_csr(grid, offsets, j_idx, r_list) -> dict:
    """Assemble a list dict from a CSR produced elsewhere (e.g. the C port)."""
    counts = np.diff(offsets)
    return _finish_list(grid, counts, [np.asarray(j_idx, dtype=np.int64)], r_list)


def row_ci(lst: dict) -> np.ndarray:
    """pairlist.py:84-88: i-cluster of every row."""
    nc = lst["offsets"].shape[0] - 1
    return np.repeat(np.arange(nc, dtype=np.int64), np.diff(lst["offsets"]))


def row_min_dist_sq(lst: dict, clustered_positions, lengths) -> np.ndarray:
    """pairlist.py:220-239: exact min over admitted slot pairs of the min-image
    d^2, einsum("pabd,pabd->pab") (numpy's own summation order), +inf when
    no slot pair is admitted."""
    m = lst["m"]
    pos = np.asarray(clustered_positions, dtype=np.float64).reshape(-1, m, 3)
    ci = row_ci(lst)
    n_rows = lst["j_idx"].shape[0]
    out = np.empty(n_rows, dtype=np.float64)
    for s in range(0, n_rows, _CHUNK):
        e = min(s + _CHUNK, n_rows)
        dr = min_image(pos[ci[s:e]][:, :, None, :] - pos[lst["j_idx"][s:e]][:, None, :, :], lengths)
        d2 = np.einsum("pabd,pabd->pab", dr, dr)
        d2[~lst["masks"][s:e]] = np.inf
        out[s:e] = d2.min(axis=(1, 2))
    return out


def prune(lst: dict, clustered_positions, lengths) -> dict:
    """pairlist.py:242-282: keep rows with min d^2 <= r_list^2, and every
    diagonal row; masks of survivors unchanged."""
    if lst["j_idx"].shape[0] == 0:
        return lst
    ci = row_ci(lst)
    d2 = row_min_dist_sq(lst, clustered_positions, lengths)
    keep = (d2 <= lst["r_list"] * lst["r_list"]) | (ci == lst["j_idx"])
    nc = lst["offsets"].shape[0] - 1
    counts = np.bincount(ci[keep], minlength=nc).astype(np.int64)
    offsets = np.zeros(nc + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return dict(m=lst["m"], offsets=offsets, j_idx=lst["j_idx"][keep],
                masks=lst["masks"][keep], r_list=lst["r_list"])


def super_layout(offsets, j_idx, n_clusters, size=8):
    """pairlist.py:115-144: groups of `size` consecutive i-clusters, ascending
    union of their j-clusters, member row index or -1."""
    n_groups = -(-n_clusters // size)
    ci = np.repeat(np.arange(n_clusters, dtype=np.int64), np.diff(offsets))
    rows = np.arange(j_idx.shape[0], dtype=np.int64)
    g = ci // size
    k = ci - g * size
    # sort rows by (group, cj); rows of one group with equal cj form one entry
    order = np.lexsort((k, j_idx, g))
    gs, js, ks, rs = g[order], j_idx[order], k[order], rows[order]
    new = np.ones(gs.shape[0], dtype=bool)
    new[1:] = (gs[1:] != gs[:-1]) | (js[1:] != js[:-1])
    entry = np.cumsum(new) - 1
    n_entries = int(new.sum())
    super_j = js[new]
    pair_idx = np.full((n_entries, size), -1, dtype=np.int64)
    pair_idx[entry, ks] = rs
    per_group = np.bincount(gs[new], minlength=n_groups)
    super_offsets = np.zeros(n_groups + 1, dtype=np.int64)
    np.cumsum(per_group, out=super_offsets[1:])
    return super_offsets, super_j, pair_idx


def count_within(lst: dict, clustered_positions, lengths, r_cut) -> int:
    """pairlist.py:303-320: admitted slot pairs with min-image d^2 <= r_cut^2."""
    m = lst["m"]
    pos = np.asarray(clustered_positions, dtype=np.float64).reshape(-1, m, 3)
    ci = row_ci(lst)
    total = 0
    n_rows = lst["j_idx"].shape[0]
    rc2 = r_cut * r_cut
    for s in range(0, n_rows, _CHUNK):
        e = min(s + _CHUNK, n_rows)
        dr = min_image(pos[ci[s:e]][:, :, None, :] - pos[lst["j_idx"][s:e]][:, None, :, :], lengths)
        d2 = np.einsum("pabd,pabd->pab", dr, dr)
        total += int(np.count_nonzero((d2 <= rc2) & lst["masks"][s:e]))
    return total


def admitted_pair_set(lst: dict, grid: dict) -> set:
    """pairlist.py:285-300: admitted original-index pairs (lo, hi)."""
    if lst["j_idx"].shape[0] == 0:
        return set()
    m = lst["m"]
    ci = row_ci(lst)
    p, a, b = np.nonzero(lst["masks"])
    oi = grid["perm"][ci[p] * m + a]
    oj = grid["perm"][lst["j_idx"][p] * m + b]
    return set(zip(np.minimum(oi, oj).tolist(), np.maximum(oi, oj).tolist()))


def exclude_molecules(lst: dict, grid: dict, molecules) -> dict:
    """Extension (rigid water): the list with every admitted slot pair whose
    particles share a molecule id removed from the masks (rows unchanged).
    Restates csrc/search.cu k_exclude; fillers never match."""
    m = lst["m"]
    perm, fill = grid["perm"], grid["fill_mask"]
    mol = np.asarray(molecules, dtype=np.int64)[perm]
    mol = np.where(fill, -1 - np.arange(perm.shape[0]), mol)
    ci = row_ci(lst)
    mi = mol.reshape(-1, m)[ci]                 # (rows, m)
    mj = mol.reshape(-1, m)[lst["j_idx"]]
    same = mi[:, :, None] == mj[:, None, :]
    out = dict(lst)
    out["masks"] = lst["masks"] & ~same
    return out
