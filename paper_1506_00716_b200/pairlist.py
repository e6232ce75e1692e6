"""Cluster-pair list: build, prune, diagnostics -- drop-in for clustermd.pairlist.

Mirrors /root/reference/pkg/src/clustermd/pairlist.py.  Lists are built and
pruned on the GPU (csrc/search.cu); ``ClusterPairList`` keeps the device
handle and materialises the reference's numpy fields (offsets, j_idx, masks,
super layout) on first access, set-identical to the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .gridder import ClusterGrid, DeviceArray, bbox_gap_sq
from .model import ParameterError, SimBox

VALID_SUPERCLUSTER_SIZES = (1, 8)


def _ro(a):
    a.setflags(write=False)
    return a


class ClusterPairList:
    """CSR cluster-pair list + optional super-cluster layout (pairlist.py:27-94).

    Device-resident; numpy views: offsets, j_idx, masks (n_pairs, m, m) bool,
    super_offsets / super_j_idx / super_pair_idx (supercluster_size 8)."""

    def __init__(self, handle, grid: ClusterGrid, r_list: float, n_lane: int, build_step: int,
                 supercluster_size: int, build_positions=None):
        self._h = handle
        self.grid = grid
        info = np.zeros(5, dtype=np.int64)
        _lib.check(_lib.load().nbx_list_info(handle, _lib.ptr(info)), "list_info")
        self._n_i, self._n_rows, self.m, self.n_groups, self._n_entries = (int(v) for v in info)
        self.r_list = float(r_list)
        self.n_lane = n_lane
        self.build_step = build_step
        self.supercluster_size = supercluster_size
        self._build_positions = build_positions
        self._host = None
        self._super = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.nbx_list_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n_i_clusters(self) -> int:
        return self._n_i

    @property
    def n_entries(self) -> int:
        """Live (group, j-cluster) entries of the grouped force layout."""
        if self._n_entries < 0:  # a pruned list's count stays on the device until asked for
            n = ctypes.c_int64()
            _lib.check(_lib.load().nbx_list_entries(self._h, dev.stream(), ctypes.byref(n)), "list_entries")
            self._n_entries = int(n.value)
        return self._n_entries

    def force_pairs(self, inner: bool = True) -> int:
        """Admitted slot pairs the grouped force kernel evaluates: the inner
        list's when the list was pruned with ``r_inner`` (and ``inner``),
        else the canonical admitted count (extension; syncs)."""
        n = ctypes.c_int64()
        _lib.check(_lib.load().nbx_list_force_pairs(self._h, int(bool(inner)), dev.stream(), ctypes.byref(n)),
                   "list_force_pairs")
        return int(n.value)

    @property
    def n_pairs(self) -> int:
        if self._n_rows < 0:  # canonical rows are derived from the entries on first use
            n = ctypes.c_int64()
            _lib.check(_lib.load().nbx_list_rows(self._h, dev.stream(), ctypes.byref(n)), "list_rows")
            self._n_rows = int(n.value)
        return self._n_rows

    @property
    def build_positions(self) -> np.ndarray:
        if self._build_positions is None:
            return self.grid.clustered_positions
        return self._build_positions

    def _materialise(self):
        if self._host is None:
            off = np.empty(self._n_i + 1, dtype=np.int64)
            jj = np.empty(self.n_pairs, dtype=np.int64)
            mk = np.empty(self.n_pairs, dtype=np.uint64)
            torch.cuda.synchronize()
            _lib.check(_lib.load().nbx_list_download(self._h, _lib.ptr(off), _lib.ptr(jj), _lib.ptr(mk),
                                                     dev.stream()), "list_download")
            m = self.m
            bits = ((mk[:, None] >> np.arange(m * m, dtype=np.uint64)) & np.uint64(1)).astype(bool)
            self._host = dict(offsets=_ro(off), j_idx=_ro(jj), masks=_ro(bits.reshape(-1, m, m)),
                              mask_bits=_ro(mk))
        return self._host

    offsets = property(lambda self: self._materialise()["offsets"])
    j_idx = property(lambda self: self._materialise()["j_idx"])
    masks = property(lambda self: self._materialise()["masks"])
    mask_bits = property(lambda self: self._materialise()["mask_bits"])

    def _super_layout(self):
        if self.supercluster_size == 1:
            return None
        if self._super is None:
            ne = ctypes.c_int64()
            _lib.check(_lib.load().nbx_super_layout(self._h, self.supercluster_size, dev.stream(),
                                                    ctypes.byref(ne)), "super_layout")
            ngr = -(-self._n_i // self.supercluster_size)
            so = np.empty(ngr + 1, dtype=np.int64)
            sj = np.empty(ne.value, dtype=np.int64)
            sp = np.empty((ne.value, self.supercluster_size), dtype=np.int64)
            _lib.check(_lib.load().nbx_super_download(self._h, _lib.ptr(so), _lib.ptr(sj), _lib.ptr(sp),
                                                      dev.stream()), "super_download")
            self._super = (_ro(so), _ro(sj), _ro(sp))
        return self._super

    super_offsets = property(lambda self: None if self._super_layout() is None else self._super_layout()[0])
    super_j_idx = property(lambda self: None if self._super_layout() is None else self._super_layout()[1])
    super_pair_idx = property(lambda self: None if self._super_layout() is None else self._super_layout()[2])

    @property
    def n_super_groups(self) -> int:
        return 0 if self.supercluster_size == 1 else -(-self._n_i // self.supercluster_size)

    def entries(self, ci: int) -> np.ndarray:
        return self.j_idx[self.offsets[ci]:self.offsets[ci + 1]]

    def pair_i_clusters(self) -> np.ndarray:
        return np.repeat(np.arange(self._n_i, dtype=np.int64), np.diff(self.offsets))

    def super_flags(self):
        sp = self.super_pair_idx
        return None if sp is None else sp >= 0


@dataclass(frozen=True)
class InteractionStats:
    """pairlist.py:97-103."""

    n_admitted: int
    n_within_cutoff: int
    ratio: float


def build_pair_list(grid: ClusterGrid, box: SimBox, r_list: float, *, supercluster_size: int = 1,
                    n_lane: int = 1, build_step: int = 0, halo=None, molecules=None) -> ClusterPairList:
    """All cluster pairs with AABB gap <= r_list, j >= i (pairlist.py:147-217).

    ``halo`` (extension, domain decomposition): CUDA uint8 tensor per
    particle marking particles owned by another rank; halo-halo slot pairs
    are masked out.  ``molecules`` (extension, rigid water): per-particle
    molecule ids; slot pairs within one molecule are masked out
    (exclude_molecules)."""
    if r_list <= 0.0:
        raise ParameterError(f"r_list must be positive, got {r_list}")
    if np.any(box.lengths < 2.0 * r_list):
        raise ParameterError(f"every box edge must be >= 2*r_list={2.0 * r_list} "
                             f"for the single-image convention, got {box.lengths}")
    if supercluster_size not in VALID_SUPERCLUSTER_SIZES:
        raise ParameterError(f"supercluster_size must be one of {VALID_SUPERCLUSTER_SIZES}, "
                             f"got {supercluster_size}")
    h = ctypes.c_void_p()
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_pairlist_build_ex(grid.handle, _lib.ptr(L), float(r_list), _lib.ptr(halo),
                                                 dev.stream(), ctypes.byref(h)), "pairlist_build")
    plist = ClusterPairList(h, grid, r_list, n_lane, build_step, supercluster_size)
    if molecules is not None:
        exclude_molecules(plist, molecules)
    return plist


class Molecules:
    """Molecule topology on the device for exclude_molecules: per-atom ids
    and the atoms of each molecule (CSR), built once and reused by every
    list rebuild.  ``ids``: one int per particle in [0, n)."""

    def __init__(self, ids):
        t = dev.to_device(ids, torch.int64)
        n = int(t.shape[0])
        if t.dim() != 1:
            raise ParameterError("molecule ids must be one int per particle")
        if n and not (0 <= int(t.min()) and int(t.max()) < n):
            raise ParameterError(f"molecule ids must lie in [0, n={n})")
        order = torch.argsort(t, stable=True)
        counts = torch.bincount(t, minlength=n)
        first = torch.zeros(n + 1, dtype=torch.int64, device=t.device)
        first[1:] = torch.cumsum(counts, 0)
        self.n = n
        self.atom_mol = t.to(torch.int32).contiguous()
        self.mol_first = first.to(torch.int32).contiguous()
        self.mol_atoms = order.to(torch.int32).contiguous()


def exclude_molecules(plist: ClusterPairList, molecules, count: bool = False):
    """Extension (SPC / rigid water; the reference masks only fillers and the
    diagonal, pairlist.py:106-112): remove, in place, every admitted slot pair
    whose two particles share a molecule (``molecules``: a Molecules topology,
    or one int id per particle, original order).  Applied before the prune,
    excluded pairs also no longer keep a row alive.  Returns the number of
    removed slot pairs when ``count`` (one host sync), else None."""
    g = plist.grid
    mol = molecules if isinstance(molecules, Molecules) else Molecules(molecules)
    if mol.n != g.n:
        raise ParameterError(f"molecules describe {mol.n} particles, the grid has {g.n}")
    out = ctypes.c_int64(0)
    _lib.check(_lib.load().nbx_list_exclude(plist.handle, g.handle, _lib.ptr(mol.atom_mol), _lib.ptr(mol.mol_first),
                                            _lib.ptr(mol.mol_atoms), dev.stream(),
                                            ctypes.byref(out) if count else None), "list_exclude")
    plist._host = None
    plist._super = None
    return int(out.value) if count else None


def list_step(system, m: int, target_occupancy, box: SimBox, r_list: float, *, positions=None,
              r_inner: float = 0.0, prune: bool = True, halo=None, molecules=None, supercluster_size: int = 1,
              n_lane: int = 1, build_step: int = 0) -> tuple[ClusterGrid, ClusterPairList]:
    """The rebuild of a device-resident driver (engine.py:294-334 _rebuild)
    in one native call (nbx_list_step): ``build_cluster_grid`` ->
    ``build_pair_list`` (``halo``, ``molecules``) -> ``prune_pair_list`` at
    the grid's build positions (``prune``, ``r_inner``) -> the force layout
    the first force call would build.  Same grid and list as the separate
    calls; the GPU does not wait on the interpreter between the phases.
    ``positions``: CUDA tensor (n, 3), default system.positions."""
    from .gridder import grid_cells

    if m not in (1, 2, 4, 8):
        raise ParameterError(f"cluster size m must be one of (1, 2, 4, 8), got {m}")
    if target_occupancy is None:
        target_occupancy = 2.0 * m
    if target_occupancy <= 0:
        raise ParameterError(f"target occupancy must be positive, got {target_occupancy}")
    if r_list <= 0.0:
        raise ParameterError(f"r_list must be positive, got {r_list}")
    if np.any(box.lengths < 2.0 * r_list):
        raise ParameterError(f"every box edge must be >= 2*r_list={2.0 * r_list} "
                             f"for the single-image convention, got {box.lengths}")
    if r_inner and not (0.0 < r_inner <= r_list):
        raise ParameterError(f"r_inner must be 0 (off) or in (0, r_list={r_list}], got {r_inner}")
    if supercluster_size not in VALID_SUPERCLUSTER_SIZES:
        raise ParameterError(f"supercluster_size must be one of {VALID_SUPERCLUSTER_SIZES}, "
                             f"got {supercluster_size}")
    n = system.n
    src = system.positions if positions is None else positions
    pos = dev.to_device(src, torch.float64, (n, 3))
    mol = None
    if molecules is not None:
        mol = molecules if isinstance(molecules, Molecules) else Molecules(molecules)
        if mol.n != n:
            raise ParameterError(f"molecules describe {mol.n} particles, the grid has {n}")
    L = _lib.box3(box.lengths)
    hg, hl = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(_lib.load().nbx_list_step(
        _lib.ptr(pos), n, _lib.ptr(L), m, grid_cells(n, m, target_occupancy), float(r_list), float(r_inner or 0.0),
        _lib.ptr(halo), _lib.ptr(mol.atom_mol) if mol else None, _lib.ptr(mol.mol_first) if mol else None,
        _lib.ptr(mol.mol_atoms) if mol else None, 1 if prune else 0, dev.stream(), ctypes.byref(hg),
        ctypes.byref(hl)), "list_step")
    grid = ClusterGrid(hg, box.lengths)
    return grid, ClusterPairList(hl, grid, r_list, n_lane, build_step, supercluster_size)


def build_pruned_pair_list(grid: ClusterGrid, box: SimBox, r_list: float, positions=None, *,
                           supercluster_size: int = 1, n_lane: int = 1, build_step: int = 0,
                           halo=None, molecules=None) -> ClusterPairList:
    """``prune_pair_list(build_pair_list(grid, box, r_list, ...), positions, box)``
    in one GPU search (extension): each bounding-box hit is checked against
    the exact prune criterion before it is stored, so the unpruned list is
    never materialised.  Bit-identical to the two-step result.  ``positions``
    (clustered, n_slots x 3) defaults to the grid's build positions."""
    if r_list <= 0.0:
        raise ParameterError(f"r_list must be positive, got {r_list}")
    if np.any(box.lengths < 2.0 * r_list):
        raise ParameterError(f"every box edge must be >= 2*r_list={2.0 * r_list} "
                             f"for the single-image convention, got {box.lengths}")
    if supercluster_size not in VALID_SUPERCLUSTER_SIZES:
        raise ParameterError(f"supercluster_size must be one of {VALID_SUPERCLUSTER_SIZES}, "
                             f"got {supercluster_size}")
    keep_alive = None
    if positions is None:
        p = ctypes.c_void_p(0)
    else:
        shape = tuple(positions.shape)
        if shape != (grid.n_slots, 3):
            raise ParameterError(f"positions shape {shape} does not match the slot layout {(grid.n_slots, 3)}")
        tmp = ClusterPairList.__new__(ClusterPairList)
        tmp.grid = grid
        p, keep_alive = _positions_ptr(tmp, positions)
    h = ctypes.c_void_p()
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_pairlist_build_pruned(grid.handle, _lib.ptr(L), float(r_list), p, _lib.ptr(halo),
                                                     dev.stream(), ctypes.byref(h)), "pairlist_build_pruned")
    del keep_alive
    plist = ClusterPairList(h, grid, r_list, n_lane, build_step, supercluster_size)
    if molecules is not None:  # after the fused prune: a row kept only by an excluded pair stays (no pairs)
        exclude_molecules(plist, molecules)
    return plist


def _positions_ptr(plist: ClusterPairList, positions):
    """Device pointer for clustered positions: the grid's own build snapshot
    when that is what the caller passed, else an uploaded copy."""
    g = plist.grid
    if isinstance(positions, DeviceArray):
        return positions.ptr, positions
    if g._host is not None and positions is g._host.get("clustered_positions"):
        return g.clustered_positions_device_ptr(), None
    if dev.is_device_tensor(positions):
        t = positions.to(torch.float64).contiguous()
        return _lib.ptr(t), t
    arr = np.asarray(positions, dtype=np.float64)
    t = dev.to_device(arr, torch.float64)
    return _lib.ptr(t), t


def prune_pair_list(plist: ClusterPairList, positions, box: SimBox, *, r_inner: float = 0.0) -> ClusterPairList:
    """Drop rows whose exact min admitted-slot distance exceeds r_list
    (pairlist.py:242-282); positions are clustered (n_slots, 3).

    ``r_inner`` (extension, dynamic pruning; 0 = off): the force pass also
    gets an inner list of the rows with a pair within r_inner at these
    positions (which must be the grid's build positions).  It is used while
    2 d_max <= r_inner - r_c (checked on the device every force call; the
    full list otherwise).  The list itself -- offsets, j_idx, masks -- is the
    same as without it."""
    shape = tuple(positions.shape)
    if shape != (plist.grid.n_slots, 3):
        raise ParameterError(f"positions shape {shape} does not match the list's slot layout "
                             f"{(plist.grid.n_slots, 3)}")
    if r_inner and not (0.0 < r_inner <= plist.r_list):
        raise ParameterError(f"r_inner must be 0 (off) or in (0, r_list={plist.r_list}], got {r_inner}")
    if plist._n_entries == 0:  # (-1: pruned list, count on the device -- never empty)
        return plist
    p, keep_alive = _positions_ptr(plist, positions)
    h = ctypes.c_void_p()
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_pairlist_prune_inner(plist.handle, plist.grid.handle, p, _lib.ptr(L),
                                                    float(r_inner), dev.stream(), ctypes.byref(h)),
               "pairlist_prune")
    del keep_alive
    return ClusterPairList(h, plist.grid, plist.r_list, plist.n_lane, plist.build_step,
                           plist.supercluster_size, plist._build_positions)


def admitted_pairs(plist: ClusterPairList, grid: ClusterGrid) -> set:
    """Admitted original-index pairs (lo, hi) (pairlist.py:285-300)."""
    if plist.n_pairs == 0:
        return set()
    m = plist.m
    p, a, b = np.nonzero(plist.masks)
    ci = plist.pair_i_clusters()
    oi = grid.perm[ci[p] * m + a]
    oj = grid.perm[plist.j_idx[p] * m + b]
    return set(zip(np.minimum(oi, oj).tolist(), np.maximum(oi, oj).tolist()))


def interaction_stats(plist: ClusterPairList, grid: ClusterGrid, positions, box: SimBox,
                      r_cut: float) -> InteractionStats:
    """Admitted vs within-r_cut slot pairs (pairlist.py:323-346), counted on the GPU."""
    if r_cut > plist.r_list:
        raise ParameterError(f"r_cut={r_cut} must not exceed the list radius r_list={plist.r_list}")
    if plist.n_pairs == 0:
        return InteractionStats(0, 0, 1.0)
    p, keep_alive = _positions_ptr(plist, positions)
    out = np.zeros(2, dtype=np.int64)
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_count_within(plist.handle, p, _lib.ptr(L), float(r_cut), dev.stream(),
                                            _lib.ptr(out)), "count_within")
    del keep_alive
    n_adm, n_win = int(out[0]), int(out[1])
    ratio = float(n_adm) / float(n_win) if n_win else float("inf")
    if n_adm == 0:
        ratio = 1.0 if n_win == 0 else 0.0
    return InteractionStats(n_admitted=n_adm, n_within_cutoff=n_win, ratio=ratio)


def pair_diagnostics(plist: ClusterPairList, grid: ClusterGrid, box: SimBox):
    """Per-row (bbox gap^2, exact minimum admitted slot distance^2) at the
    list's build positions, computed on the GPU (nbx_list_diagnostics) with
    the reference's FP64 operation order: bit-identical to gridder.bbox_gap_sq
    and pairlist._pair_min_dist_sq (pairlist.py:220-239, :349-360).
    Returns two float64 numpy arrays of length n_pairs."""
    n = plist.n_pairs
    if n == 0:
        return np.empty(0), np.empty(0)
    if plist._build_positions is None:
        p, keep_alive = ctypes.c_void_p(0), None
    else:
        p, keep_alive = _positions_ptr(plist, plist._build_positions)
    out = torch.empty((2, n), dtype=torch.float64, device=dev.require_cuda())
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_list_diagnostics(plist.handle, grid.handle, p, _lib.ptr(L), _lib.ptr(out[0]),
                                                _lib.ptr(out[1]), dev.stream()), "list_diagnostics")
    del keep_alive
    host = out.cpu().numpy()
    return host[0], host[1]


def write_pairs_csv(plist: ClusterPairList, grid: ClusterGrid, box: SimBox, path) -> None:
    """Per-row diagnostics CSV (pairlist.py:349-376): bbox vs exact distance.

    The distances come from the GPU (pair_diagnostics, bit-identical values);
    the host only formats them, with the reference's csv dialect and
    ``repr`` of each float, so the file is byte-identical."""
    gap_sq, min_d2 = pair_diagnostics(plist, grid, box)
    ci = plist.pair_i_clusters().tolist() if plist.n_pairs else []
    cj = plist.j_idx.tolist() if plist.n_pairs else []
    gap = np.sqrt(gap_sq).tolist()
    finite = np.isfinite(min_d2)
    exact = np.where(finite, np.sqrt(np.where(finite, min_d2, 0.0)), np.nan).tolist()
    with open(path, "w", newline="") as fh:
        fh.write("i_cluster,j_cluster,bbox_distance_nm,exact_min_distance_nm\r\n")
        fh.writelines(f"{a},{b},{g!r},{e!r}\r\n" for a, b, g, e in zip(ci, cj, gap, exact))
