"""Non-bonded force kernels over cluster-pair lists -- drop-in for clustermd.kernels.

Mirrors /root/reference/pkg/src/clustermd/kernels.py: ``KernelLayout``,
``pair_interaction``/``lj_coulomb_terms`` (the functional form),
``compute_nonbonded_into`` / ``compute_nonbonded`` /
``compute_nonbonded_original`` and ``flop_count``.  The force pass runs in
csrc/force.cu (FP32 pair math, FP64 energy and final force accumulation,
bit-reproducible).  ``n_lane``/``j_unroll`` describe the reference's CPU
traversal only; they are validated and kept but do not change the GPU
schedule or the result.

``compute_nonbonded_device`` is the device-resident entry (CUDA tensors in,
CUDA tensors out, no host synchronisation) used by the engine and bench.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .gridder import ClusterGrid
from .model import ForcesEnergies, NonbondedParams, ParameterError, SimBox, SingularityError
from .pairlist import ClusterPairList, interaction_stats

VALID_LANE_COUNTS = (1, 2, 4, 8)

# kernels.py:34-42 -- the reference's flop cost model per evaluated slot pair
FLOPS_DISTANCE = 17
FLOPS_LJ = 12
FLOPS_COULOMB = 11
FLOPS_PER_PAIR = FLOPS_DISTANCE + FLOPS_LJ + FLOPS_COULOMB
# extension: erfc + exp of the Ewald real-space term
FLOPS_EWALD_EXTRA = 12


def flops_per_pair(params: NonbondedParams) -> int:
    return FLOPS_PER_PAIR + (FLOPS_EWALD_EXTRA if params.elec == "ewald" else 0)


@dataclass(frozen=True)
class KernelLayout:
    """Block shape m x n_lane of the reference traversal (kernels.py:45-69)."""

    m: int
    n_lane: int
    j_unroll: int = 0

    def __post_init__(self):
        if self.m not in (1, 2, 4, 8):
            raise ParameterError(f"m must be one of (1, 2, 4, 8), got {self.m}")
        if self.n_lane not in VALID_LANE_COUNTS:
            raise ParameterError(f"n_lane must be one of {VALID_LANE_COUNTS}, got {self.n_lane}")
        if self.j_unroll == 0:
            object.__setattr__(self, "j_unroll", max(1, self.n_lane // self.m))
        if self.j_unroll < 1:
            raise ParameterError(f"j_unroll must be >= 1, got {self.j_unroll}")


@dataclass(frozen=True)
class FlopCount:
    """kernels.py:72-81."""

    useful_flops: int
    total_flops: int

    @property
    def ratio(self) -> float:
        return self.useful_flops / self.total_flops if self.total_flops else 1.0


def lj_coulomb_terms(r2, type_i, type_j, q_i, q_j, params: NonbondedParams):
    """(e_lj, e_coulomb, f_over_r) for squared distance r2 (kernels.py:84-111),
    plus the reaction-field / Ewald extension selected by params.elec."""
    r2 = np.asarray(r2, dtype=np.float64)
    if np.any(r2 == 0.0):
        raise SingularityError("zero distance between interacting particles")
    eps = params.lj_table[type_i, type_j, 0]
    sig = params.lj_table[type_i, type_j, 1]
    sr2 = (sig * sig) / r2
    sr6 = sr2 * sr2 * sr2
    e_lj = 4.0 * eps * (sr6 * sr6 - sr6)
    f_over_r = 48.0 * eps * (sr6 * sr6 - 0.5 * sr6) / r2
    r = np.sqrt(r2)
    qq = params.coulomb_scale * np.asarray(q_i, dtype=np.float64) * q_j
    if params.elec == "cutoff":
        e_c = qq / r
        f_over_r = f_over_r + qq / (r2 * r)
        if params.shift_potential:
            e_c = e_c - qq / params.r_cut
    elif params.elec == "reaction_field":
        e_c = qq * (1.0 / r + params.k_rf * r2 - params.c_rf)
        f_over_r = f_over_r + qq * (1.0 / (r2 * r) - 2.0 * params.k_rf)
    else:
        beta = params.ewald_beta
        erfc_br = np.vectorize(math.erfc)(beta * r)
        e_c = qq * erfc_br / r
        f_over_r = f_over_r + qq * (erfc_br / r + 2.0 * beta / math.sqrt(math.pi)
                                    * np.exp(-beta * beta * r2)) / r2
        if params.shift_potential:
            e_c = e_c - qq * math.erfc(beta * params.r_cut) / params.r_cut
    if params.shift_potential:
        rc2 = params.r_cut * params.r_cut
        src2 = (sig * sig) / rc2
        src6 = src2 * src2 * src2
        e_lj = e_lj - 4.0 * eps * (src6 * src6 - src6)
    return e_lj, e_c, f_over_r


def pair_interaction(r2, type_i, type_j, q_i, q_j, params: NonbondedParams):
    """Total pair energy and f_over_r (kernels.py:114-121)."""
    e_lj, e_c, f_over_r = lj_coulomb_terms(r2, type_i, type_j, q_i, q_j, params)
    return e_lj + e_c, f_over_r


_last_params: list = []  # [(params, struct, table)]: run_md / the bench call with one params object


def _params_struct(params: NonbondedParams):
    if _last_params and _last_params[0][0] is params:
        return _last_params[0][1], _last_params[0][2]
    table = np.ascontiguousarray(params.lj_table, dtype=np.float64)
    p = _lib.NbxParams(
        n_types=params.n_types, lj_table=table.ctypes.data, coulomb_scale=params.coulomb_scale,
        r_cut=params.r_cut, shift_potential=int(bool(params.shift_potential)),
        elec=_lib.ELEC[params.elec], k_rf=params.k_rf, c_rf=params.c_rf, ewald_beta=params.ewald_beta)
    if getattr(params, "__dataclass_params__", None) is not None and params.__dataclass_params__.frozen:
        _last_params[:] = [(params, p, table)]
    return p, table


def _check_shapes(plist, grid, layout, n_pos):
    if layout.m != grid.m or plist.m != grid.m:
        raise ParameterError(f"layout m={layout.m}, grid m={grid.m}, list m={plist.m} must agree")
    if n_pos != grid.n:
        raise ParameterError(f"positions must have shape ({grid.n}, 3), got ({n_pos}, 3)")
    if plist.grid is not grid and plist.grid.n_clusters != grid.n_clusters:
        raise ParameterError("pair list was built for a different grid")


def compute_nonbonded_device(plist: ClusterPairList, grid: ClusterGrid, positions: torch.Tensor,
                             charges: torch.Tensor, lj_types: torch.Tensor, params: NonbondedParams,
                             box: SimBox, *, energy: bool = True, clustered: bool = False,
                             out: torch.Tensor | None = None, accumulate: bool = False,
                             e_out: torch.Tensor | None = None, bad: torch.Tensor | None = None,
                             i_clusters: torch.Tensor | None = None, canonical: bool = False,
                             reprune: bool = False):
    """Device-resident force pass.  CUDA tensors in (original order), CUDA
    tensors out; nothing synchronises.  Returns (forces, energies[2], bad[2]).

    ``reprune`` (dynamic pruning, lists pruned with ``r_inner``): after the
    pass, redo the inner force list at these positions (rolling prune,
    GROMACS' nstlistPrune); its validity is then measured from them."""
    d = dev.require_cuda()
    n_out = grid.n_slots if clustered else grid.n
    if out is None:
        out = torch.empty((n_out, 3), dtype=torch.float64, device=d)
        accumulate = False
    if e_out is None:
        e_out = torch.zeros(2, dtype=torch.float64, device=d)
    if bad is None:
        bad = torch.empty(2, dtype=torch.int64, device=d)
    p, table = _params_struct(params)
    L = _lib.box3(box.lengths)
    flags = ((_lib.FORCE_ENERGY if energy else 0) | (_lib.FORCE_ACCUMULATE if accumulate else 0)
             | (_lib.FORCE_CLUSTERED if clustered else 0) | (_lib.FORCE_CANONICAL if canonical else 0)
             | (_lib.FORCE_REPRUNE if reprune else 0))
    n_sel = 0 if i_clusters is None else int(i_clusters.numel())
    _lib.check(_lib.load().nbx_force(
        plist.handle, grid.handle, _lib.ptr(positions), _lib.ptr(charges), _lib.ptr(lj_types),
        ctypes.byref(p), _lib.ptr(L), _lib.ptr(i_clusters), n_sel, flags, _lib.ptr(out),
        _lib.ptr(e_out), _lib.ptr(bad), dev.stream()), "force")
    del table
    return out, e_out, bad


def _raise_if_singular(plist, grid, pos_t, bad_h, params, box):
    if bad_h[0] == -1:
        return
    if bad_h[0] == -2:  # non-finite forces: locate the coincident pair exactly
        found = np.zeros(2, dtype=np.int64)
        L = _lib.box3(box.lengths)
        _lib.check(_lib.load().nbx_find_singular(plist.handle, grid.handle, _lib.ptr(pos_t),
                                                 float(params.r_cut), _lib.ptr(L), dev.stream(),
                                                 _lib.ptr(found)), "find_singular")
        if found[0] < 0:
            return
        bad_h = found
    oi, oj = int(grid.perm[bad_h[0]]), int(grid.perm[bad_h[1]])
    raise SingularityError(f"particles {oi} and {oj} overlap exactly", i=oi, j=oj)


def _sel_clusters(plist: ClusterPairList, i_sel) -> torch.Tensor:
    sel = np.asarray(i_sel, dtype=np.int64).reshape(-1)
    if plist.supercluster_size > 1:
        s = plist.supercluster_size
        sel = (sel[:, None] * s + np.arange(s)[None, :]).reshape(-1)
        sel = sel[sel < plist.n_i_clusters]
    return dev.to_device(sel.astype(np.int32), torch.int32)


def compute_nonbonded_into(plist: ClusterPairList, grid: ClusterGrid, positions, charges, lj_types,
                           params: NonbondedParams, box: SimBox, layout: KernelLayout, f_out,
                           i_sel=None) -> tuple[float, float]:
    """Accumulate clustered (n_slots, 3) forces for all i-clusters, or the
    subset i_sel (super groups when the list has a super layout); returns
    (e_lj, e_coulomb) of that subset (kernels.py:328-396)."""
    pos_shape = tuple(positions.shape)
    if len(pos_shape) != 2 or pos_shape[1] != 3:
        raise ParameterError(f"positions must have shape ({grid.n}, 3), got {pos_shape}")
    _check_shapes(plist, grid, layout, pos_shape[0])
    if tuple(f_out.shape) != (grid.n_slots, 3):
        raise ParameterError(f"f_out must have shape ({grid.n_slots}, 3), got {tuple(f_out.shape)}")
    pos_t = dev.to_device(positions, torch.float64)
    q_t = dev.to_device(charges, torch.float64)
    t_t = dev.to_device(lj_types, torch.int64)
    sel_t = None if i_sel is None else _sel_clusters(plist, i_sel)
    if dev.is_device_tensor(f_out) and f_out.dtype == torch.float64 and f_out.is_contiguous():
        _, e, bad = compute_nonbonded_device(plist, grid, pos_t, q_t, t_t, params, box, clustered=True,
                                             out=f_out, accumulate=True, i_clusters=sel_t)
        host_add = None
    else:
        fo, e, bad = compute_nonbonded_device(plist, grid, pos_t, q_t, t_t, params, box, clustered=True,
                                              i_clusters=sel_t)
        host_add = fo
    e_h = e.cpu().numpy()
    _raise_if_singular(plist, grid, pos_t, bad.cpu().numpy(), params, box)
    if host_add is not None:
        f_out += host_add.cpu().numpy()
    return float(e_h[0]), float(e_h[1])


def compute_nonbonded(plist: ClusterPairList, grid: ClusterGrid, positions, charges, lj_types,
                      params: NonbondedParams, box: SimBox, layout: KernelLayout) -> ForcesEnergies:
    """Forces (clustered slot order) and energies over the full list (kernels.py:399-419)."""
    f_out = np.zeros((grid.n_slots, 3), dtype=np.float64)
    e_lj, e_c = compute_nonbonded_into(plist, grid, positions, charges, lj_types, params, box, layout, f_out)
    return ForcesEnergies(forces=f_out, e_lj=e_lj, e_coulomb=e_c)


def compute_nonbonded_original(plist: ClusterPairList, grid: ClusterGrid, positions, charges, lj_types,
                               params: NonbondedParams, box: SimBox, layout: KernelLayout) -> ForcesEnergies:
    """Forces in original particle order (kernels.py:422-440); the scatter is
    fused into the GPU reduction."""
    pos_shape = tuple(positions.shape)
    if len(pos_shape) != 2 or pos_shape[1] != 3:
        raise ParameterError(f"positions must have shape ({grid.n}, 3), got {pos_shape}")
    _check_shapes(plist, grid, layout, pos_shape[0])
    # host arrays move through pinned staging (read-only charges / types are
    # recognised and uploaded once); results come back in one synchronisation
    pos_t = dev.stage_in(positions, torch.float64, "positions")
    # forces, energies and the singular-pair key in one device buffer: one
    # read-back and one synchronisation
    n = pos_shape[0]
    buf = dev.scratch("nonbonded_out", 3 * n + 4, torch.float64)
    f_d, e_d, bad_d = buf[:3 * n].view(n, 3), buf[3 * n:3 * n + 2], buf[3 * n + 2:].view(torch.int64)
    compute_nonbonded_device(plist, grid, pos_t, dev.stage_in(charges, torch.float64, "charges"),
                             dev.stage_in(lj_types, torch.int64, "lj_types"), params, box, out=f_d, e_out=e_d,
                             bad=bad_d)
    out = dev.stage_out(buf, "nonbonded_out")  # a fresh array (ForcesEnergies freezes the forces in place)
    bad_h = out[3 * n + 2:].view(np.int64)
    _raise_if_singular(plist, grid, pos_t, bad_h, params, box)
    return ForcesEnergies(forces=out[:3 * n].reshape(n, 3), e_lj=float(out[3 * n]), e_coulomb=float(out[3 * n + 1]))


def flop_count(plist: ClusterPairList, grid: ClusterGrid, layout: KernelLayout, box: SimBox,
               r_cut: float) -> FlopCount:
    """Reference cost model (kernels.py:443-473): total = every m x n_lane
    block slot of the canonical traversal, useful = pairs within r_cut."""
    if layout.m != plist.m:
        raise ParameterError(f"layout m={layout.m} does not match list m={plist.m}")
    counts = np.diff(plist.offsets)
    ju, m, nl = layout.j_unroll, layout.m, layout.n_lane
    blocks = (counts // ju) * ((ju * m + nl - 1) // nl)
    rem = counts % ju
    blocks = blocks + np.where(rem > 0, (rem * m + nl - 1) // nl, 0)
    total_slots = int(blocks.sum()) * nl * m
    stats = interaction_stats(plist, grid, plist.build_positions, box, r_cut)
    return FlopCount(useful_flops=stats.n_within_cutoff * FLOPS_PER_PAIR,
                     total_flops=total_slots * FLOPS_PER_PAIR)

