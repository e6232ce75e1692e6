"""Pair potential, list-driven force pass and brute force (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/clustermd/kernels.py:84-121 (potential),
:124-221 (canonical blocked kernel) and oracle.py:28-85 (brute force).

Electrostatics extension (parity UNPINNED: the reference only has cutoff
Coulomb with an optional potential shift, kernels.py:84-111):
  elec="cutoff"          reference form; E_c = qq/r (- qq/r_c when shifted)
  elec="reaction_field"  E_c = qq (1/r + k_rf r^2 - c_rf),  F/r = qq (1/r^3 - 2 k_rf)
                         k_rf = (eps_rf - 1)/((2 eps_rf + 1) r_c^3)  (eps_rf = 0 -> inf)
                         c_rf = 1/r_c + k_rf r_c^2.  eps_rf = 1 reproduces the
                         reference's shifted cutoff Coulomb exactly.
  elec="ewald"           E_c = qq erfc(beta r)/r (- qq erfc(beta r_c)/r_c when shifted)
                         F/r = qq (erfc(beta r)/r + 2 beta/sqrt(pi) exp(-beta^2 r^2)) / r^2
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.special import erfc

from .geometry import COULOMB_CONSTANT, min_image
from .search import row_ci

# kernels.py:34-42 -- the reference's flop cost model per evaluated slot pair
FLOPS_PER_PAIR = 17 + 12 + 11
# our extension: +12 for the erfc/exp evaluation of the Ewald real-space term
FLOPS_PER_PAIR_EWALD = FLOPS_PER_PAIR + 12


@dataclass(frozen=True)
class Physics:
    r_cut: float
    lj_table: np.ndarray            # (t, t, 2) [eps, sigma]
    coulomb_scale: float = COULOMB_CONSTANT
    shift_potential: bool = False
    elec: str = "cutoff"            # cutoff | reaction_field | ewald
    epsilon_rf: float = 1.0
    ewald_beta: float = 0.0

    def k_rf(self) -> float:
        if self.elec != "reaction_field":
            return 0.0
        if self.epsilon_rf == 0.0:
            return 1.0 / (2.0 * self.r_cut ** 3)
        return (self.epsilon_rf - 1.0) / ((2.0 * self.epsilon_rf + 1.0) * self.r_cut ** 3)

    def c_rf(self) -> float:
        return 1.0 / self.r_cut + self.k_rf() * self.r_cut * self.r_cut


def ewald_beta_for(r_cut: float, rtol: float = 1e-5) -> float:
    """beta with erfc(beta r_c) = rtol (bisection, as GROMACS calc_ewaldcoeff_q)."""
    lo, hi = 0.0, 5.0
    while erfc(hi * r_cut) > rtol:
        hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if erfc(mid * r_cut) > rtol:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def pair_terms(r2, ti, tj, qi, qj, phys: Physics):
    """kernels.py:84-111 (+ extension): returns (e_lj, e_coul, f_over_r).

    For elec="cutoff" this is the reference's expression sequence verbatim
    (sr2 = sig^2/r2, sr6 = sr2^3, ...), so results are bitwise equal."""
    r2 = np.asarray(r2, dtype=np.float64)
    eps = phys.lj_table[ti, tj, 0]
    sig = phys.lj_table[ti, tj, 1]
    sr2 = (sig * sig) / r2
    sr6 = sr2 * sr2 * sr2
    e_lj = 4.0 * eps * (sr6 * sr6 - sr6)
    f_over_r = 48.0 * eps * (sr6 * sr6 - 0.5 * sr6) / r2
    r = np.sqrt(r2)
    qq = phys.coulomb_scale * np.asarray(qi, dtype=np.float64) * qj
    if phys.elec == "cutoff":
        e_c = qq / r
        f_over_r = f_over_r + qq / (r2 * r)
        if phys.shift_potential:
            e_c = e_c - qq / phys.r_cut
    elif phys.elec == "reaction_field":
        k_rf, c_rf = phys.k_rf(), phys.c_rf()
        e_c = qq * (1.0 / r + k_rf * r2 - c_rf)
        f_over_r = f_over_r + qq * (1.0 / (r2 * r) - 2.0 * k_rf)
    elif phys.elec == "ewald":
        b = phys.ewald_beta
        erfc_br = erfc(b * r)
        e_c = qq * erfc_br / r
        f_over_r = f_over_r + qq * (erfc_br / r + 2.0 * b / math.sqrt(math.pi) * np.exp(-b * b * r2)) / r2
        if phys.shift_potential:
            e_c = e_c - qq * erfc(b * phys.r_cut) / phys.r_cut
    else:
        raise ValueError(f"unknown elec {phys.elec!r}")
    if phys.shift_potential:
        rc2 = phys.r_cut * phys.r_cut
        src2 = (sig * sig) / rc2
        src6 = src2 * src2 * src2
        e_lj = e_lj - 4.0 * eps * (src6 * src6 - src6)
    return e_lj, e_c, f_over_r


def list_forces(lst: dict, grid: dict, positions, charges, lj_type, lengths, phys: Physics):
    """kernels.py:328-396 + :124-221 in vectorized numpy: gather by perm,
    every admitted slot pair with min-image r^2 <= r_c^2 (closed ball),
    Newton-3 accumulation into clustered slots.  Returns (f_clustered,
    e_lj, e_coul).  Summation order differs from the numba kernel, so
    forces agree to ~1e-13, not bitwise (same as the reference's own
    cross-layout tolerance, test_kernels.py:188-209)."""
    m = lst["m"]
    perm = grid["perm"]
    pos = np.asarray(positions, dtype=np.float64)[perm]
    q = np.asarray(charges, dtype=np.float64)[perm]
    t = np.asarray(lj_type, dtype=np.int64)[perm]
    n_slots = perm.shape[0]
    f = np.zeros((n_slots, 3))
    p, a, b = np.nonzero(lst["masks"])
    ci = row_ci(lst)
    si = ci[p] * m + a
    sj = lst["j_idx"][p] * m + b
    dr = min_image(pos[si] - pos[sj], lengths)
    r2 = dr[:, 0] * dr[:, 0] + dr[:, 1] * dr[:, 1] + dr[:, 2] * dr[:, 2]
    inside = r2 <= phys.r_cut * phys.r_cut
    if np.any(inside & (r2 == 0.0)):
        k = int(np.nonzero(inside & (r2 == 0.0))[0][0])
        raise ZeroDivisionError(f"singular pair slots {si[k]} {sj[k]}")
    si, sj, dr, r2 = si[inside], sj[inside], dr[inside], r2[inside]
    e_lj, e_c, fr = pair_terms(r2, t[si], t[sj], q[si], q[sj], phys)
    fv = fr[:, None] * dr
    np.add.at(f, si, fv)
    np.add.at(f, sj, -fv)
    return f, float(np.sum(e_lj)), float(np.sum(e_c))


def brute_force(positions, charges, lj_type, lengths, phys: Physics, molecules=None, abs_sums=False):
    """oracle.py:28-67: all pairs within r_c, original order, O(n^2).
    ``molecules`` (extension, rigid water): pairs within one molecule are
    excluded.  ``abs_sums``: also return (sum |E_lj pair|, sum |E_c pair|),
    the scale of the cancelling sums."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    mol = None if molecules is None else np.asarray(molecules)
    n = pos.shape[0]
    charges = np.asarray(charges, dtype=np.float64)
    lj_type = np.asarray(lj_type, dtype=np.int64)
    f = np.zeros((n, 3))
    e_lj = 0.0
    e_c = 0.0
    rc2 = phys.r_cut * phys.r_cut
    a_lj = a_c = 0.0
    for i in range(n - 1):
        dr = min_image(pos[i] - pos[i + 1:], lengths)
        r2 = np.einsum("kd,kd->k", dr, dr)
        keep = r2 <= rc2
        if mol is not None:
            keep &= mol[i + 1:] != mol[i]
        idx = np.nonzero(keep)[0]
        if idx.shape[0] == 0:
            continue
        if np.any(r2[idx] == 0.0):
            raise ZeroDivisionError(f"singular pair {i}")
        a, c, fr = pair_terms(r2[idx], lj_type[i], lj_type[i + 1 + idx], charges[i],
                              charges[i + 1 + idx], phys)
        e_lj += float(np.sum(a))
        e_c += float(np.sum(c))
        a_lj += float(np.sum(np.abs(a)))
        a_c += float(np.sum(np.abs(c)))
        fv = fr[:, None] * dr[idx]
        f[i] += fv.sum(axis=0)
        f[i + 1 + idx] -= fv
    if abs_sums:
        return f, e_lj, e_c, (a_lj, a_c)
    return f, e_lj, e_c


def brute_pairs(positions, lengths, r) -> set:
    """oracle.py:70-85: all (i, j), i < j, with min-image d <= r."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    out = set()
    for i in range(pos.shape[0] - 1):
        dr = min_image(pos[i] - pos[i + 1:], lengths)
        r2 = np.einsum("kd,kd->k", dr, dr)
        for j in np.nonzero(r2 <= r * r)[0]:
            out.add((i, i + 1 + int(j)))
    return out
