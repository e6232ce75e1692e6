"""Rigid 3-site water for the SPC extension: FP64 numpy
restatements used only to CHECK the device path (test infrastructure; the
product never imports oracle/).

The reference has no constraints, so this is
parity unpinned by the reference; it is pinned here by two independent
algorithms agreeing:

  settle_positions   analytic SETTLE (Miyamoto & Kollman, J. Comput. Chem. 13,
                     952 (1992)): O at the apex, H1/H2; the new positions are
                     the unconstrained ones plus constraint displacements
                     along the OLD bond vectors, solved in closed form in the
                     frame of the old molecule plane;
  shake_positions    SHAKE (Ryckaert, Ciccotti & Berendsen 1977) iterated to
                     convergence on the same three distance constraints with
                     the same old-bond directions: converges to the same
                     solution, so the two must agree to rounding;
  rattle_velocities  RATTLE's velocity stage (Andersen 1983): remove the bond-
                     stretching components of the velocities by solving the
                     3x3 linear system of the Lagrange multipliers.

Molecules are atoms (3k, 3k+1, 3k+2) = (O, H1, H2); positions are wrapped
per atom, so every bond vector is a minimum image.
"""

from __future__ import annotations

import numpy as np

from .geometry import min_image, wrap


def _mi(dr, L):
    return min_image(dr, L)


def settle_positions(x_old, x_new, masses, L, d_oh, d_hh):
    """Constrained positions (wrapped) for unconstrained x_new, given the
    constrained x_old of the previous step; returns (x, displacement) where
    displacement = x - x_new (minimum image, per atom)."""
    x_old = np.asarray(x_old, dtype=np.float64).reshape(-1, 3, 3)
    x_new = np.asarray(x_new, dtype=np.float64).reshape(-1, 3, 3)
    mO, mH = float(masses[0]), float(masses[1])
    wohh = mO + 2.0 * mH
    rc = 0.5 * d_hh
    h = np.sqrt(d_oh * d_oh - rc * rc)
    ra = 2.0 * mH * h / wohh
    rb = h - ra
    b0 = _mi(x_old[:, 1] - x_old[:, 0], L)
    c0 = _mi(x_old[:, 2] - x_old[:, 0], L)
    B1 = _mi(x_new[:, 1] - x_new[:, 0], L)
    C1 = _mi(x_new[:, 2] - x_new[:, 0], L)
    com = (mH * B1 + mH * C1) / wohh            # relative to the new O
    a1, b1, c1 = -com, B1 - com, C1 - com
    n = np.cross(b0, c0)                         # old plane normal (local z)
    ex = np.cross(a1, n)                         # local x
    ey = np.cross(n, ex)                         # local y
    ex /= np.linalg.norm(ex, axis=1, keepdims=True)
    ey /= np.linalg.norm(ey, axis=1, keepdims=True)
    ez = n / np.linalg.norm(n, axis=1, keepdims=True)

    def loc(v):
        return np.einsum("kd,kd->k", v, ex), np.einsum("kd,kd->k", v, ey), np.einsum("kd,kd->k", v, ez)

    xb0d, yb0d, _ = loc(b0)
    xc0d, yc0d, _ = loc(c0)
    _, _, za1d = loc(a1)
    xb1d, yb1d, zb1d = loc(b1)
    xc1d, yc1d, zc1d = loc(c1)
    sinphi = za1d / ra
    cosphi = np.sqrt(1.0 - sinphi * sinphi)
    sinpsi = (zb1d - zc1d) / (2.0 * rc * cosphi)
    cospsi = np.sqrt(1.0 - sinpsi * sinpsi)
    ya2d = ra * cosphi
    xb2d = -rc * cospsi
    t1 = -rb * cosphi
    t2 = rc * sinpsi * sinphi
    yb2d = t1 - t2
    yc2d = t1 + t2
    alpha = xb2d * (xb0d - xc0d) + yb0d * yb2d + yc0d * yc2d
    beta = xb2d * (yc0d - yb0d) + xb0d * yb2d + xc0d * yc2d
    gamma = xb0d * yb1d - xb1d * yb0d + xc0d * yc1d - xc1d * yc0d
    al2be2 = alpha * alpha + beta * beta
    sintheta = (alpha * gamma - beta * np.sqrt(al2be2 - gamma * gamma)) / al2be2
    costheta = np.sqrt(1.0 - sintheta * sintheta)
    a3 = np.stack([-ya2d * sintheta, ya2d * costheta, za1d], axis=1)
    b3 = np.stack([xb2d * costheta - yb2d * sintheta, xb2d * sintheta + yb2d * costheta, zb1d], axis=1)
    c3 = np.stack([-xb2d * costheta - yc2d * sintheta, -xb2d * sintheta + yc2d * costheta, zc1d], axis=1)

    def lab(v):
        return v[:, 0:1] * ex + v[:, 1:2] * ey + v[:, 2:3] * ez

    # new positions relative to the unconstrained oxygen
    rel = np.stack([com + lab(a3), com + lab(b3), com + lab(c3)], axis=1)
    disp = rel - np.stack([np.zeros_like(B1), B1, C1], axis=1)
    x = wrap((x_new + disp).reshape(-1, 3), L)
    return x, disp.reshape(-1, 3)


def shake_positions(x_old, x_new, masses, L, d_oh, d_hh, tol=1e-15, max_iter=10000):
    """Iterative SHAKE on the same constraints (validation of settle_positions)."""
    x_old = np.asarray(x_old, dtype=np.float64).reshape(-1, 3, 3)
    x_new = np.asarray(x_new, dtype=np.float64).reshape(-1, 3, 3)
    m = np.asarray(masses[:3], dtype=np.float64)
    bonds = [(0, 1, d_oh), (0, 2, d_oh), (1, 2, d_hh)]
    rel_new = np.stack([np.zeros_like(x_new[:, 0]), _mi(x_new[:, 1] - x_new[:, 0], L),
                        _mi(x_new[:, 2] - x_new[:, 0], L)], axis=1)
    rel_old = np.stack([np.zeros_like(x_old[:, 0]), _mi(x_old[:, 1] - x_old[:, 0], L),
                        _mi(x_old[:, 2] - x_old[:, 0], L)], axis=1)
    r = rel_new.copy()
    for _ in range(max_iter):
        worst = 0.0
        for i, j, d in bonds:
            rij = r[:, j] - r[:, i]
            diff = np.einsum("kd,kd->k", rij, rij) - d * d
            worst = max(worst, float(np.abs(diff).max()))
            s = rel_old[:, j] - rel_old[:, i]
            g = diff / (2.0 * (1.0 / m[i] + 1.0 / m[j]) * np.einsum("kd,kd->k", rij, s))
            r[:, i] += (g / m[i])[:, None] * s
            r[:, j] -= (g / m[j])[:, None] * s
        if worst < tol:
            break
    disp = r - rel_new
    x = wrap((x_new + disp).reshape(-1, 3), L)
    return x, disp.reshape(-1, 3)


def rattle_velocities(x, v, masses, L):
    """Velocities with the bond-stretching components removed (RATTLE stage 2):
    r_b . (v_j - v_i) = 0 for the three bonds of every molecule."""
    x = np.asarray(x, dtype=np.float64).reshape(-1, 3, 3)
    v = np.array(v, dtype=np.float64).reshape(-1, 3, 3)
    m = np.asarray(masses[:3], dtype=np.float64)
    bonds = [(0, 1), (0, 2), (1, 2)]
    r = [_mi(x[:, j] - x[:, i], L) for i, j in bonds]
    A = np.zeros((x.shape[0], 3, 3))
    rhs = np.zeros((x.shape[0], 3))
    # correction: v_i += lam_b r_b / m_i, v_j -= lam_b r_b / m_j
    for c, (ic, jc) in enumerate(bonds):
        rhs[:, c] = -np.einsum("kd,kd->k", r[c], v[:, jc] - v[:, ic])
        for b, (ib, jb) in enumerate(bonds):
            coef = 0.0
            coef += (-1.0 / m[jb]) if jb == jc else 0.0
            coef += (1.0 / m[ib]) if ib == jc else 0.0
            coef -= (-1.0 / m[jb]) if jb == ic else 0.0
            coef -= (1.0 / m[ib]) if ib == ic else 0.0
            A[:, c, b] = coef * np.einsum("kd,kd->k", r[c], r[b])
    lam = np.linalg.solve(A, rhs[:, :, None])[:, :, 0]
    for b, (ib, jb) in enumerate(bonds):
        v[:, ib] += (lam[:, b] / m[ib])[:, None] * r[b]
        v[:, jb] -= (lam[:, b] / m[jb])[:, None] * r[b]
    return v.reshape(-1, 3)
