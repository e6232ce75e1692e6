"""Synthetic inputs for the nbnxn path: SPC-geometry water boxes.

The recipe is the one BASELINE.md section 2 fixes for the reference CPU
measurements (and SURVEY.md section 8d for the benchmark):

  * n_mol = n/3 molecules at 33.43 nm^-3, cubic box edge (n_mol/33.43)^(1/3);
  * molecule sites on a k^3 lattice (k = smallest int with k^3 >= n_mol),
    jittered uniformly by +-0.1 lattice spacing (first RNG draw);
  * random orientation from a normalised Gaussian quaternion (w, x, y, z)
    (second RNG draw);
  * O at the site, H1 = O + R (0.1, 0, 0), H2 = O + R (0.1 cos 109.47 deg,
    0.1 sin 109.47 deg, 0); atom order O, H, H; positions wrapped;
  * lj_type [0, 1, 1], charges [-0.82, +0.41, +0.41], masses
    [15.9994, 1.008, 1.008]; LJ table O-O (0.650194 kJ/mol, 0.316557 nm),
    every H entry epsilon 0 with a positive placeholder sigma 0.1 (the
    reference's validate_system requires sigma > 0, model.py:219-220).

Velocities are zero unless a temperature is given (Maxwell-Boltzmann with
the net momentum removed, cli.py:231-238).
"""

from __future__ import annotations

import math

import numpy as np

from .model import BOLTZMANN_KJ_MOL_K, ParameterError, ParticleSystem, SimBox, wrap_position

SPC_DENSITY_MOL_NM3 = 33.43
SPC_OH = 0.1
SPC_ANGLE_DEG = 109.47
SPC_CHARGES = (-0.82, 0.41, 0.41)
SPC_MASSES = (15.9994, 1.008, 1.008)
SPC_LJ_TABLE = np.array(
    [[[0.650194, 0.316557], [0.0, 0.1]],
     [[0.0, 0.1], [0.0, 0.1]]]
)


def _rotation(qs: np.ndarray) -> np.ndarray:
    w, x, y, z = qs[:, 0], qs[:, 1], qs[:, 2], qs[:, 3]
    r = np.empty((qs.shape[0], 3, 3))
    r[:, 0, 0] = 1 - 2 * (y * y + z * z)
    r[:, 0, 1] = 2 * (x * y - z * w)
    r[:, 0, 2] = 2 * (x * z + y * w)
    r[:, 1, 0] = 2 * (x * y + z * w)
    r[:, 1, 1] = 1 - 2 * (x * x + z * z)
    r[:, 1, 2] = 2 * (y * z - x * w)
    r[:, 2, 0] = 2 * (x * z - y * w)
    r[:, 2, 1] = 2 * (y * z + x * w)
    r[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def spc_water(n_atoms: int, seed: int = 2024, temperature: float = 0.0):
    """SPC-geometry water box with n_atoms (a multiple of 3).

    Returns (ParticleSystem, lj_table)."""
    if n_atoms < 3 or n_atoms % 3:
        raise ValueError(f"n_atoms must be a positive multiple of 3, got {n_atoms}")
    n_mol = n_atoms // 3
    edge = (n_mol / SPC_DENSITY_MOL_NM3) ** (1.0 / 3.0)
    k = 1
    while k * k * k < n_mol:
        k += 1
    spacing = edge / k
    rng = np.random.default_rng(seed)
    i = np.arange(n_mol)
    sites = np.stack([i // (k * k), (i // k) % k, i % k], axis=1).astype(np.float64) * spacing
    sites = sites + rng.uniform(-0.1, 0.1, (n_mol, 3)) * spacing
    qs = rng.normal(size=(n_mol, 4))
    qs /= np.linalg.norm(qs, axis=1, keepdims=True)
    rot = _rotation(qs)
    theta = math.radians(SPC_ANGLE_DEG)
    h1 = np.array([SPC_OH, 0.0, 0.0])
    h2 = np.array([SPC_OH * math.cos(theta), SPC_OH * math.sin(theta), 0.0])
    pos = np.empty((n_mol, 3, 3))
    pos[:, 0] = sites
    pos[:, 1] = sites + rot @ h1
    pos[:, 2] = sites + rot @ h2
    box = SimBox([edge, edge, edge])
    positions = wrap_position(pos.reshape(-1, 3), box)
    masses = np.tile(np.asarray(SPC_MASSES), n_mol)
    if temperature > 0.0:
        scale = np.sqrt(BOLTZMANN_KJ_MOL_K * temperature / masses)
        vel = scale[:, None] * rng.standard_normal((n_atoms, 3))
        total = masses.sum()
        for _ in range(2):
            vel = vel - np.einsum("k,kd->d", masses, vel) / total
    else:
        vel = np.zeros((n_atoms, 3))
    system = ParticleSystem(
        positions=positions,
        velocities=vel,
        masses=masses,
        charges=np.tile(np.asarray(SPC_CHARGES), n_mol),
        lj_type=np.tile(np.array([0, 1, 1], dtype=np.int64), n_mol),
        box=box,
    )
    return system, SPC_LJ_TABLE.copy()


def tuned_occupancy(n_atoms: int, box_edge: float, m: int) -> float:
    """m^(2/3) rho^(1/3) L: columns whose clusters are about as tall as they
    are wide; passed as build_cluster_grid's
    target_occupancy (gridder.py:69-71)."""
    rho = n_atoms / box_edge ** 3
    return m ** (2.0 / 3.0) * rho ** (1.0 / 3.0) * box_edge


# ---------------------------------------------------------------- reference fluids and system files
# the reference's generators (cli.py:158-250) and JSON system
# files (model.py:232-277), so fixtures and CLI-style workflows run unchanged.
ARGON_EPSILON = 0.996   # kJ/mol (cli.py:52)
ARGON_SIGMA = 0.34      # nm
ARGON_MASS = 39.948     # u
NEON_MASS = 20.180      # u (second species of the charged fluid)


class GenerationError(RuntimeError):
    """The requested density cannot host the lattice with the minimum separation (cli.py:59)."""


def _fluid_species(kind: str, n: int, charge: float):
    """(lj_table, lj_type, masses, charges) of the reference's two fluids."""
    if kind == "lj_fluid":
        return (np.array([[[ARGON_EPSILON, ARGON_SIGMA]]]), np.zeros(n, dtype=np.int64),
                np.full(n, ARGON_MASS), np.zeros(n))
    if kind == "charged_fluid":
        eps, sig = (ARGON_EPSILON, 0.8), (ARGON_SIGMA, 0.30)
        mix = (math.sqrt(eps[0] * eps[1]), 0.5 * (sig[0] + sig[1]))   # geometric eps, arithmetic sigma
        table = np.array([[[eps[0], sig[0]], list(mix)], [list(mix), [eps[1], sig[1]]]])
        alt = np.arange(n) % 2
        q = charge * np.where(alt == 0, 1.0, -1.0)
        if n % 2:
            q[-1] = 0.0  # neutral box for odd counts
        return table, alt.astype(np.int64), np.where(alt == 0, ARGON_MASS, NEON_MASS), q
    raise ParameterError(f"unknown system kind {kind!r}")


def generate_system(kind: str, n: int, density: float, temperature: float, seed: int,
                    charge: float = 0.2) -> tuple[ParticleSystem, np.ndarray]:
    """Deterministic lattice-plus-jitter fluid in a cubic box (cli.py:158-250):
    same arguments, same random stream, same system as the reference."""
    if n < 1:
        raise ParameterError(f"n must be >= 1, got {n}")
    if density <= 0.0:
        raise ParameterError(f"density must be positive, got {density}")
    if temperature < 0.0:
        raise ParameterError(f"temperature must be >= 0, got {temperature}")
    table, types, masses, charges = _fluid_species(kind, n, charge)
    edge = (n / density) ** (1.0 / 3.0)
    k = max(1, int(round(n ** (1.0 / 3.0))))
    while k ** 3 < n:
        k += 1
    spacing = edge / k
    min_sep = 0.8 * float(table[:, :, 1].max())
    if spacing <= min_sep:
        raise GenerationError(f"density {density} nm^-3 packs lattice spacing {spacing:.4f} nm "
                              f"below the minimum separation {min_sep:.4f} nm")
    i = np.arange(n)
    pos = np.stack([i // (k * k), (i // k) % k, i % k], axis=1).astype(np.float64) * spacing
    rng = np.random.default_rng(seed)
    if n > 1:
        jitter = 0.45 * (spacing - min_sep)
        pos = pos + rng.uniform(-jitter, jitter, (n, 3))
    if temperature > 0.0:
        vel = np.sqrt(BOLTZMANN_KJ_MOL_K * temperature / masses)[:, None] * rng.standard_normal((n, 3))
        if n > 1:
            total = masses.sum()
            for _ in range(2):  # the second pass removes the rounding residue
                vel = vel - np.einsum("k,kd->d", masses, vel) / total
    else:
        vel = np.zeros((n, 3))
    box = SimBox([edge, edge, edge])
    return ParticleSystem(positions=pos, velocities=vel, masses=masses, charges=charges, lj_type=types,
                          box=box), table


_SYSTEM_KEYS = ("box", "positions", "velocities", "masses", "charges", "lj_type", "lj_table")


def save_system(path, system: ParticleSystem, lj_table) -> None:
    """System + LJ table as deterministic JSON, the reference's file format (model.py:232-246)."""
    import json

    doc = dict(zip(_SYSTEM_KEYS, (system.box.lengths.tolist(), system.positions.tolist(),
                                  system.velocities.tolist(), system.masses.tolist(), system.charges.tolist(),
                                  system.lj_type.tolist(), np.asarray(lj_table, dtype=np.float64).tolist())))
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")


def load_system(path) -> tuple[ParticleSystem, np.ndarray]:
    """Inverse of save_system (model.py:249-277); ParameterError on missing keys."""
    import json

    with open(path) as fh:
        doc = json.load(fh)
    missing = [k for k in _SYSTEM_KEYS if k not in doc]
    if missing:
        raise ParameterError(f"system file {path} missing keys: {missing}")
    system = ParticleSystem(positions=doc["positions"], velocities=doc["velocities"], masses=doc["masses"],
                            charges=doc["charges"], lj_type=doc["lj_type"], box=SimBox(doc["box"]))
    table = np.array(doc["lj_table"], dtype=np.float64)
    table.setflags(write=False)
    return system, table
