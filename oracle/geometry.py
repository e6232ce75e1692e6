"""Periodic geometry restated from the reference (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/clustermd/model.py:147-172.  The operation
order is kept literally because the GPU search/prune kernels are required to
reproduce these FP64 results bit for bit.
"""

from __future__ import annotations

import numpy as np

# model.py:17 -- 1/(4 pi eps0) in kJ mol^-1 nm e^-2
COULOMB_CONSTANT = 138.935458
# model.py:20
BOLTZMANN_KJ_MOL_K = 0.008314462618


def wrap(p, lengths) -> np.ndarray:
    """model.py:147-156: np.mod into [0, L), then fold a result equal to L."""
    lengths = np.asarray(lengths, dtype=np.float64)
    out = np.mod(np.asarray(p, dtype=np.float64), lengths)
    return np.where(out >= lengths, out - lengths, out)


def min_image(dr, lengths) -> np.ndarray:
    """model.py:159-172: dr - floor(dr/L + 0.5)*L, folded to [-L/2, L/2)."""
    lengths = np.asarray(lengths, dtype=np.float64)
    dr = np.asarray(dr, dtype=np.float64)
    out = dr - np.floor(dr / lengths + 0.5) * lengths
    half = 0.5 * lengths
    out = np.where(out >= half, out - lengths, out)
    return np.where(out < -half, out + lengths, out)
