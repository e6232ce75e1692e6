"""ctypes binding of oracle/c/oracle.c (TEST INFRASTRUCTURE / CPU BASELINE ONLY).

Build with ``make -C oracle/c`` (``__graft_entry__.build()`` does it).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import search
from .forces import Physics

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None

_ELEC = {"cutoff": 0, "reaction_field": 1, "ewald": 2}


def build() -> Path:
    import subprocess

    subprocess.run(["make", "-s", "-C", str(_HERE / "c")], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        INT = ctypes.c_int
        _lib.orc_search_n2.restype = I64
        _lib.orc_search_n2.argtypes = [I64, P, P, D, P, P, P, INT]
        _lib.orc_search_cols.restype = I64
        _lib.orc_search_cols.argtypes = [I64, P, P, P, I64, P, D, P, P, P, INT]
        _lib.orc_row_min_d2.restype = None
        _lib.orc_row_min_d2.argtypes = [I64, INT, P, P, P, P, P, P, INT]
        _lib.orc_count_within.restype = I64
        _lib.orc_count_within.argtypes = [I64, INT, P, P, P, P, P, D, INT]
        _lib.orc_force.restype = INT
        _lib.orc_force.argtypes = [I64, INT, P, P, P, P, P, P, INT, P, P, P, INT, INT, D, D, D, D,
                                   D, P, INT, P, P, P]
        _lib.orc_max_threads.restype = INT
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def search_list(grid: dict, lengths, r_list: float, method: str = "cols", threads: int | None = None) -> dict:
    """pairlist.py:147-201 criterion in C; method "n2" is the reference's own
    O(n_c^2) loop, "cols" the O(N) candidate-column variant (same result)."""
    threads = threads or default_threads()
    L = np.ascontiguousarray(lengths, dtype=np.float64)
    nc = grid["n_clusters"]
    bb = np.ascontiguousarray(grid["bboxes"].reshape(nc, 6), dtype=np.float64)
    counts = np.zeros(nc, dtype=np.int64)
    if method == "n2":
        lib().orc_search_n2(nc, _p(bb), _p(L), r_list, _p(counts), None, None, threads)
    else:
        cells = grid["cells"]
        col_first = np.searchsorted(grid["cell_of_cluster"], np.arange(cells * cells + 1)).astype(np.int64)
        coc = np.ascontiguousarray(grid["cell_of_cluster"], dtype=np.int64)
        lib().orc_search_cols(nc, _p(bb), _p(coc), _p(col_first), cells, _p(L), r_list, _p(counts),
                              None, None, threads)
    offsets = np.zeros(nc + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    j_idx = np.empty(int(offsets[-1]), dtype=np.int64)
    if method == "n2":
        lib().orc_search_n2(nc, _p(bb), _p(L), r_list, None, _p(j_idx), _p(offsets), threads)
    else:
        lib().orc_search_cols(nc, _p(bb), _p(coc), _p(col_first), cells, _p(L), r_list, None,
                              _p(j_idx), _p(offsets), threads)
    return search.list_from_csr(grid, offsets, j_idx, r_list)


def prune_list(lst: dict, clustered_positions, lengths, threads: int | None = None) -> dict:
    """pairlist.py:242-282 with the row distance in C (einsum order)."""
    threads = threads or default_threads()
    n_rows = lst["j_idx"].shape[0]
    if n_rows == 0:
        return lst
    nc = lst["offsets"].shape[0] - 1
    bits = np.ascontiguousarray(search.pack_masks(lst["masks"]))
    pos = np.ascontiguousarray(clustered_positions, dtype=np.float64)
    L = np.ascontiguousarray(lengths, dtype=np.float64)
    d2 = np.empty(n_rows)
    lib().orc_row_min_d2(nc, lst["m"], _p(lst["offsets"]), _p(np.ascontiguousarray(lst["j_idx"])),
                         _p(bits), _p(pos), _p(L), _p(d2), threads)
    ci = search.row_ci(lst)
    keep = (d2 <= lst["r_list"] * lst["r_list"]) | (ci == lst["j_idx"])
    counts = np.bincount(ci[keep], minlength=nc).astype(np.int64)
    offsets = np.zeros(nc + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return dict(m=lst["m"], offsets=offsets, j_idx=lst["j_idx"][keep], masks=lst["masks"][keep],
                r_list=lst["r_list"])


def count_within(lst: dict, clustered_positions, lengths, r_cut: float, threads: int | None = None) -> int:
    threads = threads or default_threads()
    nc = lst["offsets"].shape[0] - 1
    bits = np.ascontiguousarray(search.pack_masks(lst["masks"]))
    pos = np.ascontiguousarray(clustered_positions, dtype=np.float64)
    L = np.ascontiguousarray(lengths, dtype=np.float64)
    return int(lib().orc_count_within(nc, lst["m"], _p(lst["offsets"]),
                                      _p(np.ascontiguousarray(lst["j_idx"])), _p(bits), _p(pos),
                                      _p(L), r_cut, threads))


def type_tables(phys: Physics):
    """kernels.py:315-325."""
    eps = np.ascontiguousarray(phys.lj_table[:, :, 0])
    sig = np.ascontiguousarray(phys.lj_table[:, :, 1])
    if phys.shift_potential:
        rc2 = phys.r_cut * phys.r_cut
        src2 = (sig * sig) / rc2
        src6 = src2 * src2 * src2
        shift = 4.0 * eps * (src6 * src6 - src6)
    else:
        shift = np.zeros_like(eps)
    return eps, sig, np.ascontiguousarray(shift)


def list_forces(lst: dict, grid: dict, positions, charges, lj_type, lengths, phys: Physics,
                threads: int | None = None, packed_masks=None):
    """kernels.py:328-396 (gather by perm + _kernel_blocks) in C, FP64.
    Returns (f_clustered (n_slots,3), e_lj, e_coul)."""
    threads = threads or default_threads()
    perm = grid["perm"]
    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64)[perm])
    q = np.ascontiguousarray(np.asarray(charges, dtype=np.float64)[perm])
    t = np.ascontiguousarray(np.asarray(lj_type, dtype=np.int64)[perm])
    nc = lst["offsets"].shape[0] - 1
    bits = packed_masks if packed_masks is not None else np.ascontiguousarray(search.pack_masks(lst["masks"]))
    eps, sig, shift = type_tables(phys)
    L = np.ascontiguousarray(lengths, dtype=np.float64)
    f = np.zeros((perm.shape[0], 3))
    e = np.zeros(2)
    bad = np.full(2, -1, dtype=np.int64)
    st = lib().orc_force(nc, lst["m"], _p(lst["offsets"]), _p(np.ascontiguousarray(lst["j_idx"])),
                         _p(bits), _p(pos), _p(q), _p(t), eps.shape[0], _p(eps), _p(sig), _p(shift),
                         _ELEC[phys.elec], int(phys.shift_potential), phys.coulomb_scale, phys.r_cut,
                         phys.k_rf(), phys.c_rf(), phys.ewald_beta, _p(L), threads, _p(f), _p(e), _p(bad))
    if st == 2:
        raise ZeroDivisionError(f"singular pair: original {int(perm[bad[0]])} {int(perm[bad[1]])}")
    return f, float(e[0]), float(e[1])
