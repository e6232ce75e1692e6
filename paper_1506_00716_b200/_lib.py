"""ctypes binding of the C ABI in include/nbx.h (libnbx.so, sm_100a).

The product path has no CPU fallback: if libnbx.so is missing or no CUDA
device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .model import ParameterError, SingularityError

# NBX_LIB: an alternative build of the same library (A/B kernel variants,
# tools/build_variant.sh); default the in-tree libnbx.so
LIB_PATH = Path(os.environ.get("NBX_LIB") or (Path(__file__).resolve().parent / "libnbx.so"))

NBX_OK, NBX_ERR_PARAM, NBX_ERR_SINGULAR, NBX_ERR_CUDA = 0, 1, 2, 3
ELEC = {"cutoff": 0, "reaction_field": 1, "ewald": 2}
FORCE_ENERGY, FORCE_ACCUMULATE, FORCE_CLUSTERED, FORCE_CANONICAL, FORCE_REPRUNE = 1, 2, 4, 8, 16

# every symbol include/nbx.h declares (tests check the exports)
EXPORTS = (
    "nbx_version", "nbx_last_error", "nbx_grid_build", "nbx_grid_info", "nbx_grid_download",
    "nbx_grid_clustered_positions", "nbx_scatter_to_original", "nbx_grid_free",
    "nbx_pairlist_build", "nbx_pairlist_prune", "nbx_list_info", "nbx_list_rows", "nbx_list_entries", "nbx_list_download",
    "nbx_super_layout", "nbx_super_download", "nbx_count_within", "nbx_list_free",
    "nbx_force", "nbx_find_singular", "nbx_launch_count", "nbx_timing_enable", "nbx_timing_query",
    "nbx_max_displacement", "nbx_max_displacement_ex", "nbx_vv_update", "nbx_pairlist_build_ex",
    "nbx_dd_unique_id", "nbx_dd_create", "nbx_dd_set_layout", "nbx_dd_exchange_positions",
    "nbx_dd_reduce_forces", "nbx_dd_allreduce_sum", "nbx_dd_free", "nbx_pairlist_build_pruned",
    "nbx_dd_assign", "nbx_dd_assign_local", "nbx_dd_classify", "nbx_dd_allgather_home", "nbx_dd_p2p_alloc", "nbx_dd_p2p_open", "nbx_dd_p2p_error", "nbx_dd_p2p_error_seen",
    "nbx_pairlist_prune_inner", "nbx_list_force_pairs", "nbx_list_diagnostics", "nbx_list_exclude", "nbx_settle", "nbx_vv_constrained", "nbx_dd_force", "nbx_dd_force_seq", "nbx_list_step",
)


class NbxParams(ctypes.Structure):
    _fields_ = [
        ("n_types", ctypes.c_int32),
        ("lj_table", ctypes.c_void_p),
        ("coulomb_scale", ctypes.c_double),
        ("r_cut", ctypes.c_double),
        ("shift_potential", ctypes.c_int32),
        ("elec", ctypes.c_int32),
        ("k_rf", ctypes.c_double),
        ("c_rf", ctypes.c_double),
        ("ewald_beta", ctypes.c_double),
    ]


_lib = None


def load():
    """Load libnbx.so (raises loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the nbnxn path)"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "nbx_version": (ctypes.c_int, []),
        "nbx_last_error": (ctypes.c_char_p, []),
        "nbx_grid_build": (ctypes.c_int, [P, I64, P, I32, I64, P, PP]),
        "nbx_grid_info": (ctypes.c_int, [P, P]),
        "nbx_grid_download": (ctypes.c_int, [P, P, P, P, P, P, P, P]),
        "nbx_grid_clustered_positions": (P, [P]),
        "nbx_scatter_to_original": (ctypes.c_int, [P, P, I32, P, P]),
        "nbx_grid_free": (None, [P]),
        "nbx_pairlist_build": (ctypes.c_int, [P, P, D, P, PP]),
        "nbx_pairlist_build_ex": (ctypes.c_int, [P, P, D, P, P, PP]),
        "nbx_pairlist_build_pruned": (ctypes.c_int, [P, P, D, P, P, P, PP]),
        "nbx_pairlist_prune": (ctypes.c_int, [P, P, P, P, P, PP]),
        "nbx_pairlist_prune_inner": (ctypes.c_int, [P, P, P, P, ctypes.c_double, P, PP]),
        "nbx_list_force_pairs": (ctypes.c_int, [P, ctypes.c_int32, P, P]),
        "nbx_list_info": (ctypes.c_int, [P, P]),
        "nbx_list_rows": (ctypes.c_int, [P, P, P]),
        "nbx_list_entries": (ctypes.c_int, [P, P, P]),
        "nbx_list_download": (ctypes.c_int, [P, P, P, P, P]),
        "nbx_super_layout": (ctypes.c_int, [P, I32, P, P]),
        "nbx_super_download": (ctypes.c_int, [P, P, P, P, P]),
        "nbx_count_within": (ctypes.c_int, [P, P, P, D, P, P]),
        "nbx_list_free": (None, [P]),
        "nbx_force": (ctypes.c_int, [P, P, P, P, P, ctypes.POINTER(NbxParams), P, P, I64, I32, P, P, P, P]),
        "nbx_find_singular": (ctypes.c_int, [P, P, P, D, P, P, P]),
        "nbx_launch_count": (ctypes.c_int64, []),
        "nbx_timing_enable": (None, [I32]),
        "nbx_timing_query": (ctypes.c_int, [P, P]),
        "nbx_max_displacement": (ctypes.c_int, [P, P, I64, P, P, P]),
        "nbx_max_displacement_ex": (ctypes.c_int, [P, P, I64, P, P, P, ctypes.c_int32, P]),
        "nbx_vv_update": (ctypes.c_int, [P, P, P, P, I64, D, I32, P, P]),
        "nbx_dd_unique_id": (ctypes.c_int, [P]),
        "nbx_dd_create": (ctypes.c_int, [P, I32, I32, PP]),
        "nbx_dd_set_layout": (ctypes.c_int, [P, P, I64, I64, I64, P]),
        "nbx_dd_exchange_positions": (ctypes.c_int, [P, P, P]),
        "nbx_dd_reduce_forces": (ctypes.c_int, [P, P, P]),
        "nbx_dd_allreduce_sum": (ctypes.c_int, [P, P, I64, P]),
        "nbx_dd_free": (None, [P]),
        "nbx_dd_assign": (ctypes.c_int, [P, P, I64, D, P, D, P, P, P, P, P]),
        "nbx_dd_classify": (ctypes.c_int, [P, I64, D, P, ctypes.c_int32, D, P, P, P]),
        "nbx_dd_assign_local": (ctypes.c_int, [P, P, P, P, I64, D, P, D, P, P, P, P, P, P, P, P, P]),
        "nbx_dd_allgather_home": (ctypes.c_int, [P, P, P, I64, I64, P, P]),
        "nbx_dd_p2p_alloc": (ctypes.c_int, [P, I64, P]),
        "nbx_dd_p2p_open": (ctypes.c_int, [P, P, P]),
        "nbx_dd_p2p_error": (ctypes.c_int, [P, P]),
        "nbx_dd_p2p_error_seen": (ctypes.c_int, [P, P]),
        "nbx_list_diagnostics": (ctypes.c_int, [P, P, P, P, P, P, P]),
        "nbx_list_exclude": (ctypes.c_int, [P, P, P, P, P, P, P]),
        "nbx_list_step": (ctypes.c_int, [P, ctypes.c_int64, P, ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                         ctypes.c_double, P, P, P, P, ctypes.c_int32, P, PP, PP]),
        "nbx_settle": (ctypes.c_int, [P, P, P, I64, D, D, D, D, D, I32, P, P]),
        "nbx_vv_constrained": (ctypes.c_int, [P, P, P, P, I64, D, D, D, D, D, ctypes.c_int32, P, P]),
        "nbx_dd_force": (ctypes.c_int, [P, P, P, P, P, P, ctypes.POINTER(NbxParams), P, I32, P, P, P, P]),
        "nbx_dd_force_seq": (ctypes.c_int, [P, P, P, P, P, P, ctypes.POINTER(NbxParams), P, I32, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == NBX_OK:
        return
    msg = load().nbx_last_error().decode(errors="replace")
    if status == NBX_ERR_PARAM:
        raise ParameterError(msg)
    if status == NBX_ERR_SINGULAR:
        raise SingularityError(msg)
    raise RuntimeError(f"nbx CUDA failure in {what}: {msg}")


def ptr(a) -> ctypes.c_void_p:
    """Raw pointer of a torch tensor or numpy array (None -> NULL)."""
    if a is None:
        return ctypes.c_void_p(0)
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


def box3(lengths) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(lengths, dtype=np.float64).reshape(3))
