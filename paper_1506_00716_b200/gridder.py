"""Gridding into fixed-size clusters -- drop-in for clustermd.gridder.

Mirrors /root/reference/pkg/src/clustermd/gridder.py: same names, argument
meaning and errors.  The grid itself is built and kept on the GPU
(``nbx_grid_build``, csrc/grid.cu); the numpy fields of ``ClusterGrid`` are
materialised from the device on first access and are bit-identical to the
reference's.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .model import ParameterError, ParticleSystem, SimBox

VALID_CLUSTER_SIZES = (1, 2, 4, 8)


class DeviceArray:
    """A library-owned device buffer (pointer + shape) kept alive by `owner`."""

    def __init__(self, ptr: ctypes.c_void_p, shape: tuple, owner):
        self.ptr = ptr
        self.shape = shape
        self.owner = owner


class _CudaView:
    """__cuda_array_interface__ over a library-owned FP64 device buffer."""

    def __init__(self, ptr: int, shape: tuple):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _ro(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


class ClusterGrid:
    """Device-resident clustered layout (gridder.py:23-66).

    Fields (numpy, read-only, materialised lazily): perm, inverse_perm,
    fill_mask, cell_of_cluster, clustered_positions, bboxes; plus m,
    n_clusters, cell_counts, n_slots, n, cluster_centers().
    """

    def __init__(self, handle: ctypes.c_void_p, box_lengths: np.ndarray):
        self._h = handle
        info = np.zeros(5, dtype=np.int64)
        _lib.check(_lib.load().nbx_grid_info(handle, _lib.ptr(info)), "grid_info")
        self._n, self.m, cells, self.n_clusters, _ = (int(v) for v in info)
        self.cell_counts = (cells, cells)
        self.box_lengths = np.array(box_lengths, dtype=np.float64)
        self._host = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.nbx_grid_free(h)
            self._h = None

    # -- sizes
    @property
    def n_slots(self) -> int:
        return self.n_clusters * self.m

    @property
    def n(self) -> int:
        return self._n

    # -- device views
    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def clustered_positions_device_ptr(self) -> ctypes.c_void_p:
        return ctypes.c_void_p(_lib.load().nbx_grid_clustered_positions(self._h))

    @property
    def clustered_positions_device(self) -> DeviceArray:
        """The build-time clustered positions without leaving the device."""
        return DeviceArray(self.clustered_positions_device_ptr(), (self.n_slots, 3), self)

    # -- host materialisation (per field: a caller that reads one field --
    # e.g. clustered_positions to hand it back to prune_pair_list -- does not
    # pay for the downloads of the others)
    _FIELDS = ("perm", "inverse_perm", "fill_mask", "cell_of_cluster", "clustered_positions", "bboxes")

    def _field(self, name: str) -> np.ndarray:
        if self._host is None:
            self._host = {}
        if name not in self._host:
            ns, nc, n = self.n_slots, self.n_clusters, self.n
            shapes = dict(perm=((ns,), np.int64), inverse_perm=((n,), np.int64), fill_mask=((ns,), np.uint8),
                          cell_of_cluster=((nc,), np.int64), clustered_positions=((ns, 3), np.float64),
                          bboxes=((nc, 2, 3), np.float64))
            shape, dt = shapes[name]
            if name == "clustered_positions":
                # the largest field, read back by every drop-in rebuild: one
                # D2H into pinned staging (a pageable cudaMemcpy runs at a
                # fraction of the link), then one host copy
                cpos = torch.as_tensor(_CudaView(self.clustered_positions_device_ptr().value, shape),
                                       device=dev.require_cuda())
                self._host[name] = _ro(dev.stage_out(cpos, "grid_clustered_positions"))
                return self._host[name]
            buf = np.empty(shape, dtype=dt)
            args = [None] * 6
            args[self._FIELDS.index(name)] = buf
            torch.cuda.synchronize()
            _lib.check(_lib.load().nbx_grid_download(self._h, *(_lib.ptr(a) for a in args), dev.stream()),
                       "grid_download")
            if name == "fill_mask":
                buf = buf.astype(bool)
            self._host[name] = _ro(buf)
        return self._host[name]

    def _materialise(self) -> dict:
        for name in self._FIELDS:
            self._field(name)
        return self._host

    perm = property(lambda self: self._field("perm"))
    inverse_perm = property(lambda self: self._field("inverse_perm"))
    fill_mask = property(lambda self: self._field("fill_mask"))
    cell_of_cluster = property(lambda self: self._field("cell_of_cluster"))
    clustered_positions = property(lambda self: self._field("clustered_positions"))
    bboxes = property(lambda self: self._field("bboxes"))

    def cluster_centers(self) -> np.ndarray:
        """Bounding-box midpoints (gridder.py:64-66)."""
        return 0.5 * (self.bboxes[:, 0] + self.bboxes[:, 1])


def grid_cells(n: int, m: int, target_occupancy=None) -> int:
    """gridder.py:82-91."""
    occ = 2.0 * m if target_occupancy is None else target_occupancy
    return max(1, int(round(math.sqrt(n / occ))))


def build_cluster_grid(system: ParticleSystem, m: int, target_occupancy: float | None = None,
                       positions=None) -> ClusterGrid:
    """Grid in x/y, order columns by z, pack into m-clusters (gridder.py:69-146).

    ``positions`` optionally overrides system.positions with a CUDA tensor
    (device-resident callers avoid the host->device copy)."""
    if m not in VALID_CLUSTER_SIZES:
        raise ParameterError(f"cluster size m must be one of {VALID_CLUSTER_SIZES}, got {m}")
    if target_occupancy is None:
        target_occupancy = 2.0 * m
    if target_occupancy <= 0:
        raise ParameterError(f"target occupancy must be positive, got {target_occupancy}")
    n = system.n
    cells = grid_cells(n, m, target_occupancy)
    src = system.positions if positions is None else positions
    if dev.is_device_tensor(src):
        pos = dev.to_device(src, torch.float64, (n, 3))
    else:  # host arrays through the pinned staging of the drop-in API
        pos = dev.stage_in(np.asarray(src, dtype=np.float64).reshape(n, 3), torch.float64, "grid_positions")
    box = _lib.box3(system.box.lengths)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().nbx_grid_build(_lib.ptr(pos), n, _lib.ptr(box), m, cells, dev.stream(),
                                          ctypes.byref(h)), "grid_build")
    return ClusterGrid(h, system.box.lengths)


def scatter_to_original(grid: ClusterGrid, clustered_values):
    """Per-slot array back to particle order, fillers dropped (gridder.py:149-162).

    CUDA tensors stay on the device (nbx_scatter_to_original); host arrays
    are indexed on the host."""
    if dev.is_device_tensor(clustered_values):
        v = clustered_values
        if v.shape[0] != grid.n_slots:
            raise ParameterError(f"expected leading axis {grid.n_slots}, got {v.shape[0]}")
        k = int(np.prod(v.shape[1:])) if v.dim() > 1 else 1
        vin = v.to(torch.float64).contiguous().reshape(grid.n_slots, k)
        out = torch.empty((grid.n, k), dtype=torch.float64, device=v.device)
        _lib.check(_lib.load().nbx_scatter_to_original(grid.handle, _lib.ptr(vin), k, _lib.ptr(out),
                                                       dev.stream()), "scatter")
        return out.reshape((grid.n,) + tuple(v.shape[1:])).to(v.dtype)
    values = np.asarray(clustered_values)
    if values.shape[0] != grid.n_slots:
        raise ParameterError(f"expected leading axis {grid.n_slots}, got {values.shape[0]}")
    out = np.zeros((grid.n,) + values.shape[1:], dtype=values.dtype)
    real = ~grid.fill_mask
    out[grid.perm[real]] = values[real]
    return out


def bbox_gap_sq(lo_i, hi_i, lo_j, hi_j, lengths) -> np.ndarray:
    """Periodic AABB gap^2 (gridder.py:165-185); the GPU search evaluates the
    same expression in csrc/common.cuh (gap_sq)."""
    lo_j = np.asarray(lo_j, dtype=np.float64)
    hi_j = np.asarray(hi_j, dtype=np.float64)
    out = np.zeros(lo_j.shape[:-1], dtype=np.float64)
    for d in range(3):
        L = lengths[d]
        a = lo_j[..., d] - hi_i[d]
        b = lo_i[d] - hi_j[..., d]
        g = np.minimum(np.maximum(0.0, np.maximum(a, b)),
                       np.minimum(np.maximum(0.0, np.maximum(a - L, b + L)),
                                  np.maximum(0.0, np.maximum(a + L, b - L))))
        out = out + g * g
    return out


def cluster_min_distance(grid: ClusterGrid, i: int, j: int, box: SimBox) -> float:
    """Conservative AABB distance between clusters i and j (gridder.py:188-196)."""
    if not (0 <= i < grid.n_clusters and 0 <= j < grid.n_clusters):
        raise ParameterError(f"cluster indices ({i}, {j}) out of range [0, {grid.n_clusters})")
    lo_i, hi_i = grid.bboxes[i]
    lo_j, hi_j = grid.bboxes[j]
    return float(np.sqrt(bbox_gap_sq(lo_i, hi_i, lo_j, hi_j, box.lengths)))
