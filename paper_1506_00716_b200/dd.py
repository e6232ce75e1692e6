"""Spatial domain decomposition of the non-bonded pass over several GPUs.

One rank per GPU; the box is cut into N slabs along x (the reference's
SlabPartition concept, engine.py:141-263, reused as the rank decomposition).
Each rank owns the particles of its slab ("home") and receives, from its +x
neighbour only, the particles within r_comm = r_list of the shared face
("halo"): a 1-D half shell.  Every particle pair is then evaluated exactly
once:

  * home-home pairs by their owner;
  * home(r)-halo pairs (they straddle the face between r and r+1) by r;
  * halo-halo pairs never (masked out of r's list: nbx_pairlist_build_ex),
    they are home-home pairs of r+1.

Per force pass the communication is two NCCL point-to-point exchanges with
the neighbours (no collective on the data path):

  1. coordinates of the particles within r_comm of the -x face go to rank
     r-1, the halo coordinates come from rank r+1;
  2. after the local pass, the forces on halo particles go back to rank r+1,
     and rank r adds the forces rank r-1 computed on its face particles.

Energies are summed with one all-reduce of two doubles on energy steps.  At
list rebuilds the home sets are re-derived from an all-gather of all home
positions (SURVEY.md 8e "all-gather every nstlist"), so particles migrate
between slabs only at rebuilds, exactly when the lists are rebuilt; the half
shell stays complete in between because r_comm = r_list covers the Verlet
buffer.  Requirements (checked): every slab is at least r_comm wide, and a
domain's x extent w_slab + r_comm stays below L_x - r_comm, so no pair inside
one domain is seen through a periodic image that another rank also owns.

The class is backend-agnostic (torch.distributed with NCCL on GPUs, gloo on
CPU in the tests); the local force evaluation is injected (the GPU pass in
production, the oracle in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .model import ParameterError


def _wrap_np(x, L):
    out = np.mod(x, L)
    return np.where(out >= L, out - L, out)


@dataclass
class DomainLayout:
    """Particle sets of one rank after a rebuild (global ids ascending), as
    tensors on the device of the positions they were derived from."""

    home: torch.Tensor        # global ids owned here
    halo: torch.Tensor        # global ids received from the +x neighbour
    send: torch.Tensor | None  # global ids (subset of home) sent to the -x neighbour (None: native fast path)
    send_local: torch.Tensor  # their indices in the local array [home; halo]

    @property
    def n_home(self) -> int:
        return int(self.home.shape[0])

    @property
    def n_local(self) -> int:
        return int(self.home.shape[0] + self.halo.shape[0])

    @property
    def local_ids(self) -> torch.Tensor:
        return torch.cat([self.home, self.halo])


class SlabDecomposition:
    """Slab geometry + halo bookkeeping + neighbour exchanges for one rank."""

    def __init__(self, box_lengths, n_ranks: int, rank: int, r_comm: float, boundaries=None, group=None):
        self.L = np.asarray(box_lengths, dtype=np.float64)
        self.N = int(n_ranks)
        self.rank = int(rank)
        self.r_comm = float(r_comm)
        self.group = group
        Lx = float(self.L[0])
        if boundaries is None:
            boundaries = np.linspace(0.0, Lx, self.N + 1)
            boundaries[-1] = Lx
        self.boundaries = np.asarray(boundaries, dtype=np.float64)
        if self.boundaries.shape != (self.N + 1,):
            raise ParameterError("boundaries must have n_ranks + 1 entries")
        widths = np.diff(self.boundaries)
        if self.N > 1:
            if np.any(widths < self.r_comm):
                raise ParameterError(f"every slab must be >= r_comm={self.r_comm} wide (single-neighbour halo), "
                                     f"got widths {widths}")
            if Lx <= widths.max() + 2.0 * self.r_comm:
                raise ParameterError(f"box length {Lx} too short for {self.N} slabs with r_comm={self.r_comm}")
        self.layout: DomainLayout | None = None
        self._native = None

    def enable_native(self) -> None:
        """Move the per-step exchanges into libnbx (NCCL on the compute stream).
        Collective: every rank must call it.  Needs an initialised
        torch.distributed group for the one-time id broadcast."""
        if self.N == 1 or self._native is not None:
            return
        import ctypes

        import torch.distributed as dist

        from . import _lib

        lib = _lib.load()
        uid = np.zeros(128, dtype=np.uint8)
        if self.rank == 0:
            _lib.check(lib.nbx_dd_unique_id(_lib.ptr(uid)), "dd_unique_id")
        obj = [uid.tobytes()]
        dist.broadcast_object_list(obj, src=0, group=self.group)
        uid = np.frombuffer(obj[0], dtype=np.uint8).copy()
        h = ctypes.c_void_p()
        _lib.check(lib.nbx_dd_create(_lib.ptr(uid), self.N, self.rank, ctypes.byref(h)), "dd_create")
        self._native = h

    def enable_p2p(self, capacity: int) -> bool:
        """Switch the per-step exchanges to NVLink peer stores (libnbx
        ``nbx_dd_p2p_*``): each rank exports a CUDA IPC region for up to
        ``capacity`` halo / face particles (the global particle count is
        always enough), the handles are all-gathered once, and rank-1 /
        rank+1 map each other's regions.  Collective; needs enable_native().
        Returns False (NCCL path kept) when NBX_DD_P2P=0 or there is one rank."""
        import os

        if self.N == 1 or self._native is None or os.environ.get("NBX_DD_P2P", "1") == "0":
            return False
        import torch.distributed as dist

        from . import _lib

        lib = _lib.load()
        h = np.zeros(64, dtype=np.uint8)
        _lib.check(lib.nbx_dd_p2p_alloc(self._native, int(capacity), _lib.ptr(h)), "dd_p2p_alloc")
        allh = [None] * self.N
        dist.all_gather_object(allh, h.tobytes(), group=self.group)
        down = np.frombuffer(allh[(self.rank - 1) % self.N], dtype=np.uint8).copy()
        up = np.frombuffer(allh[(self.rank + 1) % self.N], dtype=np.uint8).copy()
        st = lib.nbx_dd_p2p_open(self._native, _lib.ptr(down), _lib.ptr(up))
        # every rank must take the same path: fall back together if any failed
        ok = torch.tensor([1 if st == _lib.NBX_OK else 0], device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if int(ok.item()) == 0:
            lib.nbx_dd_p2p_open(self._native, None, None)
            self.p2p = False
            return False
        self.p2p = True
        return True

    def check_p2p(self) -> None:
        """Raise when a peer wait timed out since the exchanges started (the
        halo rows or the returned face forces of some step were then stale).
        Called where the host synchronises anyway: every list rebuild
        (DomainForces.rebuild) and the end of a run (bench.py)."""
        if self.p2p_error():
            raise RuntimeError(f"rank {self.rank}: NVLink peer exchange timed out (a neighbour stalled for > 5 s); "
                               "forces since the last check are invalid")

    def p2p_error(self, seen: bool = False) -> bool:
        """True when a peer wait timed out (host sync).  ``seen``: the flag as
        read by the last native assign's own sync (no extra sync)."""
        if not getattr(self, "p2p", False):
            return False
        import ctypes

        from . import _lib

        out = ctypes.c_int32(0)
        fn = _lib.load().nbx_dd_p2p_error_seen if seen else _lib.load().nbx_dd_p2p_error
        _lib.check(fn(self._native, ctypes.byref(out)), "dd_p2p_error")
        return out.value != 0

    def close(self) -> None:
        """Free the native communicator (collective under NCCL; idempotent)."""
        h = getattr(self, "_native", None)
        self._native = None
        if h is None:
            return
        try:
            from . import _lib
        except ImportError:  # interpreter shutdown: module globals already gone
            return
        lib = getattr(_lib, "_lib", None)
        if lib is not None:
            lib.nbx_dd_free(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # never raise from a finaliser (interpreter exit)
            pass

    # ---------------------------------------------------------------- load balance
    def rebalance(self, times, alpha: float = 0.5) -> np.ndarray:
        """Move the slab boundaries toward equal force time per rank (the
        role of the reference's rebalance_slabs, engine.py:208-263, by a
        different rule).  Each slab's measured time is spread uniformly over
        its width, giving a piecewise-linear cumulative cost along x; the new
        boundaries are its N-quantiles (equal cost per slab), blended with
        the old ones by ``alpha`` (damping), then widened where needed so
        every slab keeps the single-neighbour halo (>= r_comm) and the
        periodic-image bound of the constructor.  ``times`` (one positive
        float per rank) must be identical on every rank (e.g. all-gathered),
        so every rank computes the same boundaries.  Returns them."""
        t = np.asarray(times, dtype=np.float64).reshape(-1)
        if t.shape != (self.N,):
            raise ParameterError(f"expected {self.N} per-rank times, got shape {t.shape}")
        if not np.all(np.isfinite(t)) or np.any(t <= 0.0):
            raise ParameterError("per-rank times must be positive and finite")
        if not 0.0 < alpha <= 1.0:
            raise ParameterError(f"alpha must be in (0, 1], got {alpha}")
        if self.N == 1:
            return self.boundaries
        b = self.boundaries
        cum = np.concatenate([[0.0], np.cumsum(t)])
        quant = np.interp(cum[-1] * np.arange(self.N + 1) / self.N, cum, b)
        new = alpha * quant + (1.0 - alpha) * b
        self.boundaries = self._clamped(new)
        return self.boundaries

    def _clamped(self, new) -> np.ndarray:
        """Boundaries ``new`` with every slab width in [r_comm, L - 2 r_comm]
        (excess / deficit redistributed over the free slabs)."""
        b = self.boundaries
        new = np.asarray(new, dtype=np.float64).copy()
        new[0], new[-1] = b[0], b[-1]
        Lx = float(self.L[0])
        w_max = Lx - 2.0 * self.r_comm - 1e-9 * Lx
        w = np.diff(new)
        for _ in range(2 * self.N):  # clamp to [r_comm, w_max], redistribute the excess / deficit
            lo, hi = w < self.r_comm, w > w_max
            if not (lo.any() or hi.any()):
                break
            w = np.clip(w, self.r_comm, w_max)
            free = ~(lo | hi)
            if free.any():
                w[free] += (Lx - w.sum()) * w[free] / w[free].sum()
        new = np.concatenate([[b[0]], b[0] + np.cumsum(w)])
        new[-1] = b[-1]
        return new

    def balance_counts(self, x) -> np.ndarray:
        """Boundaries with equal particle counts per slab for the x
        coordinates ``x`` (all particles; identical on every rank): the
        count quantiles of x, widths clamped as in ``rebalance``.  A one-time set-up for boxes whose density is not uniform
        along x (the generated water boxes fill their last lattice layers
        partially), with no per-rebuild cost."""
        if self.N == 1:
            return self.boundaries
        xs = np.sort(_wrap_np(np.asarray(x, dtype=np.float64).reshape(-1), self.L[0]))
        n = xs.shape[0]
        k = (np.arange(1, self.N) * n) // self.N
        new = self.boundaries.copy()
        new[1:-1] = 0.5 * (xs[np.maximum(k - 1, 0)] + xs[np.minimum(k, n - 1)])
        self.boundaries = self._clamped(new)
        return self.boundaries

    # ---------------------------------------------------------------- geometry
    def owner(self, x) -> np.ndarray:
        xw = _wrap_np(np.asarray(x, dtype=np.float64), self.L[0])
        return np.clip(np.searchsorted(self.boundaries[1:-1], xw, side="right"), 0, self.N - 1)

    def assign(self, positions_global) -> DomainLayout:
        """Home / halo / send sets from the global positions (identical on every
        rank).  Runs where the positions live (device tensors stay on the GPU)."""
        pos = positions_global if isinstance(positions_global, torch.Tensor) else \
            torch.as_tensor(np.asarray(positions_global, dtype=np.float64))
        pos = pos.reshape(-1, 3)
        dev = pos.device
        if self._native is not None and pos.is_cuda:
            return self._assign_native(pos.contiguous())
        Lx = float(self.L[0])
        x = torch.remainder(pos[:, 0], Lx)
        x = torch.where(x >= Lx, x - Lx, x)
        inner = torch.as_tensor(self.boundaries[1:-1], dtype=torch.float64, device=dev)
        own = torch.bucketize(x, inner, right=True).clamp_(0, self.N - 1)
        r = self.rank
        home = torch.nonzero(own == r).flatten()
        if self.N == 1:
            empty = torch.empty(0, dtype=torch.int64, device=dev)
            self.layout = DomainLayout(home=home, halo=empty, send=empty, send_local=empty)
            return self.layout
        b_lo = float(self.boundaries[r])
        sel = (x[home] - b_lo) < self.r_comm
        send = home[sel]
        send_local = torch.nonzero(sel).flatten()
        nb = (r + 1) % self.N
        nb_lo = float(self.boundaries[nb])
        halo = torch.nonzero((own == nb) & ((x - nb_lo) < self.r_comm)).flatten()
        self.layout = DomainLayout(home=home, halo=halo, send=send, send_local=send_local)
        if self._native is not None:
            from . import _device, _lib

            _lib.check(_lib.load().nbx_dd_set_layout(self._native, _lib.ptr(send_local), int(send_local.numel()),
                                                     int(home.numel()), int(halo.numel()), _device.stream()),
                       "dd_set_layout")
        return self.layout

    def assign_local(self, pos: torch.Tensor, charges: torch.Tensor, lj_type: torch.Tensor):
        """assign() plus the rank's local inputs in [home; halo] order, in one
        native call (nbx_dd_assign_local): returns (layout, local positions,
        charges, types, halo flags) -- the latter four views of buffers
        reused by the next call."""
        from . import _device, _lib

        n = pos.shape[0]
        dev = pos.device
        if getattr(self, "_lbuf_n", -1) != n:
            self._lbuf = dict(ids=torch.empty((3, max(n, 1)), dtype=torch.int64, device=dev),
                              pos=torch.empty((max(n, 1), 3), dtype=torch.float64, device=dev),
                              q=torch.empty(max(n, 1), dtype=torch.float64, device=dev),
                              t=torch.empty(max(n, 1), dtype=torch.int64, device=dev),
                              halo=torch.empty(max(n, 1), dtype=torch.uint8, device=dev))
            self._lbuf_n = n
        b = self._lbuf
        counts = np.zeros(3 + self.N, dtype=np.int64)
        bnd = np.ascontiguousarray(self.boundaries, dtype=np.float64)
        _lib.check(_lib.load().nbx_dd_assign_local(
            self._native, _lib.ptr(pos), _lib.ptr(charges), _lib.ptr(lj_type), n, float(self.L[0]), _lib.ptr(bnd),
            self.r_comm, _lib.ptr(b["ids"][0]), _lib.ptr(b["ids"][1]), _lib.ptr(b["ids"][2]), _lib.ptr(b["pos"]),
            _lib.ptr(b["q"]), _lib.ptr(b["t"]), _lib.ptr(b["halo"]), _lib.ptr(counts), _device.stream()),
            "dd_assign_local")
        if self.p2p_error(seen=True):  # read by the assign's own sync
            raise RuntimeError(f"rank {self.rank}: NVLink peer exchange timed out (a neighbour stalled for > 5 s); "
                               "forces since the last check are invalid")
        nh, nl, ns = (int(c) for c in counts[:3])
        self.home_counts = counts[3:].copy()
        # home ids outlive the buffers (callers keep them per step); halo and
        # send_local are views until the next list step, send is not formed
        # (the native exchanges use send_local)
        home = b["ids"][0, :nh].clone()
        self.layout = DomainLayout(home=home, halo=b["ids"][1, :nl], send=None, send_local=b["ids"][2, :ns])
        m = nh + nl
        return self.layout, b["pos"][:m], b["q"][:m], b["t"][:m], b["halo"][:m]

    def _assign_native(self, pos: torch.Tensor) -> DomainLayout:
        """assign() inside libnbx (flags + stable compaction, one host sync)."""
        from . import _device, _lib

        n = pos.shape[0]
        if getattr(self, "_abuf_n", -1) != n:
            self._abuf = torch.empty((3, max(n, 1)), dtype=torch.int64, device=pos.device)
            self._abuf_n = n
        counts = np.zeros(3 + self.N, dtype=np.int64)
        bnd = np.ascontiguousarray(self.boundaries, dtype=np.float64)
        _lib.check(_lib.load().nbx_dd_assign(self._native, _lib.ptr(pos), n, float(self.L[0]), _lib.ptr(bnd),
                                             self.r_comm, _lib.ptr(self._abuf[0]), _lib.ptr(self._abuf[1]),
                                             _lib.ptr(self._abuf[2]), _lib.ptr(counts), _device.stream()), "dd_assign")
        nh, nl, ns = (int(c) for c in counts[:3])
        self.home_counts = counts[3:].copy()
        home = self._abuf[0, :nh].clone()
        halo = self._abuf[1, :nl].clone()
        send_local = self._abuf[2, :ns].clone()
        self.layout = DomainLayout(home=home, halo=halo, send=home.index_select(0, send_local), send_local=send_local)
        _lib.check(_lib.load().nbx_dd_set_layout(self._native, _lib.ptr(send_local), ns, nh, nl, _device.stream()),
                   "dd_set_layout")
        return self.layout

    # ---------------------------------------------------------------- migration
    def _classify(self, pos: torch.Tensor):
        """(owner rank, face flag) of particles ``pos`` (n, 3) by assign()'s
        rule; face: within r_comm above the owner's lower boundary."""
        n = pos.shape[0]
        if pos.is_cuda:
            from . import _device, _lib

            own = torch.empty(n, dtype=torch.int32, device=pos.device)
            face = torch.empty(n, dtype=torch.uint8, device=pos.device)
            bnd = np.ascontiguousarray(self.boundaries, dtype=np.float64)
            _lib.check(_lib.load().nbx_dd_classify(_lib.ptr(pos.contiguous()), n, float(self.L[0]), _lib.ptr(bnd),
                                                   self.N, self.r_comm, _lib.ptr(own), _lib.ptr(face),
                                                   _device.stream()), "dd_classify")
            return own.long(), face.bool()
        Lx = float(self.L[0])
        x = torch.remainder(pos[:, 0], Lx)
        x = torch.where(x >= Lx, x - Lx, x)
        inner = torch.as_tensor(self.boundaries[1:-1], dtype=torch.float64, device=pos.device)
        own = torch.bucketize(x, inner, right=True).clamp_(0, self.N - 1)
        lo = torch.as_tensor(self.boundaries, dtype=torch.float64, device=pos.device)[own]
        return own, (x - lo) < self.r_comm

    def _exchange(self, sends: list, recv_from: list) -> list:
        """Variable-length neighbour exchange: ``sends`` = [(peer, rows
        (k, 4) float64)], ``recv_from`` = [peer] (same length, pairwise
        matched across ranks).  Counts first, then the rows; returns the
        received (k', 4) tensors in ``recv_from`` order."""
        import torch.distributed as dist

        dev = sends[0][1].device if sends else torch.device("cpu")
        cnt_out = [torch.tensor([t.shape[0]], dtype=torch.int64, device=dev) for _, t in sends]
        cnt_in = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in recv_from]
        ops = [dist.P2POp(dist.irecv, c, peer, group=self.group) for c, peer in zip(cnt_in, recv_from)]
        ops += [dist.P2POp(dist.isend, c, peer, group=self.group) for c, (peer, _) in zip(cnt_out, sends)]
        for q in dist.batch_isend_irecv(ops):
            q.wait()
        got = [torch.empty((int(c.item()), 4), dtype=torch.float64, device=dev) for c in cnt_in]
        ops = [dist.P2POp(dist.irecv, g, peer, group=self.group) for g, peer in zip(got, recv_from) if g.numel()]
        ops += [dist.P2POp(dist.isend, t.contiguous(), peer, group=self.group) for peer, t in sends if t.numel()]
        if ops:
            for q in dist.batch_isend_irecv(ops):
                q.wait()
        return got

    def migrate(self, home_ids: torch.Tensor, home_pos: torch.Tensor):
        """List-step bookkeeping from this rank's own particles only (the
        scalable replacement of allgather_home + assign): particles that left
        the slab go to the neighbour that now owns them, the new home set is
        sorted by global id, and the face particles travel down as the lower
        neighbour's halo.  The same layout as ``assign`` on the gathered
        positions, with two neighbour exchanges instead of an all-gather of
        every position and an O(N_total) scan on every rank.  Requires that
        no particle moved by more than one slab since the last list step
        (raises otherwise -- use assign).  Returns (layout, local positions
        (n_home + n_halo, 3): home rows then halo rows)."""
        N, r = self.N, self.rank
        ids = torch.as_tensor(home_ids, device=home_pos.device).reshape(-1).to(torch.int64)
        pos = home_pos.reshape(-1, 3)
        if N == 1:
            self.assign(pos)  # one slab: everything is home
            return self.layout, pos.contiguous()
        own, _ = self._classify(pos)
        up, down = (r + 1) % N, (r - 1) % N
        stay = own == r
        rec = torch.cat([ids.to(torch.float64)[:, None], pos], 1)  # ids < 2^53: exact in FP64
        if N == 2:
            leave = [(up, ~stay)]
            recv_from = [up]
        else:
            leave = [(up, own == up), (down, own == down)]
            recv_from = [down, up]
        far = ~stay
        for _, m in leave:
            far &= ~m
        if bool(far.any()):
            raise RuntimeError("migrate: a particle moved by more than one slab since the last list step; "
                               "use assign on the gathered positions")
        got = self._exchange([(peer, rec[m]) for peer, m in leave], recv_from)
        allrec = torch.cat([rec[stay]] + got, 0)
        order = torch.argsort(allrec[:, 0])
        allrec = allrec[order]
        home = allrec[:, 0].to(torch.int64)
        hpos = allrec[:, 1:].contiguous()
        own2, face = self._classify(hpos)
        send_local = torch.nonzero(face).flatten()
        halo_rec = self._exchange([(down, allrec[send_local])], [up])[0]
        halo = halo_rec[:, 0].to(torch.int64)
        self.layout = DomainLayout(home=home, halo=halo, send=home[send_local], send_local=send_local)
        self.home_counts = None  # per-rank counts are no longer known here (allgather_home recounts)
        if self._native is not None:
            from . import _device, _lib

            _lib.check(_lib.load().nbx_dd_set_layout(self._native, _lib.ptr(send_local), int(send_local.numel()),
                                                     int(home.numel()), int(halo.numel()), _device.stream()),
                       "dd_set_layout")
        return self.layout, torch.cat([hpos, halo_rec[:, 1:]], 0)

    # ---------------------------------------------------------------- exchanges
    def _p2p(self, send_t: torch.Tensor | None, send_to: int, recv_t: torch.Tensor | None, recv_from: int):
        """One grouped send + receive (ncclGroupStart/End under NCCL): both
        directions progress together, so neighbour pairs cannot deadlock."""
        import torch.distributed as dist

        ops = []
        if recv_t is not None and recv_t.numel():
            ops.append(dist.P2POp(dist.irecv, recv_t, recv_from, group=self.group))
        if send_t is not None and send_t.numel():
            ops.append(dist.P2POp(dist.isend, send_t.contiguous(), send_to, group=self.group))
        if ops:
            for q in dist.batch_isend_irecv(ops):
                q.wait()

    def exchange_positions(self, local_pos: torch.Tensor) -> None:
        """local_pos[:n_home] holds current home positions; fills the halo rows."""
        lay = self.layout
        if self.N == 1 or lay is None:
            return
        if self._native is not None:
            from . import _device, _lib

            _lib.check(_lib.load().nbx_dd_exchange_positions(self._native, _lib.ptr(local_pos), _device.stream()),
                       "dd_exchange")
            return
        send_t = local_pos.index_select(0, lay.send_local)
        recv_t = local_pos[lay.n_home:]
        buf = torch.empty_like(recv_t)
        self._p2p(send_t, (self.rank - 1) % self.N, buf, (self.rank + 1) % self.N)
        recv_t.copy_(buf)

    def reduce_halo_forces(self, local_f: torch.Tensor) -> torch.Tensor:
        """Send halo forces to their owner (+x), add the forces the -x
        neighbour computed on our face particles.  Returns home forces."""
        lay = self.layout
        home_f = local_f[:lay.n_home]
        if self.N == 1:
            return home_f
        if self._native is not None:
            from . import _device, _lib

            _lib.check(_lib.load().nbx_dd_reduce_forces(self._native, _lib.ptr(local_f), _device.stream()),
                       "dd_reduce")
            return home_f
        recv = torch.empty((lay.send.shape[0], 3), dtype=local_f.dtype, device=local_f.device)
        self._p2p(local_f[lay.n_home:], (self.rank + 1) % self.N, recv, (self.rank - 1) % self.N)
        home_f.index_add_(0, lay.send_local, recv)
        return home_f

    def allreduce_energies(self, e: torch.Tensor) -> torch.Tensor:
        if self.N == 1:
            return e
        if self._native is not None and e.is_cuda:
            from . import _device, _lib

            _lib.check(_lib.load().nbx_dd_allreduce_sum(self._native, _lib.ptr(e), int(e.numel()), _device.stream()),
                       "dd_allreduce")
            return e
        import torch.distributed as dist

        dist.all_reduce(e, group=self.group)
        return e

    def allgather_home(self, ids: torch.Tensor, pos: torch.Tensor, n_total: int) -> torch.Tensor:
        """Global (n_total, 3) positions from every rank's home rows."""
        ids = torch.as_tensor(ids, device=pos.device)
        if self._native is not None and pos.is_cuda and getattr(self, "home_counts", None) is not None:
            from . import _device, _lib

            cap = int(self.home_counts.max())
            out = torch.empty((n_total, 3), dtype=torch.float64, device=pos.device)
            _lib.check(_lib.load().nbx_dd_allgather_home(self._native, _lib.ptr(ids.contiguous()),
                                                         _lib.ptr(pos.contiguous()), int(ids.shape[0]), cap,
                                                         _lib.ptr(out), _device.stream()), "dd_allgather")
            return out
        if self.N == 1:
            out = torch.empty((n_total, 3), dtype=pos.dtype, device=pos.device)
            out[ids] = pos
            return out
        import torch.distributed as dist

        dev = pos.device
        nccl = dist.get_backend(self.group) == "nccl"
        cnt = torch.tensor([ids.shape[0]], dtype=torch.int64, device=dev)
        if nccl:
            counts = torch.empty(self.N, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(counts, cnt, group=self.group)
        else:
            parts = [torch.zeros_like(cnt) for _ in range(self.N)]
            dist.all_gather(parts, cnt, group=self.group)
            counts = torch.cat(parts)
        cmax = int(counts.max().item())  # one host sync
        pad_ids = torch.full((cmax,), -1, dtype=torch.int64, device=dev)
        pad_ids[:ids.shape[0]] = ids
        pad_pos = torch.zeros((cmax, 3), dtype=pos.dtype, device=dev)
        pad_pos[:ids.shape[0]] = pos
        all_ids = torch.empty((self.N, cmax), dtype=torch.int64, device=dev)
        all_pos = torch.empty((self.N, cmax, 3), dtype=pos.dtype, device=dev)
        if nccl:
            dist.all_gather_into_tensor(all_ids, pad_ids, group=self.group)
            dist.all_gather_into_tensor(all_pos, pad_pos, group=self.group)
        else:
            dist.all_gather(list(all_ids.unbind(0)), pad_ids, group=self.group)
            dist.all_gather(list(all_pos.unbind(0)), pad_pos, group=self.group)
        ids_cat = all_ids.reshape(-1)
        pos_cat = all_pos.reshape(-1, 3)
        keep = ids_cat >= 0
        out = torch.empty((n_total, 3), dtype=pos.dtype, device=dev)
        out[ids_cat[keep]] = pos_cat[keep]
        return out


def local_occupancy(target_occupancy: float, n_local: int, n_total: int, box_lengths, width: float,
                    r_comm: float) -> float:
    """Grid occupancy for a domain whose particles fill a (width + r_comm) x L_y
    strip of the L_x x L_y grid plane: keeps the columns as narrow as the
    single-domain grid would make them."""
    Lx = float(box_lengths[0])
    frac = min(1.0, (width + r_comm) / Lx)
    n_equiv = max(1.0, n_local / frac)
    return target_occupancy * n_local / n_equiv if n_equiv > 0 else target_occupancy


@dataclass
class _Domain:
    """What build_cluster_grid needs of a system when positions come separately."""

    n: int
    box: object


class DomainForces:
    """GPU non-bonded pass of one rank: local grid + halo-masked list, rebuilt
    every nstlist steps; per step halo exchange, force pass, halo reduction."""

    def __init__(self, dd: SlabDecomposition, system, params, m: int = 4, target_occupancy: float | None = None,
                 r_inner: float = 0.0):
        self.r_inner = r_inner  # dynamic pruning (pairlist.prune_pair_list); 0 = off
        self.dd = dd
        self.system = system
        self.params = params
        self.m = m
        self.occ = target_occupancy
        self.grid = None
        self.plist = None

    def rebuild(self, positions_global: torch.Tensor, balance: bool = False) -> DomainLayout:
        """Re-decompose (optionally rebalancing the slabs from the ranks'
        measured force-pass times first: collective) and rebuild the local
        grid and list."""
        native = self.dd._native is not None and positions_global.is_cuda
        if not native:
            self.dd.check_p2p()
        if balance and self.dd.N > 1 and getattr(self, "_ev", None) is not None:
            import torch.distributed as dist

            self._ev[1].synchronize()
            t = torch.tensor([max(self._ev[0].elapsed_time(self._ev[1]), 1e-6)], dtype=torch.float64,
                             device=positions_global.device)
            allt = [torch.zeros_like(t) for _ in range(self.dd.N)]
            dist.all_gather(allt, t, group=self.dd.group)
            self.dd.rebalance(torch.cat(allt).cpu().numpy())
        if native:  # the P2P timeout flag is checked by assign_local (no extra sync)
            self._ensure_globals(positions_global.device)
            lay, lpos, lq, lt, lhalo = self.dd.assign_local(positions_global.contiguous(), self.q_all, self.t_all)
            return self._build_local(lay, lpos, lq, lt, lhalo)
        lay = self.dd.assign(positions_global)
        return self._build_local(lay, positions_global.index_select(0, lay.local_ids).contiguous())

    def rebuild_local(self, home_ids: torch.Tensor, home_pos: torch.Tensor) -> DomainLayout:
        """List step from this rank's own particles (SlabDecomposition.migrate:
        neighbour exchanges only, no global all-gather), same slabs."""
        self.dd.check_p2p()
        lay, local_pos = self.dd.migrate(home_ids, home_pos)
        return self._build_local(lay, local_pos.contiguous())

    def _ensure_globals(self, dev) -> None:
        if not hasattr(self, "q_all"):
            self.q_all = torch.as_tensor(np.array(self.system.charges), device=dev)
            self.t_all = torch.as_tensor(np.array(self.system.lj_type), device=dev)

    def _build_local(self, lay: DomainLayout, local_pos: torch.Tensor, q=None, t=None, halo=None) -> DomainLayout:
        from . import list_step

        dev = local_pos.device
        self._ensure_globals(dev)
        self.local_pos = local_pos
        if q is None:
            ids = lay.local_ids
            q = self.q_all.index_select(0, ids)
            t = self.t_all.index_select(0, ids)
            halo = torch.zeros(lay.n_local, dtype=torch.uint8, device=dev)
            halo[lay.n_home:] = 1
        self.q, self.t, self.halo = q, t, halo
        n = lay.n_local
        sys_local = _Domain(n, self.system.box)
        occ = self.occ
        if occ is not None and self.dd.N > 1:
            w = float(np.diff(self.dd.boundaries).max())
            occ = local_occupancy(occ, n, self.system.n, self.system.box.lengths, w, self.dd.r_comm)
        self.grid, self.plist = list_step(sys_local, self.m, occ, self.system.box, self.params.r_list,
                                          positions=self.local_pos, r_inner=self.r_inner, halo=self.halo)
        if getattr(self, "_fcap", -1) < n:  # grow-only force / energy buffers
            self._fbuf = torch.empty((max(n, 1), 3), dtype=torch.float64, device=dev)
            self._fcap = n
            self.e = torch.zeros(2, dtype=torch.float64, device=dev)
            self.bad = torch.empty(2, dtype=torch.int64, device=dev)
        self.f = self._fbuf[:n]
        return lay

    def forces(self, energy: bool = True):
        """Halo exchange -> local pass -> halo reduction.  Returns (home
        forces (n_home, 3), energies (2,) summed over ranks when requested).

        ``overlap`` (NBX_DD_OVERLAP=1): one nbx_dd_force call -- on the
        NVLink peer path the halo travels while the force kernel runs the
        interior work items (groups that read no halo coordinate), the
        boundary items follow once it has landed.  Off by default: measured
        on 2 B200 at 1.5M atoms the peer exchange costs less than the split
        of the persistent force launch (962 vs 922 us per force step), so
        the three steps in sequence are faster at <= 4 GPUs; results are
        bit-identical either way (tools/dd_p2p_check.py)."""
        import os

        from . import compute_nonbonded_device

        overlap = getattr(self, "overlap", os.environ.get("NBX_DD_OVERLAP", "0") == "1")
        if self.local_pos.is_cuda:  # this rank's force-pass time (slab rebalancing)
            if getattr(self, "_ev", None) is None:
                self._ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            self._ev[0].record()
        # halo-first reduction (nbx_dd_force_seq): bit-identical, measured no
        # faster at 1.5M on 4 B200 (488 vs 483 us per force step), so opt-in
        seq_native = getattr(self, "halo_first", os.environ.get("NBX_DD_HALO_FIRST", "0") == "1")
        if self.dd._native is not None and self.local_pos.is_cuda and (overlap or seq_native):
            import ctypes

            from . import _device, _lib
            from .kernels import _params_struct

            p, table = _params_struct(self.params)
            L = _lib.box3(self.system.box.lengths)
            flags = _lib.FORCE_ENERGY if energy else 0
            # overlap: interior work items while the halo travels; halo_first:
            # the sequential step with the halo forces leaving before the rest
            # of the reduction (nbx_dd_force_seq)
            fn = _lib.load().nbx_dd_force if overlap else _lib.load().nbx_dd_force_seq
            _lib.check(fn(
                self.dd._native, self.plist.handle, self.grid.handle, _lib.ptr(self.local_pos), _lib.ptr(self.q),
                _lib.ptr(self.t), ctypes.byref(p), _lib.ptr(L), flags, _lib.ptr(self.f), _lib.ptr(self.e),
                _lib.ptr(self.bad), _device.stream()), "dd_force")
            del table
            home_f = self.f[:self.dd.layout.n_home]
            self._ev[1].record()
            e = self.dd.allreduce_energies(self.e.clone()) if energy else self.e
            return home_f, e
        self.dd.exchange_positions(self.local_pos)
        compute_nonbonded_device(self.plist, self.grid, self.local_pos, self.q, self.t, self.params,
                                 self.system.box, energy=energy, out=self.f, e_out=self.e, bad=self.bad)
        home_f = self.dd.reduce_halo_forces(self.f)
        if self.local_pos.is_cuda:
            self._ev[1].record()
        e = self.dd.allreduce_energies(self.e.clone()) if energy else self.e
        return home_f, e
