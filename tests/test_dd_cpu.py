"""Domain decomposition host logic on CPU: world_size 2 over gloo.

The slab/halo bookkeeping and the neighbour exchanges of
paper_1506_00716_b200.dd run unchanged; the local force pass (a CUDA kernel
in production) is the FP64 oracle here, with the same halo-halo masking the
GPU list builder applies.  The decomposed forces and energies must equal the
single-domain oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_oracle_forces(pos_local, q, t, halo, L, phys):
    from oracle import native, search

    occ = None
    og = search.build_grid(pos_local, L, 4, occ)
    ol = native.prune_list(native.search_list(og, L, 1.1), og["clustered_positions"], L)
    h = halo[og["perm"]].reshape(-1, 4) & ~og["fill_mask"].reshape(-1, 4)
    ci = search.row_ci(ol)
    both = h[ci][:, :, None] & h[ol["j_idx"]][:, None, :]
    ol = dict(ol, masks=ol["masks"] & ~both)
    fc, elj, ec = native.list_forces(ol, og, pos_local, q, t, L, phys, threads=2)
    return search.scatter_to_original(og, fc), elj, ec


def _worker(rank, world, port, out_q):
    import datetime

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    try:
        from oracle import forces as of
        from paper_1506_00716_b200.dd import SlabDecomposition
        from paper_1506_00716_b200.systems import spc_water

        s, table = spc_water(3000 * 4)  # 12k atoms, L = 4.93 nm
        L = s.box.lengths
        phys = of.Physics(r_cut=1.0, lj_table=table, shift_potential=True)
        dd = SlabDecomposition(L, world, rank, r_comm=1.1)
        lay = dd.assign(s.positions)
        ids = lay.local_ids.numpy()
        local = torch.zeros((lay.n_local, 3), dtype=torch.float64)
        local[:lay.n_home] = torch.from_numpy(s.positions[lay.home.numpy()])
        dd.exchange_positions(local)
        assert np.array_equal(local[lay.n_home:].numpy(), s.positions[lay.halo.numpy()])
        halo = np.zeros(lay.n_local, dtype=bool)
        halo[lay.n_home:] = True
        f, elj, ec = _local_oracle_forces(local.numpy(), s.charges[ids], s.lj_type[ids], halo, L, phys)
        home_f = dd.reduce_halo_forces(torch.from_numpy(f))
        e = dd.allreduce_energies(torch.tensor([elj, ec], dtype=torch.float64))
        glob = dd.allgather_home(lay.home, home_f, s.n)
        if rank == 0:
            out_q.put((glob.numpy(), e.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_slab_decomposition_equals_single_domain():
    from oracle import forces as of
    from oracle import native, search
    from paper_1506_00716_b200.systems import spc_water

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    f_dd, e_dd = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    s, table = spc_water(12000)
    L = s.box.lengths
    og = search.build_grid(s.positions, L, 4, None)
    ol = native.prune_list(native.search_list(og, L, 1.1), og["clustered_positions"], L)
    fc, elj, ec = native.list_forces(ol, og, s.positions, s.charges, s.lj_type, L,
                                     of.Physics(r_cut=1.0, lj_table=table, shift_potential=True), threads=2)
    f_ref = search.scatter_to_original(og, fc)
    assert np.abs(f_dd - f_ref).max() <= 1e-9 * np.abs(f_ref).max()
    assert abs(e_dd[0] - elj) <= 1e-9 * abs(elj) and abs(e_dd[1] - ec) <= 1e-9 * abs(ec)


def test_slab_geometry_checks():
    from paper_1506_00716_b200.dd import SlabDecomposition
    from paper_1506_00716_b200.model import ParameterError

    with pytest.raises(ParameterError):
        SlabDecomposition([4.0, 4.0, 4.0], 4, 0, r_comm=1.1)   # slabs narrower than r_comm
    dd = SlabDecomposition([9.8, 9.8, 9.8], 4, 1, r_comm=1.1)
    own = dd.owner(np.array([0.0, 2.44, 2.46, 9.79, -0.01, 9.8]))
    assert own.tolist() == [0, 0, 1, 3, 3, 0]
    lay = dd.assign(np.array([[0.1, 0, 0], [2.5, 0, 0], [3.0, 0, 0], [4.0, 0, 0], [5.0, 0, 0], [6.0, 0, 0]]))
    assert lay.home.tolist() == [1, 2, 3]          # slab 1 = [2.45, 4.9)
    assert lay.send.tolist() == [1, 2]             # within r_comm of its -x face
    assert lay.halo.tolist() == [4, 5]             # slab 2 within r_comm of 4.9


def test_rebalance_rule():
    """Equal times keep the slabs; a slow rank's slab shrinks toward the cost
    quantile (damped by alpha); widths stay >= r_comm and below the
    periodic-image bound; every rank computes the same boundaries."""
    from paper_1506_00716_b200.dd import SlabDecomposition
    from paper_1506_00716_b200.model import ParameterError

    L = [24.6, 24.6, 24.6]
    dd = SlabDecomposition(L, 4, 0, r_comm=1.1)
    b0 = dd.boundaries.copy()
    assert np.allclose(dd.rebalance([1.0, 1.0, 1.0, 1.0]), b0)
    dd = SlabDecomposition(L, 4, 0, r_comm=1.1)
    b = dd.rebalance([2.0, 1.0, 1.0, 1.0], alpha=1.0)
    # slab 0 holds 2/5 of the cost in 6.15 nm: the first quantile (1/4 of the
    # cost) sits at 6.15 * (5/4) / 2 = 3.84 nm
    assert abs(b[1] - 6.15 * 1.25 / 2.0) < 1e-9
    assert np.all(np.diff(b) >= 1.1 - 1e-12) and b[0] == 0.0 and b[-1] == 24.6
    other = SlabDecomposition(L, 4, 3, r_comm=1.1)
    assert np.array_equal(other.rebalance([2.0, 1.0, 1.0, 1.0], alpha=1.0), b)
    dd = SlabDecomposition(L, 4, 0, r_comm=2.0)
    b = dd.rebalance([1000.0, 1.0, 1.0, 1.0], alpha=1.0)  # extreme: quantiles 1.54 nm apart, clamped at r_comm
    assert np.allclose(b, [0.0, 2.0, 4.0, 6.0, 24.6])
    with pytest.raises(ParameterError):
        dd.rebalance([1.0, -1.0, 1.0, 1.0])


def _worker_uneven(rank, world, port, out_q):
    """as _worker, with the slab boundaries moved by the rebalancing rule"""
    import datetime

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    try:
        from oracle import forces as of
        from paper_1506_00716_b200.dd import SlabDecomposition
        from paper_1506_00716_b200.systems import spc_water

        s, table = spc_water(3000 * 4)
        L = s.box.lengths
        phys = of.Physics(r_cut=1.0, lj_table=table, shift_potential=True)
        dd = SlabDecomposition(L, world, rank, r_comm=1.1)
        t = torch.tensor([1.0 + rank], dtype=torch.float64)  # rank 1 "slower"
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        dd.rebalance(torch.cat(allt).numpy(), alpha=0.5)
        lay = dd.assign(s.positions)
        ids = lay.local_ids.numpy()
        local = torch.zeros((lay.n_local, 3), dtype=torch.float64)
        local[:lay.n_home] = torch.from_numpy(s.positions[lay.home.numpy()])
        dd.exchange_positions(local)
        halo = np.zeros(lay.n_local, dtype=bool)
        halo[lay.n_home:] = True
        f, elj, ec = _local_oracle_forces(local.numpy(), s.charges[ids], s.lj_type[ids], halo, L, phys)
        home_f = dd.reduce_halo_forces(torch.from_numpy(f))
        e = dd.allreduce_energies(torch.tensor([elj, ec], dtype=torch.float64))
        glob = dd.allgather_home(lay.home, home_f, s.n)
        if rank == 0:
            out_q.put((glob.numpy(), e.numpy(), dd.boundaries.copy()))
    finally:
        dist.destroy_process_group()


def test_rebalanced_decomposition_equals_single_domain():
    from oracle import forces as of
    from oracle import native, search
    from paper_1506_00716_b200.systems import spc_water

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_uneven, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    f_dd, e_dd, bnd = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    s, table = spc_water(12000)
    L = s.box.lengths
    assert abs(bnd[1] - 0.5 * L[0]) > 0.1  # the boundary did move
    og = search.build_grid(s.positions, L, 4, None)
    ol = native.prune_list(native.search_list(og, L, 1.1), og["clustered_positions"], L)
    fc, elj, ec = native.list_forces(ol, og, s.positions, s.charges, s.lj_type, L,
                                     of.Physics(r_cut=1.0, lj_table=table, shift_potential=True), threads=2)
    f_ref = search.scatter_to_original(og, fc)
    assert np.abs(f_dd - f_ref).max() <= 1e-9 * np.abs(f_ref).max()
    assert abs(e_dd[0] - elj) <= 1e-9 * abs(elj) and abs(e_dd[1] - ec) <= 1e-9 * abs(ec)


def test_balance_counts_equal_particles_per_slab():
    from paper_1506_00716_b200.dd import SlabDecomposition

    rng = np.random.default_rng(5)
    L = np.array([12.0, 5.0, 5.0])
    # density falls off along x (a partially filled last layer)
    x = np.concatenate([rng.uniform(0.0, 9.0, 9000), rng.uniform(9.0, 12.0, 1000)])
    for n_ranks in (2, 3, 4):
        d = SlabDecomposition(L, n_ranks, 0, r_comm=1.1)
        b = d.balance_counts(x)
        counts = np.bincount(d.owner(x), minlength=n_ranks)
        assert counts.max() - counts.min() <= 2, counts
        assert b[0] == 0.0 and b[-1] == L[0] and np.all(np.diff(b) >= 1.1)
    # the width clamps win over the counts (a slab may not be narrower than r_comm)
    d = SlabDecomposition(L, 4, 0, r_comm=1.1)
    b = d.balance_counts(np.full(100, 3.0))
    assert np.all(np.diff(b) >= 1.1 - 1e-12) and np.all(np.diff(b) <= L[0] - 2.2 + 1e-9)


def _migrate_worker(rank, world, port, out_q):
    import datetime

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    try:
        from paper_1506_00716_b200.dd import SlabDecomposition

        rng = np.random.default_rng(11)
        L = np.array([3.3 * world + 1.0, 4.0, 4.0])
        n = 4000
        x0 = rng.uniform(0.0, 1.0, (n, 3)) * L
        dd = SlabDecomposition(L, world, rank, r_comm=1.1)
        lay = dd.assign(torch.from_numpy(x0))
        ok = True
        for step in range(3):  # displacements up to 0.5 nm (< the slab width), wrapped or not
            x1 = x0 + rng.uniform(-0.5, 0.5, (n, 3))
            if step == 1:
                x1 = np.mod(x1, L)
            lay_m, local = dd.migrate(lay.home, torch.from_numpy(x1[lay.home.numpy()]))
            ref = SlabDecomposition(L, world, rank, r_comm=1.1).assign(torch.from_numpy(x1))
            ok &= all(torch.equal(getattr(lay_m, f), getattr(ref, f)) for f in ("home", "halo", "send", "send_local"))
            ok &= bool(np.array_equal(local.numpy(), x1[ref.local_ids.numpy()]))
            lay, x0 = lay_m, x1
        # a particle two slabs away (possible from 4 slabs on) is refused
        far = torch.from_numpy(x0[lay.home.numpy()])
        if world >= 4 and far.shape[0]:
            far[0, 0] += 2.0 * 3.3
            try:
                dd.migrate(lay.home, far)
                ok = False
            except RuntimeError:
                pass
        out_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_migrate_equals_assign(world):
    """Neighbour-only migration (the list step without the global all-gather)
    gives every rank the layout and local positions assign() computes from
    the gathered positions."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_migrate_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
