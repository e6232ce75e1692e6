"""nbx_list_step (pairlist.list_step): the one-call rebuild of the device
drivers gives the same grid and lists as the separate build_cluster_grid /
build_pair_list / exclude_molecules / prune_pair_list calls (bit-identical),
and the same forces as a list whose force layout the force call builds."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _spc(n):
    import paper_1506_00716_b200 as nbx
    from paper_1506_00716_b200.systems import spc_water, tuned_occupancy

    s, table = spc_water(n, seed=2024)
    return nbx, s, table, tuned_occupancy(n, float(s.box.lengths[0]), 4)


def _same_lists(a, b):
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.j_idx, b.j_idx)
    assert np.array_equal(a.mask_bits, b.mask_bits)


@pytest.mark.parametrize("m,molecules,r_inner,halo", [(4, False, 0.0, False), (4, True, 1.05, False),
                                                      (8, True, 0.0, False), (4, False, 0.0, True)])
def test_list_step_matches_separate_calls(m, molecules, r_inner, halo):
    nbx, s, table, occ = _spc(24000)
    pos = torch.from_numpy(np.array(s.positions)).cuda()
    mol = nbx.Molecules(np.arange(s.n) // 3) if molecules else None
    hl = None
    if halo:  # mark the particles of the upper x half as another rank's halo
        hl = torch.from_numpy((np.asarray(s.positions)[:, 0] > 0.5 * s.box.lengths[0]).astype(np.uint8)).cuda()
    g1 = nbx.build_cluster_grid(s, m, occ, positions=pos)
    b1 = nbx.build_pair_list(g1, s.box, 1.1, molecules=mol, halo=hl)
    p1 = nbx.prune_pair_list(b1, g1.clustered_positions_device, s.box, r_inner=r_inner)
    g2, p2 = nbx.list_step(s, m, occ, s.box, 1.1, positions=pos, r_inner=r_inner, molecules=mol, halo=hl)
    for f in ("perm", "inverse_perm", "fill_mask", "cell_of_cluster", "clustered_positions", "bboxes"):
        assert np.array_equal(getattr(g1, f), getattr(g2, f)), f
    _same_lists(p1, p2)
    assert p1.n_entries == p2.n_entries
    assert p1.force_pairs(inner=True) == p2.force_pairs(inner=True)
    params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                                 ewald_beta=nbx.ewald_beta(1.0))
    q = torch.from_numpy(np.array(s.charges)).cuda()
    t = torch.from_numpy(np.array(s.lj_type)).cuda()
    f1, e1, _ = nbx.compute_nonbonded_device(p1, g1, pos, q, t, params, s.box)
    f2, e2, _ = nbx.compute_nonbonded_device(p2, g2, pos, q, t, params, s.box)
    assert torch.equal(f1, f2) and torch.equal(e1, e2)  # bit-identical: same layout, same order


def test_list_step_without_prune_and_errors():
    from paper_1506_00716_b200.model import ParameterError

    nbx, s, table, occ = _spc(3000)
    g1 = nbx.build_cluster_grid(s, 4, occ)
    b1 = nbx.build_pair_list(g1, s.box, 1.1)
    _, b2 = nbx.list_step(s, 4, occ, s.box, 1.1, prune=False)
    _same_lists(b1, b2)
    with pytest.raises(ParameterError):
        nbx.list_step(s, 3, occ, s.box, 1.1)
    with pytest.raises(ParameterError):
        nbx.list_step(s, 4, occ, s.box, 1.1, r_inner=1.2)
