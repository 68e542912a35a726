"""The distributed (ghost-plane) kernel path on one GPU: z-slab handles that
exchange ghost planes by device copies (osbli_create_loopback) must reproduce
the single-domain run BITWISE (ghosts are exact copies and the per-point
arithmetic does not depend on the decomposition), including the diagnostics
(per-plane partials summed in global plane order)."""
import math

import numpy as np
import pytest

from inputs import TGV_PHYS, perturbed_tgv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def osbli():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_1609_01277_b200 as pkg
    return pkg


@pytest.mark.parametrize("schedule", [0, 1, 2])
@pytest.mark.parametrize("order,nslabs,shape", [(4, 2, (24, 20, 16)), (4, 3, (24, 20, 17)),
                                                (12, 2, (20, 18, 24)), (12, 4, (33, 17, 26)),
                                                (8, 8, (16, 16, 64)), (12, 2, (64, 48, 80)),
                                                (12, 3, (96, 64, 48)), (4, 2, (128, 64, 40))])
def test_loopback_slabs_bitwise_equal_single_domain(osbli, order, nslabs, shape, schedule):
    """The three stage schedules (plain; z-split: interior z-pass, then the two
    face ranges in one launch; xy-split: face xy-pass, then the interior one;
    DESIGN.md §6) on 2-8 slabs, uneven splits included.  The wide grids give the
    xy-pass tiles that stage by TMA and the z-pass TMA boxes through ghost planes."""
    dx = 2 * math.pi / max(shape)
    dt = 2e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.02)
    ref = osbli.Solver(*shape, order, dx, dt, **TGV_PHYS)
    ref.set_state(Q)
    ref.step(3)
    grp = osbli.LoopbackGroup(*shape, order, dx, dt, nslabs, **TGV_PHYS)
    for sl in grp.slabs:
        sl.set_slab_schedule(schedule)
    grp.set_state(Q)
    assert [s.z0 for s in grp.slabs] == [osbli.slab_bounds(shape[2], nslabs, r)[0]
                                         for r in range(nslabs)]
    grp.step(3)
    assert np.array_equal(grp.get_state(), ref.get_state())
    d_ref, d_grp = ref.diagnostics(), grp.slabs[nslabs - 1].diagnostics()
    assert (d_ref.kinetic_energy, d_ref.enstrophy, d_ref.dissipation) == \
        (d_grp.kinetic_energy, d_grp.enstrophy, d_grp.dissipation)
    # residual hook per slab == the corresponding planes of the full residual
    R = ref.residual()
    for s in grp.slabs:
        assert np.array_equal(s.residual(), R[:, s.z0:s.z0 + s.nz])
    with pytest.raises(osbli.OsbliError):
        grp.slabs[0].step(1)  # members advance together only
    grp.close()


@pytest.mark.parametrize("order,nslabs,shape", [(4, 2, (24, 20, 16)), (12, 3, (20, 18, 40))])
def test_loopback_two_register_rk3(osbli, order, nslabs, shape):
    """OSBLI_RK3_2R on the ghost-plane path (its z-pass writes into the destination
    buffer's interior planes; the ghost planes and the split schedule must not care)."""
    dx = 2 * math.pi / max(shape)
    dt = 2e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.02)
    ref = osbli.Solver(*shape, order, dx, dt, scheme=osbli.OSBLI_RK3_2R, **TGV_PHYS)
    ref.set_state(Q)
    ref.step(3)
    grp = osbli.LoopbackGroup(*shape, order, dx, dt, nslabs, scheme=osbli.OSBLI_RK3_2R,
                              **TGV_PHYS)
    grp.set_state(Q)
    grp.step(3)
    assert np.array_equal(grp.get_state(), ref.get_state())
    grp.close()


@pytest.mark.parametrize("scheme,visc,nslabs,order", [(0, False, 2, 6), (2, True, 3, 8),
                                                      (1, True, 4, 4), (0, True, 2, 12),
                                                      (2, False, 5, 2)])
def test_loopback_switch_combinations(osbli, scheme, visc, nslabs, order):
    """The ghost-plane path with the time schemes and Sutherland viscosity (the
    variants that slabs support) equals the single-domain run bitwise."""
    shape = (20, 18, 6 * nslabs + 5)
    dx = 2 * math.pi / max(shape)
    dt = 1e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05, seed=11 + nslabs)
    ref = osbli.Solver(*shape, order, dx, dt, scheme=scheme, **TGV_PHYS)
    grp = osbli.LoopbackGroup(*shape, order, dx, dt, nslabs, scheme=scheme, **TGV_PHYS)
    if visc:
        ref.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, 110.4 / 288.0)
        for sl in grp.slabs:
            sl.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, 110.4 / 288.0)
    ref.set_state(Q)
    ref.step(2)
    grp.set_state(Q)
    grp.step(2)
    assert np.array_equal(grp.get_state(), ref.get_state())
    d_ref, d_grp = ref.diagnostics(), grp.slabs[0].diagnostics()
    assert (d_ref.kinetic_energy, d_ref.dissipation) == (d_grp.kinetic_energy, d_grp.dissipation)
    grp.close()


@pytest.mark.parametrize("schedule", [0, 1, 2])
@pytest.mark.parametrize("order,symz,cons,shape", [(4, False, False, (24, 20, 26)),
                                                   (12, False, False, (24, 20, 26)),
                                                   (8, True, False, (24, 20, 26)),
                                                   (6, False, True, (24, 20, 26)),
                                                   (12, False, False, (96, 64, 26)),
                                                   (8, True, True, (96, 64, 26))])
def test_single_rank_nccl_path_bitwise(osbli, order, symz, cons, shape, schedule):
    """One rank with an NCCL unique id runs the distributed code path with NCCL:
    its ghost planes come from itself through ncclSend/ncclRecv (or the mirror),
    the z-pass reads ghost planes, the diagnostics go through ncclAllGather.
    The result equals the single-domain run bitwise.  This exercises the NCCL
    calls of the multi-GPU path on one GPU without ranks waiting on each other
    (the 96 x 64 grids: TMA staging through the ghost planes)."""
    dx, dt = 2 * math.pi / 26, 1e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05)
    uid = osbli.nccl_unique_id()
    dist = osbli.Solver(*shape, order, dx, dt, rank=0, nranks=1, unique_id=uid, **TGV_PHYS)
    # 1: exchange on the comm stream behind the interior z-pass; 2: the new state's
    # faces exchanged behind the interior xy-pass, waited for by the next stage
    dist.set_slab_schedule(schedule)
    ref = osbli.Solver(*shape, order, dx, dt, **TGV_PHYS)
    for s in (dist, ref):
        if symz:
            s.set_boundary(2, osbli.OSBLI_BC_SYMMETRY)
        if cons:
            s.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
        s.set_state(Q)
        s.step(3)
    assert np.array_equal(dist.get_state(), ref.get_state())
    d1, d2 = dist.diagnostics(), ref.diagnostics()
    assert (d1.kinetic_energy, d1.enstrophy, d1.dissipation) == \
        (d2.kinetic_energy, d2.enstrophy, d2.dissipation)
    if not cons:
        assert np.array_equal(dist.residual(), ref.residual())


def test_loopback_nonfinite_is_agreed_by_every_slab(osbli):
    """A non-finite value in one slab poisons every member of the group (the
    collective flag policy of osbli_diagnostics / osbli_sync): none of them may
    step again, so no slab waits on a peer that refuses."""
    shape, order = (16, 12, 24), 4
    Q = perturbed_tgv(*shape, dx=0.3, amp=0.02)
    Q[0, 20, 3, 4] = 0.0  # rho = 0 in the last slab
    grp = osbli.LoopbackGroup(*shape, order, 0.3, 1e-3, 3, **TGV_PHYS)
    grp.set_state(Q)
    grp.step(1)
    with pytest.raises(osbli.OsbliError) as ei:
        grp.slabs[0].diagnostics()
    assert ei.value.status == "E_NONFINITE"
    for sl in grp.slabs:
        with pytest.raises(osbli.OsbliError) as ei:
            sl.sync()
        assert ei.value.status == "E_STATE"
    with pytest.raises(osbli.OsbliError):
        grp.step(1)
    assert np.isfinite(grp.slabs[0].get_state()).any()  # get_state stays valid
    grp.close()


def test_loopback_member_destroyed_is_reported_not_crashed(osbli):
    """Destroying one member breaks the group: the others report E_STATE from
    calls that need the siblings instead of dereferencing the destroyed one."""
    shape, order = (16, 12, 24), 4
    grp = osbli.LoopbackGroup(*shape, order, 0.3, 1e-3, 3, **TGV_PHYS)
    grp.set_state(perturbed_tgv(*shape, dx=0.3, amp=0.02))
    grp.slabs[1].close()
    for r in (0, 2):
        with pytest.raises(osbli.OsbliError) as ei:
            grp.slabs[r].diagnostics()
        assert ei.value.status == "E_STATE"
        with pytest.raises(osbli.OsbliError) as ei:
            grp.slabs[r].residual()
        assert ei.value.status == "E_STATE"
    grp.close()


@pytest.mark.parametrize("schedule", [0, 2])
def test_single_rank_nccl_fused_diagnostics_bitwise(osbli, schedule):
    """osbli_step_diag through the distributed path (ncclAllGather of the per-step
    plane partials, collective non-finite check) equals the single domain bitwise."""
    shape, order = (24, 20, 26), 8
    dx, dt = 2 * math.pi / 26, 1e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05)
    dist = osbli.Solver(*shape, order, dx, dt, rank=0, nranks=1, unique_id=osbli.nccl_unique_id(),
                        **TGV_PHYS)
    dist.set_slab_schedule(schedule)
    ref = osbli.Solver(*shape, order, dx, dt, **TGV_PHYS)
    out = []
    for s in (dist, ref):
        s.set_state(Q)
        out.append([(d.kinetic_energy, d.enstrophy, d.dissipation) for d in s.step_diag(70)])
    assert out[0] == out[1]
    assert np.array_equal(dist.get_state(), ref.get_state())
