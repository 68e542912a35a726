"""SURVEY §8(f) N2(b) and N4 on the GPU: conservative viscous work (D-27) and
Sutherland viscosity mu(T) (D-26), through the C ABI, against the oracle."""
import math

import numpy as np
import pytest

from inputs import perturbed_tgv
from tests.test_oracle_symmetry import first_half, mirror_double

pytestmark = pytest.mark.gpu
TOL = 1e-11
SUTH = 110.4 / 288.0
PHYS = dict(Re=50.0, Pr=0.71, Minf=0.1, gamma=1.4)


@pytest.fixture(scope="module")
def osbli():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_1609_01277_b200 as pkg
    return pkg


def relerr(a, b):
    a, b = np.asarray(a).reshape(5, -1), np.asarray(b).reshape(5, -1)
    return np.array([np.max(np.abs(a[f] - b[f])) / max(np.max(np.abs(b[f])), 1e-300)
                     for f in range(5)])


def solver(osbli, shape, order, dx, dt, visc, cons, scheme=1, sym=()):
    s = osbli.Solver(*shape, order, dx, dt, scheme=scheme, **PHYS)
    if visc:
        s.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, SUTH)
    if cons:
        s.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
    for d in sym:
        s.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
    return s


def oparams(orc, shape, order, dx, dt, visc, cons, sym=()):
    return orc.OracleParams(*shape, order, dx, dt=dt, energy_form=int(cons), visc_law=int(visc),
                            suth=SUTH if visc else 0.0,
                            sym=tuple(1 if d in sym else 0 for d in range(3)), **PHYS)


CASES = [(4, (40, 36, 33)), (8, (24, 20, 17)), (12, (36, 34, 30)), (6, (13, 11, 9))]


@pytest.mark.parametrize("visc,cons", [(1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("order,shape", CASES)
def test_variant_residual_and_steps(osbli, oracle_lib, visc, cons, order, shape):
    dx = 2 * math.pi / max(shape)
    dt = 0.2 * dx / 11.0
    Q = perturbed_tgv(*shape, dx=dx, amp=0.1, kmax=3)
    s = solver(osbli, shape, order, dx, dt, visc, cons)
    po = oparams(oracle_lib, shape, order, dx, dt, visc, cons)
    s.set_state(Q)
    assert np.all(relerr(s.residual(), oracle_lib.residual(po, Q)) < TOL)
    s.step(4)
    Qo = oracle_lib.step(po, Q, 1, 4)
    assert np.all(relerr(s.get_state(), Qo) < TOL)
    d = s.diagnostics()
    do = oracle_lib.diagnostics(po, Qo)
    for a, b in zip((d.kinetic_energy, d.enstrophy, d.dissipation), do):
        assert abs(a - b) <= 1e-12 * abs(b)


@pytest.mark.parametrize("scheme", [0, 2])
def test_variant_other_schemes(osbli, oracle_lib, scheme):
    shape, order = (24, 22, 20), 8
    dx = 2 * math.pi / 24
    dt = 0.1 * dx / 11.0
    Q = perturbed_tgv(*shape, dx=dx, amp=0.1, kmax=3)
    s = solver(osbli, shape, order, dx, dt, 1, 1, scheme=scheme)
    s.set_state(Q)
    s.step(3)
    Qo = oracle_lib.step(oparams(oracle_lib, shape, order, dx, dt, 1, 1), Q, scheme, 3)
    assert np.all(relerr(s.get_state(), Qo) < TOL)


def test_conservative_energy_telescopes_on_gpu(osbli, oracle_lib):
    shape, order = (32, 30, 28), 6
    dx = 2 * math.pi / 32
    Q = perturbed_tgv(*shape, dx=dx, amp=0.1, kmax=3)
    s = solver(osbli, shape, order, dx, 1e-3, 0, 1)
    s.set_state(Q)
    R = s.residual()
    for f in range(5):
        assert abs(R[f].sum()) / np.abs(R[f]).sum() < 1e-13, f
    s2 = solver(osbli, shape, order, dx, 1e-3, 0, 0)
    s2.set_state(Q)
    R2 = s2.residual()
    assert abs(R2[4].sum()) / np.abs(R2[4]).sum() > 1e-10


@pytest.mark.parametrize("axes", [(0,), (1, 2), (0, 1, 2)])
def test_variants_with_symmetry(osbli, oracle_lib, axes):
    shape, order = (20, 18, 16), 8
    dx, dt = 0.3, 2e-4
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05, kmax=2)
    s = solver(osbli, shape, order, dx, dt, 1, 1, sym=axes)
    s.set_state(Q)
    po = oparams(oracle_lib, shape, order, dx, dt, 1, 1, sym=axes)
    assert np.all(relerr(s.residual(), oracle_lib.residual(po, Q)) < TOL)
    s.step(2)
    G = s.get_state()
    assert np.all(relerr(G, oracle_lib.step(po, Q, 1, 2)) < TOL)
    full = tuple(n * (2 if d in axes else 1) for d, n in enumerate(shape))
    sp = solver(osbli, full, order, dx, dt, 1, 1)
    sp.set_state(mirror_double(Q, axes))
    sp.step(2)
    assert np.all(relerr(G, first_half(sp.get_state(), axes, shape)) < 1e-13)


def test_sutherland_on_slabs_bitwise(osbli):
    shape, order, nslabs = (24, 20, 30), 8, 3
    dx, dt = 2 * math.pi / 30, 2e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05)
    ref = solver(osbli, shape, order, dx, dt, 1, 0)
    ref.set_state(Q)
    ref.step(3)
    grp = osbli.LoopbackGroup(*shape, order, dx, dt, nslabs, **PHYS)
    for sl in grp.slabs:
        sl.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, SUTH)
    grp.set_state(Q)
    grp.step(3)
    assert np.array_equal(grp.get_state(), ref.get_state())
    grp.close()


@pytest.mark.parametrize("visc,scheme,nslabs,order,symz", [(False, 1, 2, 4, False),
                                                           (True, 1, 3, 8, False),
                                                           (True, 2, 2, 12, True),
                                                           (False, 0, 4, 6, True)])
def test_conservative_work_on_slabs_bitwise(osbli, visc, scheme, nslabs, order, symz):
    """The conservative viscous work on slab handles: the flux H's ghost planes
    are exchanged every stage (mirrored at symmetric faces); equal to the single
    domain bitwise."""
    shape = (20, 18, 7 * nslabs + 4)
    dx, dt = 2 * math.pi / max(shape), 2e-4
    Q = perturbed_tgv(*shape, dx=dx, amp=0.1, kmax=3)
    ref = solver(osbli, shape, order, dx, dt, visc, 1, scheme=scheme, sym=(2,) if symz else ())
    grp = osbli.LoopbackGroup(*shape, order, dx, dt, nslabs, scheme=scheme, **PHYS)
    for sl in grp.slabs:
        if visc:
            sl.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, SUTH)
        sl.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
        if symz:
            sl.set_boundary(2, osbli.OSBLI_BC_SYMMETRY)
    ref.set_state(Q)
    ref.step(3)
    grp.set_state(Q)
    grp.step(3)
    assert np.array_equal(grp.get_state(), ref.get_state())
    with pytest.raises(osbli.OsbliError) as ei:
        grp.slabs[0].residual()
    assert ei.value.status == "E_UNSUPPORTED"
    grp.close()


def test_variant_switches_back(osbli, oracle_lib):
    """Turning the variants off restores the default operator exactly."""
    shape, order = (16, 16, 16), 4
    dx = 2 * math.pi / 16
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05)
    s = solver(osbli, shape, order, dx, 1e-3, 1, 1)
    s.set_state(Q)
    s.residual()
    s.set_viscosity(osbli.OSBLI_VISC_CONSTANT)
    s.set_energy_form(osbli.OSBLI_ENERGY_EXPANDED)
    d = osbli.Solver(*shape, order, dx, 1e-3, **PHYS)
    d.set_state(Q)
    assert np.array_equal(s.residual(), d.residual())
    with pytest.raises(osbli.OsbliError):
        s.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, -1.0)
    with pytest.raises(osbli.OsbliError):
        s.set_energy_form(7)
