"""N3 on the GPU: symmetry boundaries against the oracle, and against the
GPU's own periodic run of the mirror-doubled domain."""
import math

import numpy as np
import pytest

from inputs import TGV_PHYS, perturbed_tgv
from tests.test_oracle_symmetry import first_half, mirror_double

pytestmark = pytest.mark.gpu
TOL = 1e-11


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


@pytest.mark.parametrize("axes,order,shape", [((0,), 4, (40, 20, 18)), ((1,), 12, (36, 44, 16)),
                                              ((2,), 8, (33, 17, 40)), ((0, 1, 2), 12, (36, 34, 30)),
                                              ((0, 2), 6, (13, 11, 9))])
def test_symmetry_parity_with_oracle_and_mirror(osbli, oracle_lib, axes, order, shape):
    dx = 0.25
    dt = 1e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.03, kmax=2)
    sym = tuple(1 if d in axes else 0 for d in range(3))
    s = osbli.Solver(*shape, order, dx, dt, **TGV_PHYS)
    for d in axes:
        s.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
    s.set_state(Q)
    R = s.residual()
    po = oracle_lib.OracleParams(*shape, order, dx, dt=dt, sym=sym, **TGV_PHYS)
    assert np.all(relerr(R, oracle_lib.residual(po, Q)) < TOL)
    s.step(3)
    G = s.get_state()
    assert np.all(relerr(G, oracle_lib.step(po, Q, 1, 3)) < TOL)
    d_sym = s.diagnostics()
    # the GPU's periodic solver on the mirror-doubled domain
    full = tuple(n * (2 if d in axes else 1) for d, n in enumerate(shape))
    sp = osbli.Solver(*full, order, dx, dt, **TGV_PHYS)
    sp.set_state(mirror_double(Q, axes))
    sp.step(3)
    P = first_half(sp.get_state(), axes, shape)
    assert np.all(relerr(G, P) < 1e-13)
    d_per = sp.diagnostics()
    for a, b in ((d_sym.kinetic_energy, d_per.kinetic_energy), (d_sym.enstrophy, d_per.enstrophy),
                 (d_sym.dissipation, d_per.dissipation)):
        assert abs(a - b) <= 1e-13 * abs(b)


@pytest.mark.parametrize("axes,order,nslabs", [((2,), 4, 2), ((0, 2), 12, 3), ((0, 1, 2), 8, 4),
                                                ((1,), 6, 2)])
def test_symmetry_on_slabs_bitwise(osbli, axes, order, nslabs):
    """Slab handles with symmetry boundaries: the outer slabs mirror their own
    planes instead of exchanging across the periodic wrap; the result equals the
    single-domain symmetric run bitwise (fields and diagnostics)."""
    shape = (20, 18, 8 * nslabs + 3)
    dx, dt = 0.3, 1e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05, kmax=2)
    ref = osbli.Solver(*shape, order, dx, dt, **TGV_PHYS)
    grp = osbli.LoopbackGroup(*shape, order, dx, dt, nslabs, **TGV_PHYS)
    for d in axes:
        ref.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
        for sl in grp.slabs:
            sl.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
    ref.set_state(Q)
    ref.step(3)
    grp.set_state(Q)
    grp.step(3)
    assert np.array_equal(grp.get_state(), ref.get_state())
    d_ref, d_grp = ref.diagnostics(), grp.slabs[0].diagnostics()
    assert (d_ref.kinetic_energy, d_ref.enstrophy, d_ref.dissipation) == \
        (d_grp.kinetic_energy, d_grp.enstrophy, d_grp.dissipation)
    R = ref.residual()
    for sl in grp.slabs:
        assert np.array_equal(sl.residual(), R[:, sl.z0:sl.z0 + sl.nz])
    grp.close()
