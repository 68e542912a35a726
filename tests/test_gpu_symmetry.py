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


def test_symmetry_z_unsupported_for_slabs(osbli):
    grp = osbli.LoopbackGroup(16, 16, 16, 4, 0.3, 1e-3, 2, **TGV_PHYS)
    with pytest.raises(osbli.OsbliError) as ei:
        grp.slabs[0].set_boundary(2, osbli.OSBLI_BC_SYMMETRY)
    assert ei.value.status == "E_UNSUPPORTED"
    grp.slabs[0].set_boundary(0, osbli.OSBLI_BC_SYMMETRY)
    grp.close()
