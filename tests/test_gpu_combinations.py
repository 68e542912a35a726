"""Seeded combinations of every switch of the path — order, time scheme,
symmetry boundaries, Sutherland viscosity, conservative viscous work, source
term, grid shape (ragged, tiny, anisotropic) — against the oracle: residual and
two steps to 1e-11 (each switch is also pinned on its own in
the other test files, this catches their interactions)."""
import math

import numpy as np
import pytest

from inputs import perturbed_tgv

pytestmark = pytest.mark.gpu
TOL = 1e-11
SUTH = 110.4 / 288.0


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


def _cases(n=40, seed=1609):
    rng = np.random.default_rng(seed)
    out = []
    for c in range(n):
        order = int(rng.choice([2, 4, 6, 8, 10, 12]))
        m = order // 2
        shape = tuple(int(rng.integers(max(3, m), 41)) for _ in range(3))
        sym = tuple(int(rng.random() < 0.35) for _ in range(3))
        out.append(dict(order=order, shape=shape, scheme=int(rng.integers(0, 3)), sym=sym,
                        visc=bool(rng.random() < 0.4), cons=bool(rng.random() < 0.4),
                        src=bool(rng.random() < 0.3), Re=float(rng.choice([50.0, 1600.0]))))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: "o{order}-s{scheme}-{shape}".format(**c))
def test_switch_combinations(osbli, oracle_lib, case):
    shape, order, scheme = case["shape"], case["order"], case["scheme"]
    phys = dict(Re=case["Re"], Pr=0.71, Minf=0.1, gamma=1.4)
    dx = 2 * math.pi / max(shape)
    dt = (0.1 if scheme else 0.02) * dx / 11.0
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05, kmax=2, seed=7 + order)
    S = 0.01 * perturbed_tgv(*shape, dx=dx, amp=0.5, kmax=1, seed=3) if case["src"] else None
    s = osbli.Solver(*shape, order, dx, dt, scheme=scheme, **phys)
    for d in range(3):
        if case["sym"][d]:
            s.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
    if case["visc"]:
        s.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, SUTH)
    if case["cons"]:
        s.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
    if S is not None:
        s.set_source(S)
    po = oracle_lib.OracleParams(*shape, order, dx, dt=dt, sym=case["sym"],
                                 energy_form=int(case["cons"]), visc_law=int(case["visc"]),
                                 suth=SUTH if case["visc"] else 0.0, **phys)
    s.set_state(Q)
    Ro = oracle_lib.residual(po, Q)
    if S is not None:
        Ro = Ro + S
    assert np.all(relerr(s.residual(), Ro) < TOL)
    s.step(2)
    if S is None:
        Qo = oracle_lib.step(po, Q, scheme, 2)
        assert np.all(relerr(s.get_state(), Qo) < TOL)
    s.close()
