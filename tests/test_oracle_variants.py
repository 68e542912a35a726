"""Pins for the oracle's equation variants:

* conservative viscous work, D_j(u_i tau_ij) by first-derivative stencils of the
  pointwise flux H_j = u_i tau_ij (reading D-27);
* Sutherland viscosity mu(T) = T^1.5 (1 + S)/(T + S) ("viscosity can be
  treated either as a constant or as a spatially-varying term"; reading D-26).

Each is pinned against what the mathematics fixes, not against the oracle
itself: exact telescoping of the divergence form, convergence to the exact
continuous residual (Taylor jets with mu(T), independent code), reduction to the
constant-viscosity operator where mu = 1, and the mirror-doubled periodic
equivalence of symmetry boundaries.
"""
import math

import numpy as np
import pytest

from inputs import TGV_PHYS, mms_primitives, mms_state, perturbed_tgv
from inputs.generators import _coords
from tests.test_oracle_symmetry import first_half, mirror_double

SUTH = 110.4 / 288.0
LOW_RE = dict(Re=10.0, Pr=0.71, Minf=0.1, gamma=1.4)


@pytest.mark.parametrize("order", [4, 8])
@pytest.mark.parametrize("visc_law", [0, 1])
def test_conservative_work_conserves_energy(oracle_lib, order, visc_law):
    """With the viscous work in divergence form every equation telescopes (mu = 1):
    sum R_E = 0 to round-off at finite Re (the expanded form does not, D-5)."""
    n = (18, 16, 14)
    Q = perturbed_tgv(*n, amp=0.05)
    kw = dict(visc_law=visc_law, suth=SUTH if visc_law else 0.0)
    p = oracle_lib.OracleParams(*n, order, 2 * math.pi / 18, energy_form=1, **kw, **LOW_RE)
    R = oracle_lib.residual(p, Q)
    # with mu(T) the product-rule viscous terms (D-26) telescope in no equation
    # but continuity
    for f in (range(5) if visc_law == 0 else [0]):
        assert abs(R[f].sum()) / np.abs(R[f]).sum() < 1e-13, f
    pe = oracle_lib.OracleParams(*n, order, 2 * math.pi / 18, energy_form=0, **kw, **LOW_RE)
    Re_ = oracle_lib.residual(pe, Q)
    assert abs(Re_[4].sum()) / np.abs(Re_[4]).sum() > 1e-10
    # the two forms differ only in the energy equation
    assert np.array_equal(R[:4], Re_[:4])


def test_conservative_equals_expanded_when_inviscid(oracle_lib):
    n = (12, 10, 9)
    Q = perturbed_tgv(*n, amp=0.05)
    phys = dict(Re=math.inf, Pr=0.71, Minf=0.1, gamma=1.4)
    a = oracle_lib.residual(oracle_lib.OracleParams(*n, 6, 0.5, energy_form=1, **phys), Q)
    b = oracle_lib.residual(oracle_lib.OracleParams(*n, 6, 0.5, **phys), Q)
    assert np.array_equal(a, b)


LEVELS = {4: (16, 24, 32, 48), 8: (24, 32, 48)}


@pytest.mark.parametrize("order", [4, 8])
@pytest.mark.parametrize("energy_form,visc_law", [(1, 0), (0, 1), (1, 1)])
def test_variant_mms_convergence(oracle_lib, order, energy_form, visc_law):
    """The discrete residual converges to the exact continuous residual (jets,
    mu(T) by the chain rule) at the nominal order, at Re = 10 where the viscous
    terms are O(1) of the residual."""
    from oracle import jets
    suth = SUTH if visc_law else None
    errs = []
    Ns = LEVELS[order]
    for n in Ns:
        dx = 2 * math.pi / n
        p = oracle_lib.OracleParams(n, n, n, order, dx, energy_form=energy_form,
                                    visc_law=visc_law, suth=SUTH if visc_law else 0.0, **LOW_RE)
        R = oracle_lib.residual(p, mms_state(n))
        X, Y, Z = _coords(n, n, n, dx)
        Rx = jets.exact_residual(mms_primitives, X, Y, Z, suth=suth, **LOW_RE)
        errs.append([np.abs(R[f] - Rx[f]).max() / np.abs(Rx[f]).max() for f in range(5)])
    errs = np.array(errs)
    slope = np.log(errs[-2] / errs[-1]) / np.log(Ns[-1] / Ns[-2])
    assert np.all(slope > order - (0.3 if order == 4 else 0.7)), slope
    assert np.all(slope < order + 0.5), slope
    if visc_law:
        # the pin bites: mu(T) changes the exact residual by far more than the
        # discretisation error left at the finest level
        X, Y, Z = _coords(Ns[-1], Ns[-1], Ns[-1], 2 * math.pi / Ns[-1])
        R1 = jets.exact_residual(mms_primitives, X, Y, Z, **LOW_RE)
        Rs = jets.exact_residual(mms_primitives, X, Y, Z, suth=SUTH, **LOW_RE)
        for f in range(1, 5):
            d = np.abs(Rs[f] - R1[f]).max() / np.abs(Rs[f]).max()
            assert d > 20 * errs[-1][f], (f, d, errs[-1][f])


def test_sutherland_reduces_to_constant_viscosity_at_unit_temperature(oracle_lib):
    """mu(1) = 1 and grad T = 0 when T == 1 (rho = gamma M^2 p): the Sutherland
    residual equals the constant-viscosity one to round-off, and so do the
    TGV diagnostics at t = 0 (T == 1, reading D-2)."""
    n = (12, 11, 10)
    Q = perturbed_tgv(*n, amp=0.05, dx=0.5)
    # force T = 1: rho = gamma M^2 p, keep the velocity
    g, M = 1.4, 0.1
    u = Q[1:4] / Q[0]
    ke = 0.5 * (u ** 2).sum(axis=0)
    p = (g - 1) * (Q[4] - Q[0] * ke)
    rho = g * M * M * p
    Qt = np.ascontiguousarray(np.concatenate([rho[None], rho * u, (p / (g - 1) + rho * ke)[None]]))
    a = oracle_lib.residual(oracle_lib.OracleParams(*n, 8, 0.5, visc_law=1, suth=SUTH,
                                                    **LOW_RE), Qt)
    b = oracle_lib.residual(oracle_lib.OracleParams(*n, 8, 0.5, **LOW_RE), Qt)
    scale = np.abs(b.reshape(5, -1)).max(axis=1)
    assert np.all(np.abs((a - b).reshape(5, -1)).max(axis=1) / scale < 1e-12)
    # and at T != 1 the two differ at O(1) of the viscous terms
    c = oracle_lib.residual(oracle_lib.OracleParams(*n, 8, 0.5, visc_law=1, suth=SUTH,
                                                    **LOW_RE), Q)
    d = oracle_lib.residual(oracle_lib.OracleParams(*n, 8, 0.5, **LOW_RE), Q)
    assert np.abs(c[1:] - d[1:]).max() > 1e-4 * np.abs(d[1:]).max()


def test_sutherland_law_values(oracle_lib):
    """mu(T) enters the dissipation linearly: for a uniform temperature T0 the
    Sutherland dissipation is mu(T0) times the constant-viscosity one, with
    mu(T0) = T0^1.5 (1 + S)/(T0 + S) evaluated here independently."""
    n = (10, 9, 8)
    Q = perturbed_tgv(*n, amp=0.05, dx=0.6)
    g, M, T0 = 1.4, 0.1, 1.7
    u = Q[1:4] / Q[0]
    ke = 0.5 * (u ** 2).sum(axis=0)
    p = (g - 1) * (Q[4] - Q[0] * ke)
    rho = g * M * M * p / T0
    Qt = np.ascontiguousarray(np.concatenate([rho[None], rho * u, (p / (g - 1) + rho * ke)[None]]))
    mu0 = T0 ** 1.5 * (1 + SUTH) / (T0 + SUTH)
    ds = oracle_lib.diagnostics(oracle_lib.OracleParams(*n, 6, 0.6, visc_law=1, suth=SUTH,
                                                        **LOW_RE), Qt)
    dc = oracle_lib.diagnostics(oracle_lib.OracleParams(*n, 6, 0.6, **LOW_RE), Qt)
    assert abs(ds[2] - mu0 * dc[2]) <= 1e-12 * abs(dc[2])
    assert ds[0] == dc[0] and ds[1] == dc[1]


@pytest.mark.parametrize("axes", [(0,), (2,), (0, 1, 2)])
def test_variants_with_symmetry_equal_mirror_doubled(oracle_lib, axes):
    """H_j = u_i tau_ij is odd under the mirror of direction j: the symmetric
    problem equals the mirror-doubled periodic one bitwise, for both variants."""
    shape = (12, 10, 8)
    dx = 0.3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05, kmax=2)
    sym = tuple(1 if d in axes else 0 for d in range(3))
    kw = dict(energy_form=1, visc_law=1, suth=SUTH, **LOW_RE)
    ps = oracle_lib.OracleParams(*shape, 6, dx, dt=2e-4, sym=sym, **kw)
    full = tuple(n * (2 if d in axes else 1) for d, n in enumerate(shape))
    pp = oracle_lib.OracleParams(*full, 6, dx, dt=2e-4, **kw)
    D = mirror_double(Q, axes)
    assert np.array_equal(oracle_lib.residual(ps, Q), first_half(oracle_lib.residual(pp, D),
                                                                  axes, shape))
    assert np.array_equal(oracle_lib.step(ps, Q, 1, 2),
                          first_half(oracle_lib.step(pp, D, 1, 2), axes, shape))


def test_jet_sqrt_is_the_square_root_jet():
    """The Jet square root (used for mu(T) = T^1.5 (1+S)/(T+S) in the exact
    residual) against closed forms: sqrt(x^2 + y) has gradient (x, 1/2)/s and
    Hessian entries d2/dx2 = y/s^3, d2/dxdy = -x/(2 s^3), d2/dy2 = -1/(4 s^3)."""
    import numpy as np
    from oracle.jets import coordinate_jets
    X, Y, Z = np.meshgrid(np.linspace(0.3, 2.0, 5), np.linspace(0.5, 1.5, 4), [0.0], indexing="ij")
    x, y, z = coordinate_jets(X, Y, Z)
    s = (x * x + y).sqrt()
    sv = np.sqrt(X * X + Y)
    assert np.allclose(s.v, sv, rtol=1e-15, atol=0)
    assert np.allclose(s.g[0], X / sv, rtol=1e-14, atol=0)
    assert np.allclose(s.g[1], 0.5 / sv, rtol=1e-14, atol=0)
    assert np.all(s.g[2] == 0.0)
    assert np.allclose(s.h[0, 0], Y / sv ** 3, rtol=1e-13, atol=0)
    assert np.allclose(s.h[0, 1], -X / (2 * sv ** 3), rtol=1e-13, atol=0)
    assert np.allclose(s.h[1, 0], s.h[0, 1], rtol=0, atol=0)
    assert np.allclose(s.h[1, 1], -1.0 / (4 * sv ** 3), rtol=1e-13, atol=0)
