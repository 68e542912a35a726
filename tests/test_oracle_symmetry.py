"""Pins for the oracle's symmetry boundaries.

A symmetry boundary mirrors the interior about the boundary face, scalars
even, the vector component normal to the boundary odd ("phi(x_N) =
phi(x_{N-1}) for scalar fields and phi_i(x_N) = -phi_i(x_{N-1}) for vector
fields (in the direction i)").  Such a problem on N points is exactly the
periodic problem on 2N points whose second half is the mirror image of the
first: the periodic run preserves the mirror symmetry and its first N points
must equal the symmetric run (bitwise: the ghost values are the same numbers).
"""
import math

import numpy as np
import pytest

from inputs import TGV_PHYS, perturbed_tgv


def mirror_double(Q, axes):
    """Q [5][nz][ny][nx] -> periodic state doubled along each axis in `axes`
    (0 = x, 1 = y, 2 = z), mirrored with the parity of each field."""
    out = Q
    for d in axes:
        ax = 3 - d  # numpy axis of direction d
        sign = np.ones((5, 1, 1, 1))
        sign[1 + d] = -1.0  # rho u_d is odd under the mirror of direction d
        out = np.concatenate([out, sign * np.flip(out, axis=ax)], axis=ax)
    return np.ascontiguousarray(out)


def first_half(Q, axes, shape):
    nx, ny, nz = shape
    return Q[:, :nz, :ny, :nx]


@pytest.mark.parametrize("axes,order", [((0,), 4), ((1,), 8), ((2,), 12), ((0, 2), 6),
                                        ((0, 1, 2), 4)])
def test_symmetry_equals_mirror_doubled_periodic(oracle_lib, axes, order):
    shape = (14, 12, 10)
    dx = 0.3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05, kmax=2)
    sym = tuple(1 if d in axes else 0 for d in range(3))
    ps = oracle_lib.OracleParams(*shape, order, dx, dt=2e-3, sym=sym, **TGV_PHYS)
    D = mirror_double(Q, axes)
    full = tuple(n * (2 if d in axes else 1) for d, n in enumerate(shape))
    pp = oracle_lib.OracleParams(*full, order, dx, dt=2e-3, **TGV_PHYS)
    R_sym = oracle_lib.residual(ps, Q)
    R_per = oracle_lib.residual(pp, D)
    assert np.array_equal(R_sym, first_half(R_per, axes, shape))
    S_sym = oracle_lib.step(ps, Q, 1, 3)
    S_per = oracle_lib.step(pp, D, 1, 3)
    assert np.array_equal(S_sym, first_half(S_per, axes, shape))
    assert np.array_equal(oracle_lib.diagnostics(ps, S_sym), oracle_lib.diagnostics(pp, S_per))


def test_symmetry_ghost_examples(oracle_lib):
    """S:362-363 analogue on a 1D field: the first derivative of an even field
    vanishes in the mean at the mirror while an odd field's does not."""
    n, order = 16, 2
    dx = 1.0
    x = np.arange(n)
    f = (x + 0.5) ** 2  # even about the face x = -1/2
    p = oracle_lib.OracleParams(n, 1, 1, order, dx, sym=(1, 0, 0))
    d = oracle_lib.derivative(p, f[None, None, :], 1, 0)[0, 0]
    # at i = 0 the ghost -1 equals f(0) (mirror), so D f(0) = (f(1) - f(0)) / 2
    assert d[0] == (f[1] - f[0]) / 2


def test_symmetric_uniform_state_at_rest_is_equilibrium(oracle_lib):
    shape = (9, 8, 7)
    rho = np.ones(shape[::-1])
    Q = np.stack([rho, 0 * rho, 0 * rho, 0 * rho, 71.4 / 0.4 * rho])
    p = oracle_lib.OracleParams(*shape, 8, 0.2, sym=(1, 1, 1), **TGV_PHYS)
    assert np.all(oracle_lib.residual(p, np.ascontiguousarray(Q)) == 0.0)
