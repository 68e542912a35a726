"""Exact single-point oracle evaluation on a periodic window (TEST INFRASTRUCTURE ONLY).

The residual at a point reads Q only inside the cube of Chebyshev radius
m = order/2 around it (first, second and nested stencils), so after
S residual evaluations (S = 3 per RK3 step, 1 per Euler step) the value at a
point depends on Q inside radius S*m.  Running the unmodified oracle on the
periodic box of half-width S*m centred on the point therefore yields, at the
centre, bitwise the same arithmetic as the full-grid run (every operation at
the centre reads the same neighbour values in the same order).  Directions in
which the box would not be smaller than the grid keep the full periodic extent.
This lets the full-size GPU runs (BASELINE configs[3], 256^3) be checked on
sampled points against the oracle.  tests/test_oracle_pins.py pins it bitwise
against the full-grid oracle.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import core


def sample_step(p: core.OracleParams, Q: np.ndarray, points, scheme: int, nsteps: int):
    """Return the oracle's Q after `nsteps` at each (i, j, k) in `points` -> [len, 5]."""
    m = p.order // 2
    S = nsteps * (1 if scheme == 0 else 3)
    h = S * m
    Q = np.asarray(Q).reshape(p.shape)
    out = np.zeros((len(points), 5))
    n = (p.nx, p.ny, p.nz)
    for t, (i, j, k) in enumerate(points):
        c = (i, j, k)
        idx = []
        centre = []
        for d in range(3):
            if 2 * h + 1 >= n[d]:
                idx.append(np.arange(n[d]))
                centre.append(c[d])
            else:
                idx.append((np.arange(-h, h + 1) + c[d]) % n[d])
                centre.append(h)
        box = Q[:, idx[2]][:, :, idx[1]][:, :, :, idx[0]]
        bp = dataclasses.replace(p, nx=len(idx[0]), ny=len(idx[1]), nz=len(idx[2]))
        Qb = core.step(bp, np.ascontiguousarray(box), scheme, nsteps)
        out[t] = Qb[:, centre[2], centre[1], centre[0]]
    return out


def sample_residual(p: core.OracleParams, Q: np.ndarray, points):
    """Oracle residual R(Q) at the sampled points -> [len, 5]."""
    m = p.order // 2
    Q = np.asarray(Q).reshape(p.shape)
    n = (p.nx, p.ny, p.nz)
    out = np.zeros((len(points), 5))
    for t, (i, j, k) in enumerate(points):
        c = (i, j, k)
        idx, centre = [], []
        for d in range(3):
            if 2 * m + 1 >= n[d]:
                idx.append(np.arange(n[d]))
                centre.append(c[d])
            else:
                idx.append((np.arange(-m, m + 1) + c[d]) % n[d])
                centre.append(m)
        box = Q[:, idx[2]][:, :, idx[1]][:, :, :, idx[0]]
        bp = dataclasses.replace(p, nx=len(idx[0]), ny=len(idx[1]), nz=len(idx[2]))
        Rb = core.residual(bp, np.ascontiguousarray(box))
        out[t] = Rb[:, centre[2], centre[1], centre[0]]
    return out


def sample_block(p: core.OracleParams, Q: np.ndarray, lo, size, scheme: int, nsteps: int):
    """Oracle Q after `nsteps` on the block of points lo[d] <= i_d < lo[d] + size[d]
    (indices taken modulo the grid, so a block may straddle the periodic wrap)
    -> [5][size_z][size_y][size_x].

    The same argument as sample_step, for a block: the box is the block widened
    by h = S*m points on each side, so every block point is at least h from the
    box faces and its value is bitwise the full-grid oracle's.  Directions where
    the box would not be smaller than the grid keep the full periodic extent.
    """
    m = p.order // 2
    S = nsteps * (1 if scheme == 0 else 3)
    h = S * m
    Q = np.asarray(Q).reshape(p.shape)
    n = (p.nx, p.ny, p.nz)
    idx, sel = [], []
    for d in range(3):
        if 2 * h + size[d] >= n[d]:
            idx.append(np.arange(n[d]))
            sel.append((np.arange(size[d]) + lo[d]) % n[d])
        else:
            idx.append((np.arange(-h, h + size[d]) + lo[d]) % n[d])
            sel.append(np.arange(h, h + size[d]))
    box = Q[:, idx[2]][:, :, idx[1]][:, :, :, idx[0]]
    bp = dataclasses.replace(p, nx=len(idx[0]), ny=len(idx[1]), nz=len(idx[2]))
    Qb = core.step(bp, np.ascontiguousarray(box), scheme, nsteps)
    return Qb[:, sel[2]][:, :, sel[1]][:, :, :, sel[0]]
