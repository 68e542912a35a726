"""Input generators (see package docstring).  All arrays: [5][nz][ny][nx], fp64.

Grid convention (reading D-9): x_i = i * dx, i = 0..N-1, isotropic
dx; the periodic box is [0, N_x dx) x [0, N_y dx) x [0, N_z dx).
"""
from __future__ import annotations

import math

import numpy as np

#: P:290 — Re = 1600, Pr = 0.71, M = 0.1, gamma = 1.4
TGV_PHYS = dict(Re=1600.0, Pr=0.71, Minf=0.1, gamma=1.4)

_MASK64 = (1 << 64) - 1


def splitmix64(counter: int) -> int:
    """Counter-based splitmix64 (Steele et al. 2014): uint64 -> uint64."""
    z = (counter + 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def _uniform(seed: int, counter: int) -> float:
    """Uniform double in [-1, 1) from (seed, counter)."""
    return (splitmix64((seed * 0x100000001B3 + counter) & _MASK64) >> 11) * (2.0 / (1 << 53)) - 1.0


def _coords(nx, ny, nz, dx):
    x = np.arange(nx) * dx
    y = np.arange(ny) * dx
    z = np.arange(nz) * dx
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return X, Y, Z


def conservative(rho, u0, u1, u2, p, gamma):
    """(rho, u, p) -> Q = (rho, rho u_i, rho E), rho E = p/(gamma-1) + 1/2 rho u_j u_j."""
    e = p / (gamma - 1.0) + 0.5 * rho * (u0 * u0 + u1 * u1 + u2 * u2)
    return np.ascontiguousarray(np.stack([rho, rho * u0, rho * u1, rho * u2, e]), dtype=np.float64)


def tgv(nx, ny, nz, dx=None, gamma=1.4, Minf=0.1):
    """Taylor-Green vortex initial state, eqs. (13)-(16), L = 1.

    T = 1 everywhere and rho = gamma M^2 p from the EOS (reading D-2).
    """
    if dx is None:
        dx = 2.0 * math.pi / nx
    X, Y, Z = _coords(nx, ny, nz, dx)
    u0 = np.sin(X) * np.cos(Y) * np.cos(Z)
    u1 = -np.cos(X) * np.sin(Y) * np.cos(Z)
    u2 = np.zeros_like(X)
    p = 1.0 / (gamma * Minf ** 2) + (np.cos(2 * X) + np.cos(2 * Y)) * (2.0 + np.cos(2 * Z)) / 16.0
    rho = gamma * Minf ** 2 * p
    return conservative(rho, u0, u1, u2, p, gamma)


def tgv_dt(n: int) -> float:
    """dt = 3.385e-3 at 64^3, halved each time the resolution doubles."""
    return 3.385e-3 * 64.0 / n


def perturbed_tgv(nx, ny, nz, dx=None, seed=1609012770, amp=1e-3, kmax=4, gamma=1.4, Minf=0.1):
    """TGV-like state on an arbitrary (anisotropic) periodic box plus a seeded
    low-pass perturbation of every primitive field (breaks the TGV symmetries).

    Base flow uses the box periods L_i = N_i dx so that every field is smooth
    and periodic for any N_i; perturbation modes have integer wavenumbers
    |k_i| <= kmax on the box, with coefficients from splitmix64(seed, counter).
    """
    if dx is None:
        dx = 2.0 * math.pi / max(nx, ny, nz)
    X, Y, Z = _coords(nx, ny, nz, dx)
    Lx, Ly, Lz = nx * dx, ny * dx, nz * dx
    ax, ay, az = 2 * math.pi * X / Lx, 2 * math.pi * Y / Ly, 2 * math.pi * Z / Lz
    base_u0 = np.sin(ax) * np.cos(ay) * np.cos(az)
    base_u1 = -np.cos(ax) * np.sin(ay) * np.cos(az)
    base_u2 = np.zeros_like(X)
    base_p = 1.0 / (gamma * Minf ** 2) + (np.cos(2 * ax) + np.cos(2 * ay)) * (2.0 + np.cos(2 * az)) / 16.0
    scale = [1.0, 1.0, 1.0, 1.0, 1.0 / (gamma * Minf ** 2)]  # rho, u0, u1, u2, p
    fields = [gamma * Minf ** 2 * base_p, base_u0, base_u1, base_u2, base_p]
    # the perturbation sum_k ca cos(k.a) + cb sin(k.a) = Re sum_k (ca - i cb) e^{i k.a},
    # evaluated separably (1D exponentials per direction, then two small
    # contractions), so that full-size grids (256^3) are generated in seconds
    ex = np.exp(1j * np.outer(np.arange(0, kmax + 1), 2 * math.pi * np.arange(nx) / nx))
    ks = np.arange(-kmax, kmax + 1)
    ey = np.exp(1j * np.outer(ks, 2 * math.pi * np.arange(ny) / ny))
    ez = np.exp(1j * np.outer(ks, 2 * math.pi * np.arange(nz) / nz))
    ctr = 0
    for f in range(5):
        C = np.zeros((len(ks), len(ks), kmax + 1), dtype=complex)  # [kz][ky][kx]
        for kx in range(0, kmax + 1):
            for ky in range(-kmax, kmax + 1):
                for kz in range(-kmax, kmax + 1):
                    if kx * kx + ky * ky + kz * kz > kmax * kmax:
                        continue
                    ca = _uniform(seed, ctr)
                    cb = _uniform(seed, ctr + 1)
                    ctr += 2
                    C[kz + kmax, ky + kmax, kx] = ca - 1j * cb
        A = C @ ex                                   # [kz][ky][x]
        B = np.einsum("ay,zax->zyx", ey, A)          # [kz][y][x]
        pert = np.real(np.tensordot(ez.T, B, axes=(1, 0)))  # [z][y][x]
        pert /= max(np.max(np.abs(pert)), 1e-300)
        fields[f] = fields[f] + amp * scale[f] * pert
    rho, u0, u1, u2, p = fields
    return conservative(rho, u0, u1, u2, p, gamma)


def entropy_wave(nx, ny=1, nz=1, dx=None, A=0.5, k=1, U=0.5, p0=None, gamma=1.4, Minf=0.1,
                 direction=0):
    """rho = 1 + A sin(2 pi k x / L), u = U e_dir, p = p0 (uniform).  An exact
    linear solution of the inviscid equations (advected density)."""
    n = (nx, ny, nz)
    if dx is None:
        dx = 1.0 / n[direction]
    X, Y, Z = _coords(nx, ny, nz, dx)
    C = (X, Y, Z)[direction]
    L = n[direction] * dx
    rho = 1.0 + A * np.sin(2 * math.pi * k * C / L)
    if p0 is None:
        p0 = 1.0 / (gamma * Minf ** 2)
    u = [np.zeros_like(X) for _ in range(3)]
    u[direction] = U * np.ones_like(X)
    p = p0 * np.ones_like(X)
    return conservative(rho, u[0], u[1], u[2], p, gamma)


def mms_primitives(x, y, z, M, gamma=1.4, Minf=0.1):
    """Smooth periodic manufactured primitive state on [0, 2pi)^3 (SURVEY §8(c) pins).

    Written against a math namespace M (numpy, or oracle.jets) providing
    sin/cos, so the same formula yields grid values and exact Taylor jets.
    """
    rho = 1.0 + 0.1 * M.sin(x) * M.cos(2.0 * y) * M.sin(z + 0.3)
    u0 = 0.5 * M.sin(x + y) * M.cos(z)
    u1 = (1.0 / 3.0) * M.cos(2.0 * x) * M.sin(z)
    u2 = 0.25 * M.sin(y) * M.cos(x - z)
    p = 1.0 / (gamma * Minf ** 2) + 0.2 * M.cos(x) * M.sin(y + 2.0 * z)
    return rho, u0, u1, u2, p


def mms_state(n, gamma=1.4, Minf=0.1):
    dx = 2.0 * math.pi / n
    X, Y, Z = _coords(n, n, n, dx)
    rho, u0, u1, u2, p = mms_primitives(X, Y, Z, np, gamma, Minf)
    return conservative(rho, u0, u1, u2, p, gamma)


def uniform_state(nx, ny, nz, rho=1.0, u=(0.3, -0.2, 0.1), p=71.4, gamma=1.4):
    o = np.ones((nz, ny, nx))
    return conservative(rho * o, u[0] * o, u[1] * o, u[2] * o, p * o, gamma)
