"""Algorithmic work per grid point — the roofline numerators.

Bytes: the compulsory HBM traffic of one low-storage RK3 step
is 5 fields x fp64 over three field-sets: stage 1 reads Q, writes Q' and W
(120 B); stage 2 reads Q, W, writes Q', W (160 B); stage 3 reads Q, W, writes
Q' (120 B) — 400 B per point-step; forward Euler 80 B.

Our two-kernel stage adds an on-HBM hand-off between the z-pass and the
xy-pass: the z-pass writes W' = A W + dt Rz (the low-storage register with
the z-part of the residual folded in) and g_i2 = D_z u_i (3 doubles); the
xy-pass reads them.  `kernel_bytes` gives each kernel's own algorithmic
traffic in this design (every operand read once and every result written
once; halo re-reads are not counted, they should hit L2).

FP64 flops (FMA = 2): counted from the discrete operators, one evaluation per
point (no halo recomputation):
  first derivative, m taps: m subtractions + m FMAs        = 3m
  second derivative (exact-cancellation form)               = 5m
  pointwise formulas (primitives, fluxes, assembly, update) = constants below.
"""
from __future__ import annotations

COMPULSORY_BYTES_RK3 = 400.0
COMPULSORY_BYTES_EULER = 80.0


def kernel_bytes(stage: int, scheme: int = 1):
    """(zpass_bytes, xypass_bytes) per point for RK3 stage 0/1/2 (Euler: stage 0, scheme 0).

    scheme 2 (two-register RK3): the z-pass never reads the register (it writes
    dt Rz into the destination buffer), the xy-pass reads Q_old instead."""
    read_w = scheme in (1, 2) and stage > 0
    write_w = scheme in (1, 2) and stage < 2
    if scheme == 2:
        z = 40.0 + 40.0 + 24.0  # read Q; write dt Rz, g_i2
        xy = 40.0 + 24.0 + 40.0 + (40.0 if read_w else 0.0) + 40.0 + (40.0 if write_w else 0.0)
        return z, xy
    z = 40.0 + (40.0 if read_w else 0.0) + 40.0 + 24.0  # read Q (and W); write W', g_i2
    xy = 40.0 + 24.0 + 40.0 + 40.0 + (40.0 if write_w else 0.0)  # read Q, g, W'; write Q' (and W)
    return z, xy


def step_kernel_bytes(scheme: int = 1):
    st = 1 if scheme == 0 else 3
    zs = sum(kernel_bytes(s, scheme)[0] for s in range(st))
    xs = sum(kernel_bytes(s, scheme)[1] for s in range(st))
    return zs, xs


def flops(m: int):
    """(zpass_flops, xypass_flops) per point per stage."""
    d1, d2 = 3 * m, 5 * m
    # z-pass: D_z of u_i(3), rho, m_i, e (5), F_i2 (3), G_2 -> 12 first; D_zz u_i, T -> 4 second
    z = 12 * d1 + 4 * d2 + 14 + 10 + 40
    # xy-pass: 32 first derivatives (incl. 6 mixed), 8 second, primitives 14,
    # flux products ~20, assembly incl. dissipation ~70, stage update 20
    xy = 32 * d1 + 8 * d2 + 14 + 20 + 70 + 20
    return float(z), float(xy)
