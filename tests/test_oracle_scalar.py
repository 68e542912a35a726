"""Pins for the oracle's scalar advection-diffusion (the paper's verification
equations) — closed forms, no GPU."""
from __future__ import annotations

import json
import math
import os
from fractions import Fraction
from math import factorial

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")


def kappas(order, theta):
    """kappa1(theta) = 2 sum a_k sin(k theta); kappa2(theta) = -(b0 + 2 sum b_k cos(k theta)),
    from the closed-form weights."""
    m = order // 2
    a = [Fraction((-1) ** (k + 1) * factorial(m) ** 2, k * factorial(m - k) * factorial(m + k))
         for k in range(1, m + 1)]
    b = [Fraction(2 * (-1) ** (k + 1) * factorial(m) ** 2,
                  k * k * factorial(m - k) * factorial(m + k)) for k in range(1, m + 1)]
    b0 = -2 * sum(b)
    k1 = 2 * sum(float(a[k - 1]) * np.sin(k * theta) for k in range(1, m + 1))
    k2 = -(float(b0) + 2 * sum(float(b[k - 1]) * np.cos(k * theta) for k in range(1, m + 1)))
    return k1, k2


def lam_h(order, kvec, u, kd, dx):
    """Discrete operator multiplier on exp(i k.x): -i sum u_j kappa1/dx - kd sum kappa2/dx^2."""
    s = 0j
    for kj, uj in zip(kvec, u):
        k1, k2 = kappas(order, kj * dx)
        s += -1j * uj * k1 / dx - kd * k2 / dx ** 2
    return s


@pytest.mark.parametrize("scheme", [0, 1, 2])
@pytest.mark.parametrize("direction", [0, 1, 2])
def test_scalar_amplification_closed_form(oracle_lib, scheme, direction):
    """phi = sin(k x_d + 0.3): phi_n = Im(P(z)^n e^{i(k x_d + 0.3)}), z = dt lambda_h(k)."""
    n = [12, 10, 9]
    n[direction] = 32
    dx, order, kw = 0.2, 8, 3
    L = n[direction] * dx
    kk = 2 * math.pi * kw / L
    u = [0.0, 0.0, 0.0]
    u[direction] = 0.7
    kd = 0.05
    dt = 0.01
    p = oracle_lib.OracleParams(*n, order, dx, dt=dt)
    C = np.arange(n[direction]) * dx
    shape = (n[2], n[1], n[0])
    phase = np.zeros(shape)
    idx = [None, None, None]
    idx[2 - direction] = slice(None)
    phase = phase + (kk * C + 0.3)[tuple(idx)]
    phi0 = np.sin(phase)
    nsteps = 25
    out = oracle_lib.scalar_step(p, u, kd, phi0, scheme, nsteps)
    kvec = [0.0, 0.0, 0.0]
    kvec[direction] = kk
    z = dt * lam_h(order, kvec, u, kd, dx)
    P = 1 + z if scheme == 0 else 1 + z + z * z / 2 + z ** 3 / 6
    exact = np.imag(P ** nsteps * np.exp(1j * phase))
    assert np.max(np.abs(out - exact)) < 1e-13


def test_paper_wave_scalar(oracle_lib):
    """c = 0.5, dx = 1e-3 on [0,1), 8th order, RK3, dt = 4e-4, t = 1: error O(1e-10)."""
    g = json.load(open(GOLDEN))["wave_1d"]
    nx = int(round(g["L"] / g["dx"]))
    p = oracle_lib.OracleParams(nx, 1, 1, g["order"], g["dx"], dt=g["dt"])
    x = np.arange(nx) * g["dx"]
    phi0 = np.sin(2 * math.pi * x)[None, None, :]
    nsteps = int(round(g["t_final"] / g["dt"]))
    out = oracle_lib.scalar_step(p, (g["c"], 0, 0), 0.0, phi0, 1, nsteps)
    err = np.max(np.abs(out[0, 0] - np.sin(2 * math.pi * (x - g["c"] * g["t_final"]))))
    assert 0.1 * g["error_order_of_magnitude"] < err < 10 * g["error_order_of_magnitude"], err


# --- the paper's 2D manufactured solution: k = 0.75, u = (1, -0.5),
#     phi_m = sin x0 cos x1 on [0, 2pi)^2, S from substituting phi_m
MMS_U, MMS_K = (1.0, -0.5, 0.0), 0.75
# P:207 bounds the Courant number by 0.025; at 12th order on dx = pi/32 RK3's
# diffusion-number limit needs <= 0.023, so the study runs at 0.02 (D-23)
MMS_COURANT = 0.02


def mms_fields(n):
    dx = 2 * math.pi / n
    x = np.arange(n) * dx
    Y, X = np.meshgrid(x, x, indexing="ij")
    phi_m = np.sin(X) * np.cos(Y)
    # d/dx_j(phi u_j) - k lap phi + S = 0  =>  S = -(u.grad phi_m) + k lap phi_m
    S = -(MMS_U[0] * np.cos(X) * np.cos(Y) - MMS_U[1] * np.sin(X) * np.sin(Y)) \
        + MMS_K * (-2.0 * np.sin(X) * np.cos(Y))
    return dx, X, Y, phi_m, S


def mms_discrete_steady(order, n):
    """Closed-form discrete steady state L_h phi_h = S = L phi_m, mode by mode:
    sin x cos y = 1/2 [sin(x+y) + sin(x-y)], phi_h = 1/2 sum Im((lambda/lambda_h) e^{i k.x})."""
    dx, X, Y, phi_m, _ = mms_fields(n)
    out = np.zeros_like(X)
    for kv in ((1.0, 1.0), (1.0, -1.0)):
        lam = -1j * (MMS_U[0] * kv[0] + MMS_U[1] * kv[1]) - MMS_K * (kv[0] ** 2 + kv[1] ** 2)
        lh = lam_h(order, (kv[0], kv[1], 0.0), MMS_U, MMS_K, dx)
        out += 0.5 * np.imag(lam / lh * np.exp(1j * (kv[0] * X + kv[1] * Y)))
    return out, phi_m


@pytest.mark.parametrize("order", [2, 4, 12])
@pytest.mark.parametrize("n", [4, 8, 16])
def test_paper_mms_oracle_reaches_discrete_steady_state(oracle_lib, order, n):
    """RK3 at Courant 0.02 (<= 0.025) to T = 100 ends on the closed-form discrete
    steady state."""
    dx, X, Y, phi_m, S = mms_fields(n)
    dt = MMS_COURANT * dx / max(abs(MMS_U[0]), abs(MMS_U[1]))
    nsteps = int(math.ceil(100.0 / dt))
    p = oracle_lib.OracleParams(n, n, 1, order, dx, dt=100.0 / nsteps)
    out = oracle_lib.scalar_step(p, MMS_U, MMS_K, np.zeros((1, n, n)), 1, nsteps, S=S[None])
    phi_h, _ = mms_discrete_steady(order, n)
    assert np.max(np.abs(out[0] - phi_h)) < 1e-12


def test_paper_mms_convergence_rates():
    """the steady error converges at the nominal order for orders 2..12 over
    dx = pi/2 .. pi/32; 12th order reaches machine precision ("anomaly").
    Pure closed form (pins the discretisation the oracle and the GPU both implement)."""
    ns = [4, 8, 16, 32, 64]
    for order in (2, 4, 6, 8, 10, 12):
        errs = []
        for n in ns:
            phi_h, phi_m = mms_discrete_steady(order, n)
            errs.append(math.sqrt(np.mean((phi_h - phi_m) ** 2)))
        use = [(n, e) for n, e in zip(ns, errs) if e > 1e-13]
        slopes = [math.log(e0 / e1) / math.log(n1 / n0) for (n0, e0), (n1, e1) in zip(use, use[1:])]
        assert abs(slopes[-1] - order) < 0.3, (order, errs, slopes)
    phi_h, phi_m = mms_discrete_steady(12, 64)
    assert math.sqrt(np.mean((phi_h - phi_m) ** 2)) < 1e-13
