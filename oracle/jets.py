"""Second-order Taylor jets and the exact continuous residual (TEST INFRASTRUCTURE ONLY).

A jet carries (value, gradient, Hessian) of a smooth field at every grid point,
propagated exactly through +, -, *, /, sqrt, sin, cos by the product / quotient /
chain rules.  ``exact_residual`` evaluates the right-hand side of the paper's
compressible Navier-Stokes equations (5)-(9) with the EOS and total
energy in conservative divergence form for a manufactured state —
the continuous operator the discrete oracle must converge to at its nominal
order (the method of manufactured solutions).  The skew-symmetric
form equals the divergence form in the continuum, so this is an
independent check of the oracle's skew splitting, expansion and signs.
"""
from __future__ import annotations

import math

import numpy as np


class Jet:
    __slots__ = ("v", "g", "h")

    def __init__(self, v, g, h):
        self.v = v  # [...]
        self.g = g  # [3, ...]
        self.h = h  # [3, 3, ...]

    @staticmethod
    def const(c, like):
        z = np.zeros_like(like.v)
        return Jet(z + c, np.zeros_like(like.g), np.zeros_like(like.h))

    def _lift(self, o):
        return o if isinstance(o, Jet) else Jet.const(o, self)

    def __add__(self, o):
        o = self._lift(o)
        return Jet(self.v + o.v, self.g + o.g, self.h + o.h)

    __radd__ = __add__

    def __neg__(self):
        return Jet(-self.v, -self.g, -self.h)

    def __sub__(self, o):
        return self + (-self._lift(o))

    def __rsub__(self, o):
        return self._lift(o) - self

    def __mul__(self, o):
        if not isinstance(o, Jet):
            return Jet(self.v * o, self.g * o, self.h * o)
        v = self.v * o.v
        g = self.g * o.v + self.v * o.g
        h = (self.h * o.v + o.h * self.v
             + np.einsum("i...,j...->ij...", self.g, o.g)
             + np.einsum("i...,j...->ij...", o.g, self.g))
        return Jet(v, g, h)

    __rmul__ = __mul__

    def recip(self):
        r = 1.0 / self.v
        g = -self.g * r * r
        h = -self.h * r * r + 2.0 * np.einsum("i...,j...->ij...", self.g, self.g) * r ** 3
        return Jet(r, g, h)

    def __truediv__(self, o):
        if not isinstance(o, Jet):
            return self * (1.0 / o)
        return self * o.recip()

    def __rtruediv__(self, o):
        return self.recip() * o

    def sqrt(self):
        """s = sqrt(a) from the product rule applied to s * s = a (no power-law
        calculus): s.g = a.g / (2 s), s.h = (a.h - 2 s.g (x) s.g) / (2 s)."""
        s = np.sqrt(self.v)
        g = self.g / (2.0 * s)
        h = (self.h - 2.0 * np.einsum("i...,j...->ij...", g, g)) / (2.0 * s)
        return Jet(s, g, h)


def _fn(a: Jet, f, df, d2f):
    v = f(a.v)
    d1 = df(a.v)
    d2 = d2f(a.v)
    return Jet(v, a.g * d1, a.h * d1 + np.einsum("i...,j...->ij...", a.g, a.g) * d2)


class _JetMath:
    @staticmethod
    def sin(a):
        if not isinstance(a, Jet):
            return math.sin(a)
        return _fn(a, np.sin, np.cos, lambda x: -np.sin(x))

    @staticmethod
    def cos(a):
        if not isinstance(a, Jet):
            return math.cos(a)
        return _fn(a, np.cos, lambda x: -np.sin(x), lambda x: -np.cos(x))


M = _JetMath()


def coordinate_jets(X, Y, Z):
    out = []
    for d, C in enumerate((X, Y, Z)):
        g = np.zeros((3,) + C.shape)
        g[d] = 1.0
        out.append(Jet(C.astype(np.float64), g, np.zeros((3, 3) + C.shape)))
    return out


def exact_residual(prim_fn, X, Y, Z, Re, Pr, Minf, gamma, suth=None):
    """Exact dQ/dt of eqs. (5)-(7) for the primitive state prim_fn(x, y, z, M).

    Returns [5, ...] (rho, rho u_i, rho E).  mu == 1 (reading D-3), or, with
    ``suth`` = S/T_ref, Sutherland's mu(T) = T^1.5 (1 + S)/(T + S) (D-26): only
    mu and its first derivatives enter, d mu/dx_j = mu'(T) dT/dx_j exactly.
    """
    x, y, z = coordinate_jets(X, Y, Z)
    rho, u0, u1, u2, p = prim_fn(x, y, z, M)
    u = [u0, u1, u2]
    nu = 0.0 if math.isinf(Re) else 1.0 / Re
    kap = 0.0 if math.isinf(Re) else 1.0 / ((gamma - 1.0) * Minf ** 2 * Pr * Re)
    m = [rho * u[i] for i in range(3)]
    E = p * (1.0 / (gamma - 1.0)) + 0.5 * rho * (u0 * u0 + u1 * u1 + u2 * u2)  # rho E
    T = p * (gamma * Minf ** 2) / rho  # EOS (10)
    G = [[u[i].g[j] for j in range(3)] for i in range(3)]  # du_i/dx_j
    div = G[0][0] + G[1][1] + G[2][2]
    if suth is None:
        mu, dmu = np.ones_like(T.v), [np.zeros_like(T.v)] * 3
    else:
        # mu(T) evaluated on the temperature jet: its gradient d mu/dx_j comes
        # from the product, quotient and square-root rules, not from a retyped
        # closed form of mu'(T)
        muj = T * T.sqrt() * (1.0 + suth) / (T + suth)
        mu = muj.v
        dmu = [muj.g[j] for j in range(3)]
    S = [[G[i][j] + G[j][i] - (2.0 / 3.0 * div if i == j else 0.0) for j in range(3)]
         for i in range(3)]
    tau = [[nu * mu * S[i][j] for j in range(3)] for i in range(3)]
    # d tau_ij / dx_j = nu (mu (lap u_i + 1/3 d_i div) + d_j mu S_ij)  (continuous identity)
    dtau = []
    for i in range(3):
        lap = sum(u[i].h[j, j] for j in range(3))
        ddiv = sum(u[k].h[i, k] for k in range(3))
        dtau.append(nu * (mu * (lap + ddiv / 3.0) + sum(dmu[j] * S[i][j] for j in range(3))))
    R = np.zeros((5,) + X.shape)
    R[0] = -sum(m[j].g[j] for j in range(3))
    for i in range(3):
        conv = sum((m[i] * u[j]).g[j] for j in range(3))
        R[1 + i] = -conv - p.g[i] + dtau[i]
    conv_e = sum(((E + p) * u[j]).g[j] for j in range(3))
    heat = kap * sum(mu * T.h[j, j] + dmu[j] * T.g[j] for j in range(3))
    # d/dx_j (u_i tau_ij) = tau_ij du_i/dx_j + u_i d tau_ij/dx_j
    visc_work = (sum(tau[i][j] * G[i][j] for i in range(3) for j in range(3))
                 + sum(u[i].v * dtau[i] for i in range(3)))
    R[4] = -conv_e + heat + visc_work
    return R
