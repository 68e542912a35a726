"""ctypes wrapper around oracle/liboracle.so (TEST INFRASTRUCTURE ONLY).

Argument marshalling only; every number is computed in ``oracle.cpp``.
Arrays use the ABI layout ``[5][nz][ny][nx]`` (x fastest), fp64.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with strict IEEE evaluation (no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17",
             "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


class _CParams(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("order", ctypes.c_int), ("dx", ctypes.c_double), ("dt", ctypes.c_double),
                ("Re", ctypes.c_double), ("Pr", ctypes.c_double), ("Minf", ctypes.c_double),
                ("gamma", ctypes.c_double), ("sym", ctypes.c_int * 3),
                ("energy_form", ctypes.c_int), ("visc_law", ctypes.c_int),
                ("suth", ctypes.c_double)]


@dataclass
class OracleParams:
    nx: int
    ny: int
    nz: int
    order: int
    dx: float
    dt: float = 0.0
    Re: float = 1600.0
    Pr: float = 0.71
    Minf: float = 0.1
    gamma: float = 1.4
    sym: tuple = (0, 0, 0)  # 1: symmetry boundaries in x, y, z; 0: periodic
    energy_form: int = 0    # 0: expanded viscous work (D-5); 1: conservative (D-27)
    visc_law: int = 0       # 0: mu = 1 (D-3); 1: Sutherland mu(T) (D-26)
    suth: float = 0.0       # Sutherland S / T_ref

    def c(self) -> _CParams:
        return _CParams(self.nx, self.ny, self.nz, self.order, self.dx, self.dt,
                        self.Re, self.Pr, self.Minf, self.gamma, (ctypes.c_int * 3)(*self.sym),
                        self.energy_form, self.visc_law, self.suth)

    @property
    def shape(self):
        return (5, self.nz, self.ny, self.nx)


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER(_CParams)
        dp = ctypes.POINTER(ctypes.c_double)
        llp = ctypes.POINTER(ctypes.c_longlong)
        _lib.oracle_weights_exact.argtypes = [ctypes.c_int, llp, llp, llp, llp]
        _lib.oracle_derivative.argtypes = [P, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
        _lib.oracle_residual.argtypes = [P, dp, dp]
        _lib.oracle_step.argtypes = [P, dp, ctypes.c_int, ctypes.c_int]
        _lib.oracle_diagnostics.argtypes = [P, dp, dp]
        _lib.oracle_run_series.argtypes = [P, dp, ctypes.c_int, ctypes.c_int, dp]
        _lib.oracle_scalar_residual.argtypes = [P, dp, ctypes.c_double, dp, dp, dp]
        _lib.oracle_scalar_step.argtypes = [P, dp, ctypes.c_double, dp, dp, ctypes.c_int,
                                            ctypes.c_int]
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def weights_exact(order: int):
    """(a_1..a_m, b_0..b_m) as Fractions, solved exactly from the moment conditions."""
    m = order // 2
    an = (ctypes.c_longlong * max(m, 1))()
    ad = (ctypes.c_longlong * max(m, 1))()
    bn = (ctypes.c_longlong * (m + 1))()
    bd = (ctypes.c_longlong * (m + 1))()
    if _L().oracle_weights_exact(order, an, ad, bn, bd) != 0:
        raise ValueError(f"invalid order {order}")
    return ([Fraction(an[k], ad[k]) for k in range(m)],
            [Fraction(bn[k], bd[k]) for k in range(m + 1)])


def derivative(p: OracleParams, f: np.ndarray, kind: int, direction: int, direction2: int = 0):
    """kind 1: D_dir f, 2: D_dir,dir f, 3: D_dir(D_dir2 f).  f is [nz][ny][nx]."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.empty_like(f)
    if _L().oracle_derivative(ctypes.byref(p.c()), _dp(f), kind, direction, direction2, _dp(out)):
        raise ValueError("bad derivative arguments")
    return out


def residual(p: OracleParams, Q: np.ndarray) -> np.ndarray:
    Q = np.ascontiguousarray(Q, dtype=np.float64).reshape(p.shape)
    R = np.empty_like(Q)
    if _L().oracle_residual(ctypes.byref(p.c()), _dp(Q), _dp(R)):
        raise ValueError("bad residual arguments")
    return R


def step(p: OracleParams, Q: np.ndarray, scheme: int, nsteps: int) -> np.ndarray:
    """Return Q advanced by nsteps (scheme 0 = Euler, 1 = RK3 2N, 2 = RK3 two-register);
    input untouched."""
    Qn = np.array(Q, dtype=np.float64, order="C").reshape(p.shape).copy()
    if _L().oracle_step(ctypes.byref(p.c()), _dp(Qn), scheme, nsteps):
        raise ValueError("bad step arguments")
    return Qn


def diagnostics(p: OracleParams, Q: np.ndarray):
    """(E_k, enstrophy, dissipation) — means over the grid points."""
    Q = np.ascontiguousarray(Q, dtype=np.float64).reshape(p.shape)
    out = np.zeros(3)
    if _L().oracle_diagnostics(ctypes.byref(p.c()), _dp(Q), _dp(out)):
        raise ValueError("bad diagnostics arguments")
    return tuple(float(v) for v in out)


def run_series(p: OracleParams, Q: np.ndarray, scheme: int, nsteps: int):
    """Diagnostics at steps 0..nsteps -> array [nsteps+1, 3]; returns (series, Q_final)."""
    Qn = np.array(Q, dtype=np.float64, order="C").reshape(p.shape).copy()
    series = np.zeros((nsteps + 1, 3))
    if _L().oracle_run_series(ctypes.byref(p.c()), _dp(Qn), scheme, nsteps, _dp(series)):
        raise ValueError("bad run_series arguments")
    return series, Qn


def _u3(u):
    return (ctypes.c_double * 3)(*[float(v) for v in u])


def scalar_residual(p: OracleParams, u, k: float, phi: np.ndarray, S=None) -> np.ndarray:
    """R = -d/dx_j(phi u_j) + k d2 phi/dx_j^2 - S for phi [nz][ny][nx]."""
    phi = np.ascontiguousarray(phi, dtype=np.float64).reshape(p.nz, p.ny, p.nx)
    Sc = None if S is None else np.ascontiguousarray(S, dtype=np.float64).reshape(phi.shape)
    Sp = None if Sc is None else _dp(Sc)
    R = np.empty_like(phi)
    if _L().oracle_scalar_residual(ctypes.byref(p.c()), _u3(u), float(k), _dp(phi), Sp, _dp(R)):
        raise ValueError("bad scalar residual arguments")
    return R


def scalar_step(p: OracleParams, u, k: float, phi: np.ndarray, scheme: int, nsteps: int, S=None):
    """phi advanced by nsteps (0 = Euler, 1 = RK3 2N, 2 = RK3 two-register); input untouched."""
    ph = np.array(phi, dtype=np.float64, order="C").reshape(p.nz, p.ny, p.nx).copy()
    Sc = None if S is None else np.ascontiguousarray(S, dtype=np.float64).reshape(ph.shape)
    Sp = None if Sc is None else _dp(Sc)
    if _L().oracle_scalar_step(ctypes.byref(p.c()), _u3(u), float(k), Sp, _dp(ph), scheme, nsteps):
        raise ValueError("bad scalar step arguments")
    return ph


def is_inviscid(Re: float) -> bool:
    return math.isinf(Re)
