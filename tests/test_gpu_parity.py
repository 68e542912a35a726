"""GPU <-> oracle parity through the C ABI (B200).  Every test here needs a GPU.

Metric (D-14, BASELINE north star): per conservative field f,
max_pts |gpu - oracle| / max_pts |oracle|  <= 1e-11.  Inputs are seeded and
synthetic (inputs/), identical on both sides.
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from inputs import (TGV_PHYS, entropy_wave, perturbed_tgv, tgv, tgv_dt, uniform_state)

pytestmark = pytest.mark.gpu

TOL = 1e-11


def relerr(a, b):
    a = np.asarray(a).reshape(5, -1)
    b = np.asarray(b).reshape(5, -1)
    return np.array([np.max(np.abs(a[f] - b[f])) / max(np.max(np.abs(b[f])), 1e-300)
                     for f in range(5)])


@pytest.fixture(scope="module")
def osbli():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_1609_01277_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def orc(oracle_lib):
    return oracle_lib


def make(osbli, shape, order, dx, dt, scheme=1, **phys):
    nx, ny, nz = shape
    ph = dict(TGV_PHYS)
    ph.update(phys)
    return osbli.Solver(nx, ny, nz, order, dx, dt, scheme=scheme, **ph)


# ---------------------------------------------------------------- residual
@pytest.mark.parametrize("order", [2, 4, 6, 8, 10, 12])
@pytest.mark.parametrize("shape", [(40, 36, 33), (13, 11, 9)])
def test_residual_parity_all_orders(osbli, orc, order, shape):
    dx = 2 * math.pi / max(shape)
    Q = perturbed_tgv(*shape, dx=dx, amp=0.02)
    s = make(osbli, shape, order, dx, 1e-3)
    s.set_state(Q)
    R = s.residual()
    Ro = orc.residual(orc.OracleParams(*shape, order, dx, **TGV_PHYS), Q)
    e = relerr(R, Ro)
    assert np.all(e < TOL), e


@pytest.mark.parametrize("order", [4, 12])
def test_residual_parity_inviscid(osbli, orc, order):
    shape = (24, 20, 16)
    dx = 2 * math.pi / 24
    Q = perturbed_tgv(*shape, dx=dx, amp=0.05)
    s = make(osbli, shape, order, dx, 1e-3, Re=math.inf)
    s.set_state(Q)
    Ro = orc.residual(orc.OracleParams(*shape, order, dx, Re=math.inf, Pr=0.71, Minf=0.1,
                                       gamma=1.4), Q)
    assert np.all(relerr(s.residual(), Ro) < TOL)


def test_uniform_state_exact_equilibrium_gpu(osbli):
    s = make(osbli, (17, 9, 11), 12, 0.3, 1e-3)
    s.set_state(uniform_state(17, 9, 11))
    assert np.all(s.residual() == 0.0)
    q0 = s.get_state()
    s.step(3)
    assert np.array_equal(s.get_state(), q0)


# ---------------------------------------------------------------- time stepping
def test_tgv32_o4_rk3_10_steps(osbli, orc):
    """BASELINE configs[0]: TGV 32^3, 4th order, RK3, Re=1600, M=0.1, 10 steps."""
    n = 32
    dx, dt = 2 * math.pi / n, tgv_dt(n)
    Q = tgv(n, n, n)
    s = make(osbli, (n, n, n), 4, dx, dt)
    s.set_state(Q)
    s.step(10)
    Qo = orc.step(orc.OracleParams(n, n, n, 4, dx, dt=dt, **TGV_PHYS), Q, 1, 10)
    e = relerr(s.get_state(), Qo)
    assert np.all(e < TOL), e
    d = s.diagnostics()
    do = orc.diagnostics(orc.OracleParams(n, n, n, 4, dx, **TGV_PHYS), Qo)
    assert abs(d.kinetic_energy - do[0]) / do[0] < 1e-12
    assert abs(d.enstrophy - do[1]) / do[1] < 1e-12
    assert abs(d.dissipation - do[2]) / do[2] < 1e-12
    assert d.step == 10 and abs(d.t - 10 * dt) < 1e-15


@pytest.mark.parametrize("order", [2, 4, 6, 8, 10, 12])
def test_anisotropic_perturbed_rk3_10_steps(osbli, orc, order):
    """SURVEY §8(d) cfg 1 companion: anisotropic 40x36x32 TGV + seeded perturbation."""
    shape = (40, 36, 32)
    dx = 2 * math.pi / 32
    dt = 0.25 * dx / (1.0 / 0.1 + 1.0)
    Q = perturbed_tgv(*shape, dx=dx, amp=1e-3)
    s = make(osbli, shape, order, dx, dt)
    s.set_state(Q)
    s.step(10)
    Qo = orc.step(orc.OracleParams(*shape, order, dx, dt=dt, **TGV_PHYS), Q, 1, 10)
    e = relerr(s.get_state(), Qo)
    assert np.all(e < TOL), e


@pytest.mark.parametrize("order", [4, 12])
def test_euler_parity(osbli, orc, order):
    shape = (24, 20, 16)
    dx = 2 * math.pi / 24
    dt = 2e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.02)
    s = make(osbli, shape, order, dx, dt, scheme=0)
    s.set_state(Q)
    s.step(3)
    Qo = orc.step(orc.OracleParams(*shape, order, dx, dt=dt, **TGV_PHYS), Q, 0, 3)
    assert np.all(relerr(s.get_state(), Qo) < TOL)


@pytest.mark.parametrize("shape,order", [((1, 1, 64), 8), ((64, 1, 1), 8), ((1, 48, 1), 12),
                                         ((5, 4, 3), 12), ((3, 7, 2), 4), ((33, 9, 65), 6)])
def test_degenerate_and_ragged_grids(osbli, orc, shape, order):
    """1D/2D problems, grids smaller than the stencil (multiple periodic wraps),
    ragged tiles in every direction."""
    dx = 0.37
    dt = 1e-3
    rng_state = perturbed_tgv(*shape, dx=dx, amp=0.05, kmax=2)
    s = make(osbli, shape, order, dx, dt)
    s.set_state(rng_state)
    s.step(2)
    Qo = orc.step(orc.OracleParams(*shape, order, dx, dt=dt, **TGV_PHYS), rng_state, 1, 2)
    Qg = s.get_state()
    for f in range(5):
        scale = max(np.max(np.abs(Qo[f])), 1.0)
        assert np.max(np.abs(Qg[f] - Qo[f])) / scale < TOL


def test_entropy_wave_closed_form_gpu(osbli):
    """Inviscid entropy wave: rho_n = 1 + A Im(P(z)^n e^{ikx})."""
    nx, A, U, kw, order = 64, 0.3, 0.7, 3, 8
    dx = 1.0 / nx
    dt = 0.2 * dx
    Q = entropy_wave(nx, 4, 4, dx=dx, A=A, k=kw, U=U, Minf=1.0)
    s = osbli.Solver(nx, 4, 4, order, dx, dt, Re=math.inf, Pr=0.71, Minf=1.0, gamma=1.4)
    s.set_state(Q)
    s.step(50)
    m = order // 2
    from fractions import Fraction
    from math import factorial
    a = [Fraction((-1) ** (k + 1) * factorial(m) ** 2, k * factorial(m - k) * factorial(m + k))
         for k in range(1, m + 1)]
    kk = 2 * math.pi * kw
    kap = 2 * sum(float(a[k - 1]) * math.sin(k * kk * dx) for k in range(1, m + 1))
    z = -1j * U * dt * kap / dx
    P = 1 + z + z * z / 2 + z ** 3 / 6
    exact = 1 + A * np.imag(P ** 50 * np.exp(1j * kk * np.arange(nx) * dx))
    Qg = s.get_state()
    assert np.max(np.abs(Qg[0] - exact[None, None, :])) < 1e-13


def test_nonfinite_detected(osbli):
    shape = (16, 8, 8)
    Q = uniform_state(*shape)
    Q[0, 3, 4, 5] = 0.0  # rho = 0 -> division by zero
    s = make(osbli, shape, 4, 0.1, 1e-3)
    s.set_state(Q)
    s.step(1)
    with pytest.raises(osbli.OsbliError) as ei:
        s.sync()
    assert ei.value.status == "E_NONFINITE"
    with pytest.raises(osbli.OsbliError) as ei:
        s.step(1)
    assert ei.value.status == "E_STATE"


def test_device_pointer_state_io(osbli, orc):
    import torch
    shape = (24, 20, 16)
    dx = 2 * math.pi / 24
    Q = perturbed_tgv(*shape, dx=dx, amp=0.02)
    s = make(osbli, shape, 8, dx, 1e-3)
    s.set_stream(torch.cuda.current_stream().cuda_stream)
    s.set_state(torch.from_numpy(Q).cuda())
    out = torch.empty((5,) + shape[::-1], dtype=torch.float64, device="cuda")
    s.get_state(out)
    assert np.array_equal(out.cpu().numpy(), Q)
    s.step(2)
    Qo = orc.step(orc.OracleParams(*shape, 8, dx, dt=1e-3, **TGV_PHYS), Q, 1, 2)
    s.get_state(out)
    assert np.all(relerr(out.cpu().numpy(), Qo) < TOL)


# ---------------------------------------------------------------- diagnostics series
def test_tgv64_series_vs_golden(osbli):
    """BASELINE configs[1]: TGV 64^3 o4 RK3 — E_k and dissipation series agree with
    the oracle's (tests/golden, written by tools/make_golden_series.py) to 1e-9."""
    path = os.path.join(os.path.dirname(__file__), "golden", "tgv64_o4_rk3_series.csv")
    if not os.path.exists(path):
        pytest.fail("golden series missing: run tools/make_golden_series.py")
    gold = np.loadtxt(path, delimiter=",", comments="#", skiprows=2)
    n, dt = 64, 3.385e-3
    s = make(osbli, (n, n, n), 4, 2 * math.pi / n, dt)
    s.set_state(tgv(n, n, n))
    worst = np.zeros(3)
    for row in gold:
        step = int(row[0])
        if step > 0:
            s.step(1)
        d = s.diagnostics()
        assert d.step == step
        got = np.array([d.kinetic_energy, d.enstrophy, d.dissipation])
        worst = np.maximum(worst, np.abs(got - row[2:5]) / np.abs(row[2:5]))
    assert worst[0] < 1e-9 and worst[2] < 1e-9, worst
    assert worst[1] < 1e-9, worst


# ---------------------------------------------------------------- full size, sampled
def _sample_points(n):
    edge = [0, 1, 31, 32, n // 2, n - 1]
    pts = [(edge[i % 6], edge[(i * 5 + 2) % 6], edge[(i * 7 + 3) % 6]) for i in range(8)]
    return pts


def test_full_size_256_o12_sampled(osbli, orc):
    """BASELINE configs[3] at full size in the bench launch configuration:
    TGV 256^3, 12th order, RK3, one step; oracle evaluated exactly at sampled
    points (oracle/windowed.py), plus the residual at the same points."""
    from oracle import windowed
    n, order = 256, 12
    dx, dt = 2 * math.pi / n, tgv_dt(n)
    Q = tgv(n, n, n)
    s = make(osbli, (n, n, n), order, dx, dt)
    s.set_state(Q)
    R = s.residual()
    pts = _sample_points(n)
    p = orc.OracleParams(n, n, n, order, dx, dt=dt, **TGV_PHYS)
    Ro = windowed.sample_residual(p, Q, pts)
    scale_r = np.max(np.abs(R.reshape(5, -1)), axis=1)
    for t, (i, j, k) in enumerate(pts):
        assert np.all(np.abs(R[:, k, j, i] - Ro[t]) / scale_r < TOL), (i, j, k)
    s.step(1)
    Qg = s.get_state()
    So = windowed.sample_step(p, Q, pts, 1, 1)
    scale = np.max(np.abs(Qg.reshape(5, -1)), axis=1)
    for t, (i, j, k) in enumerate(pts):
        assert np.all(np.abs(Qg[:, k, j, i] - So[t]) / scale < TOL), (i, j, k)
    # property at any size: discrete mass conservation
    assert abs(Qg[0].sum() - Q[0].sum()) / Q[0].sum() < 1e-13


# ---------------------------------------------------------------- N2(a): two-register RK3
@pytest.mark.parametrize("order,shape", [(4, (32, 32, 32)), (12, (40, 36, 33)), (8, (13, 11, 9))])
def test_two_register_rk3_parity(osbli, orc, order, shape):
    """OSBLI_RK3_2R (D-25) against the oracle's scheme 2, 10 steps, 1e-11."""
    dx = 2 * math.pi / max(shape)
    dt = 0.25 * dx / (1.0 / 0.1 + 1.0)
    Q = perturbed_tgv(*shape, dx=dx, amp=1e-3)
    s = make(osbli, shape, order, dx, dt, scheme=osbli.OSBLI_RK3_2R)
    s.set_state(Q)
    s.step(10)
    Qo = orc.step(orc.OracleParams(*shape, order, dx, dt=dt, **TGV_PHYS), Q, 2, 10)
    e = relerr(s.get_state(), Qo)
    assert np.all(e < TOL), e
    # the two RK3 forms differ at O(dt^4) on this nonlinear problem
    Q1 = orc.step(orc.OracleParams(*shape, order, dx, dt=dt, **TGV_PHYS), Q, 1, 10)
    assert np.max(np.abs(Q1 - Qo)) > 0.0
    # the residual hook is unaffected by the scheme
    s.set_state(Q)
    assert np.all(relerr(s.residual(), orc.residual(orc.OracleParams(*shape, order, dx,
                                                                     **TGV_PHYS), Q)) < TOL)


@pytest.mark.parametrize("order,shape", [(2, (40, 36, 33)), (4, (64, 64, 64)), (12, (72, 40, 50))])
def test_kernels_are_deterministic(osbli, order, shape):
    """Repeated evaluations are bitwise identical (a race between the xy-pass's
    warp groups shows up here first, as run-to-run differences)."""
    dx = 2 * math.pi / max(shape)
    Q = perturbed_tgv(*shape, dx=dx, amp=0.02)
    s = make(osbli, shape, order, dx, 1e-3)
    s.set_state(Q)
    R0 = s.residual()
    for _ in range(4):
        assert np.array_equal(s.residual(), R0)
    s.step(2)
    Q2 = s.get_state()
    s.set_state(Q)
    s.step(2)
    assert np.array_equal(s.get_state(), Q2)


def test_async_state_io_overlapped_handles(osbli, orc):
    """osbli_set_state_async / osbli_get_state_async: three handles on their own
    streams, each step's input copied in from pinned host memory and its result
    copied out, all enqueued before one synchronisation — the results equal the
    oracle's step (the pattern bench.py's e2e line times)."""
    import torch
    shape, order = (24, 20, 18), 8
    dx, dt = 2 * math.pi / 24, 2e-3
    Qs = [perturbed_tgv(*shape, dx=dx, amp=0.02, seed=100 + k) for k in range(3)]
    qh = [torch.from_numpy(q).pin_memory() for q in Qs]
    qo = [torch.empty_like(q).pin_memory() for q in qh]
    solvers, streams = [], []
    for k in range(3):
        s = make(osbli, shape, order, dx, dt)
        st = torch.cuda.Stream()
        s.set_stream(st.cuda_stream)
        solvers.append(s)
        streams.append(st)
    for k in range(3):
        solvers[k].set_state_async(qh[k])
        solvers[k].step(1)
        solvers[k].get_state_async(qo[k])
    torch.cuda.synchronize()
    for k in range(3):
        solvers[k].sync()
        ref = orc.step(orc.OracleParams(*shape, order, dx, dt=dt, **TGV_PHYS), Qs[k], 1, 1)
        assert np.all(relerr(qo[k].numpy(), ref) < TOL)


def test_large_grid_64bit_offsets(osbli, orc):
    """The largest per-GPU box of the weak-scaling series (BASELINE configs[4]:
    1024x512x512 on 8 GPUs = 512x512x256 per GPU), 8th order, one RK3 step: byte
    offsets beyond 2^31 in every buffer.  Sampled points (corners, tile and plane
    edges, the far end) against the windowed oracle; mass conserved."""
    import psutil
    from oracle import windowed
    nx, ny, nz, order = 512, 512, 256, 8
    if psutil.virtual_memory().available < 24e9:
        pytest.skip("needs ~24 GB of host memory for the 512x512x256 state")
    dx = 2 * math.pi / 256
    dt = tgv_dt(256)
    Q = tgv(nx, ny, nz, dx=dx)
    s = make(osbli, (nx, ny, nz), order, dx, dt)
    s.set_state(Q)
    s.step(1)
    Qg = s.get_state()
    pts = [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (31, 15, 7), (32, 16, 8), (nx // 2, ny - 1, 0),
           (nx - 1, 0, nz // 2), (257, 300, 129), (100, 511, 255)]
    p = orc.OracleParams(nx, ny, nz, order, dx, dt=dt, **TGV_PHYS)
    So = windowed.sample_step(p, Q, pts, 1, 1)
    scale = np.max(np.abs(Qg.reshape(5, -1)), axis=1)
    for t, (i, j, k) in enumerate(pts):
        assert np.all(np.abs(Qg[:, k, j, i] - So[t]) / scale < TOL), (i, j, k)
    assert abs(Qg[0].sum() - Q[0].sum()) / Q[0].sum() < 1e-13


@pytest.mark.parametrize("shape,direction", [((1, 70000, 1), 1), ((70000, 1, 2), 0)])
def test_long_one_dimensional_grids(osbli, orc, shape, direction):
    """Grids longer than 65535 points in y (and in x): every launch dimension holds."""
    order, dx, dt = 4, 1e-3, 1e-5
    Q = entropy_wave(*shape, dx=dx, A=0.2, k=3, U=0.4, Minf=1.0, direction=direction)
    phys = dict(Re=math.inf, Pr=0.71, Minf=1.0, gamma=1.4)
    s = make(osbli, shape, order, dx, dt, **phys)
    s.set_state(Q)
    s.step(2)
    Qo = orc.step(orc.OracleParams(*shape, order, dx, dt=dt, **phys), Q, 1, 2)
    assert np.all(relerr(s.get_state(), Qo) < TOL)


# ---------------------------------------------------------------- fused diagnostics
def test_tgv64_series_fused_vs_golden(osbli):
    """BASELINE configs[1] through osbli_step_diag (diagnostics fused into every
    step's first xy-pass): the E_k, enstrophy and dissipation series of the oracle
    (tests/golden) to 1e-9 over the first 1000 steps."""
    path = os.path.join(os.path.dirname(__file__), "golden", "tgv64_o4_rk3_series.csv")
    gold = np.loadtxt(path, delimiter=",", comments="#", skiprows=2)
    n, dt = 64, 3.385e-3
    s = make(osbli, (n, n, n), 4, 2 * math.pi / n, dt)
    s.set_state(tgv(n, n, n))
    nsteps = int(gold[-1, 0]) + 1
    series = s.step_diag(nsteps)
    assert [d.step for d in series] == list(range(nsteps))
    got = {d.step: np.array([d.kinetic_energy, d.enstrophy, d.dissipation]) for d in series}
    worst = np.zeros(3)
    for row in gold:
        worst = np.maximum(worst, np.abs(got[int(row[0])] - row[2:5]) / np.abs(row[2:5]))
    assert np.all(worst < 1e-9), worst


@pytest.mark.parametrize("order,shape,variant", [(12, (40, 36, 33), ""), (8, (70, 33, 20), "v"),
                                                 (4, (24, 20, 16), "c"), (6, (33, 17, 9), "s")])
def test_fused_diagnostics_equal_standalone(osbli, orc, order, shape, variant):
    """osbli_step_diag's series equals osbli_diagnostics of the same states (round-off:
    the two sum the plane in different tilings) and the oracle's, with Sutherland
    mu(T) (v), the conservative viscous work (c) and symmetry boundaries (s)."""
    dx = 2 * math.pi / max(shape)
    dt = 1e-3
    Q = perturbed_tgv(*shape, dx=dx, amp=0.02)
    a = make(osbli, shape, order, dx, dt)
    b = make(osbli, shape, order, dx, dt)
    op = orc.OracleParams(*shape, order, dx, dt=dt, **TGV_PHYS)
    for s in (a, b):
        if "v" in variant:
            s.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, 110.4 / 288.0)
        if "c" in variant:
            s.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
        if "s" in variant:
            for d in range(3):
                s.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
        s.set_state(Q)
    if "v" in variant:
        op.visc_law, op.suth = 1, 110.4 / 288.0
    if "c" in variant:
        op.energy_form = 1
    if "s" in variant:
        op.sym = (1, 1, 1)
    series = a.step_diag(3)
    Qs = Q
    for k in range(3):
        d = b.diagnostics()
        do = orc.diagnostics(op, Qs)
        f = series[k]
        assert f.step == k and d.step == k
        for x, y, z in ((f.kinetic_energy, d.kinetic_energy, do[0]), (f.enstrophy, d.enstrophy, do[1]),
                        (f.dissipation, d.dissipation, do[2])):
            assert abs(x - y) <= 1e-13 * abs(y), (k, x, y)
            assert abs(x - z) <= 1e-12 * abs(z), (k, x, z)
        b.step(1)
        Qs = orc.step(op, Qs, 1, 1)
    assert np.array_equal(a.get_state(), b.get_state())
