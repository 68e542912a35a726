"""GPU <-> oracle parity on the kernels' production code paths (B200).

The small-grid parity tests (test_gpu_parity.py) launch the xy-pass with one
plane per CTA and the z-pass with one chunk per pencil, because the launch
heuristics shrink both on grids that would not fill the 148 SMs.  The grids
here are large enough for the configuration the 256^3 bench runs:

* 96^3 o12: xy-pass segments of 8 planes (the cross-plane buffer reuse and the
  group A/B hand-offs), z-pass segments of 2 chunks (ring advance);
* 96^3 o8 and 128^3 o4: the same at other orders, 4 chunks per z pencil at 128^3;
* 256^3 o12, the bench workload itself (BASELINE configs[3]), 3 RK3 steps,
  compared on 5 blocks of 8^3 points (2560 points) straddling tile, segment,
  chunk and periodic-wrap boundaries, with the block oracle (oracle/windowed.py,
  pinned bitwise to the full-grid oracle in test_oracle_pins.py).

Every full-field case runs 10 RK3 steps (BASELINE north star: max relative
error 1e-11 per conservative field after 10 steps; D-14).  The oracle
runs (~1-2 min each on the GPU host) are started together in a thread pool when
the module's first test runs (ctypes releases the GIL), so the module costs
about the longest of them.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from inputs import TGV_PHYS, perturbed_tgv, tgv_dt

pytestmark = pytest.mark.gpu

TOL = 1e-11
STEPS = 10

FULL = {  # name: (shape, order)
    "96_o12": ((96, 96, 96), 12),
    "96_o8": ((96, 96, 96), 8),
    "128_o4": ((128, 128, 128), 4),
    # odd m (the staged-column offset of odd orders), TMA interior tiles, a ragged
    # last z chunk and two z segments per pencil
    "96x80x72_o10": ((96, 80, 72), 10),
}

N256, O256, S256 = 256, 12, 3
O256_ALL = (12, 8)  # BASELINE configs[3] (12th order) and configs[4] (8th order, weak scaling)
# (lo, size) blocks of the 256^3 grid: x tile edges at multiples of 32, y tile
# edges at multiples of 16, xy-pass segments of 8 planes, z-pass chunks of 32
# planes, and the periodic wrap in every direction
BLOCKS = [
    ((28, 12, 252), (8, 8, 8)),    # tile corner x 31|32, y 15|16; z wrap 255|0
    ((252, 252, 4), (8, 8, 8)),    # x, y wrap; xy segment boundary z 7|8
    ((28, 44, 28), (8, 8, 8)),     # z-pass chunk boundary 31|32|33
    ((124, 12, 60), (8, 8, 8)),    # z 63|64
    ((60, 124, 124), (8, 8, 8)),   # z 127|128, mid-grid tiles
]


def relerr(a, b):
    a = np.asarray(a).reshape(5, -1)
    b = np.asarray(b).reshape(5, -1)
    return np.array([np.max(np.abs(a[f] - b[f])) / max(np.max(np.abs(b[f])), 1e-300)
                     for f in range(5)])


def _dx(shape):
    return 2 * math.pi / max(shape)


def _input(shape):
    return perturbed_tgv(*shape, dx=_dx(shape), amp=1e-3)


@pytest.fixture(scope="module")
def osbli():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_1609_01277_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def refs(oracle_lib):
    """Every oracle reference of this module, computed concurrently."""
    from oracle import windowed
    orc = oracle_lib
    pool = ThreadPoolExecutor(max_workers=max(2, min(len(FULL) + 2 * len(BLOCKS), os.cpu_count() or 2)))
    out = {}

    def full_job(shape, order):
        Q = _input(shape)
        p = orc.OracleParams(*shape, order, _dx(shape), dt=tgv_dt(max(shape)), **TGV_PHYS)
        R = orc.residual(p, Q)
        Qn = orc.step(p, Q, 1, STEPS)
        return Q, R, Qn, orc.diagnostics(p, Qn)

    for name, (shape, order) in FULL.items():
        out[name] = pool.submit(full_job, shape, order)
    shape = (N256,) * 3
    Q256 = _input(shape)
    for order in O256_ALL:
        p256 = orc.OracleParams(*shape, order, _dx(shape), dt=tgv_dt(N256), **TGV_PHYS)
        for b, (lo, size) in enumerate(BLOCKS):
            out[("256", order, b)] = pool.submit(windowed.sample_block, p256, Q256, lo, size, 1,
                                                 S256)
    out["Q256"] = Q256
    yield out
    pool.shutdown(wait=True, cancel_futures=True)


@pytest.mark.parametrize("name", list(FULL))
def test_full_field_10_steps_production_paths(osbli, refs, name):
    """Every point of every field after 10 RK3 steps, the residual, and the
    diagnostics of the final state against the oracle."""
    shape, order = FULL[name]
    Q, Ro, Qo, do = refs[name].result()
    s = osbli.Solver(*shape, order, _dx(shape), tgv_dt(max(shape)), **TGV_PHYS)
    s.set_state(Q)
    e = relerr(s.residual(), Ro)
    assert np.all(e < TOL), ("residual", e)
    s.step(STEPS)
    Qg = s.get_state()
    e = relerr(Qg, Qo)
    assert np.all(e < TOL), ("state", e)
    d = s.diagnostics()
    got = np.array([d.kinetic_energy, d.enstrophy, d.dissipation])
    assert np.all(np.abs(got - np.array(do)) / np.abs(np.array(do)) < 1e-12), (got, do)
    # the same steps again: bitwise identical (races would show here first)
    s.set_state(Q)
    s.step(STEPS)
    assert np.array_equal(s.get_state(), Qg)
    s.close()


@pytest.mark.parametrize("order", O256_ALL)
def test_bench_workload_256_blocks(osbli, refs, order):
    """BASELINE configs[3] (TGV-shaped 256^3, 12th order) and configs[4] (8th order)
    in the bench's launch configuration, 3 RK3 steps, 2560 points in 5 blocks
    against the oracle; the same 3 steps repeated are bitwise identical; mass is
    conserved."""
    Q = refs["Q256"]
    shape = (N256,) * 3
    s = osbli.Solver(*shape, order, _dx(shape), tgv_dt(N256), **TGV_PHYS)
    s.set_state(Q)
    s.step(S256)
    Qg = s.get_state()
    scale = np.max(np.abs(Qg.reshape(5, -1)), axis=1)
    worst = np.zeros(5)
    for b, (lo, size) in enumerate(BLOCKS):
        ref = refs[("256", order, b)].result()
        ix = [(np.arange(size[d]) + lo[d]) % N256 for d in range(3)]
        got = Qg[:, ix[2]][:, :, ix[1]][:, :, :, ix[0]]
        err = np.max(np.abs(got - ref).reshape(5, -1), axis=1) / scale
        worst = np.maximum(worst, err)
    assert np.all(worst < TOL), worst
    assert abs(Qg[0].sum() - Q[0].sum()) / Q[0].sum() < 1e-13
    s.set_state(Q)
    s.step(S256)
    assert np.array_equal(s.get_state(), Qg)
    s.close()
