"""TMA tensor-box staging (xy-pass interior tiles, z-pass raw planes) against the
cp.async staging it replaces (OSBLI_XY_TMA=0, OSBLI_ZP_TMA=0): the
same values land in shared memory, so the states after RK3 steps must be bitwise
equal.  The switches are read once per process, so each staging runs in its own
subprocess."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RUN = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1609_01277_b200 as osbli
from inputs import TGV_PHYS, perturbed_tgv, tgv_dt
nx, ny, nz, order, scheme, steps, out, var = {args!r}
dx = 2 * np.pi / nx
s = osbli.Solver(nx, ny, nz, order, dx, tgv_dt(nx), scheme=scheme, **TGV_PHYS)
if "v" in var:
    s.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, 110.4 / 288.0)
if "c" in var:
    s.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
if "z" in var:
    s.set_boundary(2, osbli.OSBLI_BC_SYMMETRY)
s.set_state(perturbed_tgv(nx, ny, nz))
s.step(steps)
np.save(out, s.get_state())
"""


def _state(tmp_path, tag, env_extra, nx, ny, nz, order, scheme, steps, var=""):
    out = str(tmp_path / f"{tag}.npy")
    env = dict(os.environ, **env_extra)
    code = _RUN.format(root=ROOT, args=(nx, ny, nz, order, scheme, steps, out, var))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("shape,order,scheme", [((96, 96, 96), 12, 1), ((128, 96, 64), 8, 1),
                                                ((96, 80, 72), 10, 2), ((128, 128, 96), 4, 1)])
def test_tma_staging_is_bitwise_equal_to_cp_async(tmp_path, shape, order, scheme):
    nx, ny, nz = shape
    a = _state(tmp_path, "tma", {}, nx, ny, nz, order, scheme, 3)
    b = _state(tmp_path, "cpasync", {"OSBLI_XY_TMA": "0", "OSBLI_ZP_TMA": "0"}, nx, ny, nz, order,
               scheme, 3)
    assert np.isfinite(a).all()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("order,var", [(12, "v"), (8, "c"), (12, "z"), (6, "vcz")])
def test_tma_staging_bitwise_with_variants(tmp_path, order, var):
    """The equation-variant instantiation (Sutherland mu(T) v, conservative work c)
    and z symmetry (z: the z-pass boxes come from mirrored planes) stage by TMA as
    well; the result equals cp.async staging bitwise."""
    nx, ny, nz = 96, 80, 40
    a = _state(tmp_path, "tma", {}, nx, ny, nz, order, 1, 3, var)
    b = _state(tmp_path, "cpasync", {"OSBLI_XY_TMA": "0", "OSBLI_ZP_TMA": "0"}, nx, ny, nz, order,
               1, 3, var)
    assert np.isfinite(a).all()
    assert np.array_equal(a, b)
