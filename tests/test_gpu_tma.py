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
nx, ny, nz, order, scheme, steps, out = {args!r}
dx = 2 * np.pi / nx
s = osbli.Solver(nx, ny, nz, order, dx, tgv_dt(nx), scheme=scheme, **TGV_PHYS)
s.set_state(perturbed_tgv(nx, ny, nz))
s.step(steps)
np.save(out, s.get_state())
"""


def _state(tmp_path, tag, env_extra, nx, ny, nz, order, scheme, steps):
    out = str(tmp_path / f"{tag}.npy")
    env = dict(os.environ, **env_extra)
    code = _RUN.format(root=ROOT, args=(nx, ny, nz, order, scheme, steps, out))
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
