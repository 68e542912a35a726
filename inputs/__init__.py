"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds none of the method's arithmetic (no stencils, no residual,
no time stepping): it only writes down initial states — the paper's Taylor-Green
vortex, an entropy wave, a smooth manufactured state, and a seeded
low-pass perturbation drawn from a counter-based generator (splitmix64) — and
converts primitive (rho, u, p) to the conservative variables with eqs. (10)-(11)
(P:259-266), as the paper's GridBasedInitialisation does.
"""
from .generators import (  # noqa: F401
    TGV_PHYS,
    conservative,
    tgv,
    tgv_dt,
    perturbed_tgv,
    entropy_wave,
    mms_primitives,
    mms_state,
    uniform_state,
    splitmix64,
)
