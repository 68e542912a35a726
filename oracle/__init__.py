"""OpenSBLI hot-path oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product package ``paper_1609_01277_b200`` never imports it and shares no code
with it.

* ``oracle.cpp``   — plain single-threaded C++ implementation of the paper's
  discretisation (see its header for citations); built into ``liboracle.so``.
* ``core.py``      — ctypes wrapper (argument marshalling only).
* ``jets.py``      — second-order Taylor jets, used to evaluate the *continuous*
  residual of the paper's equations exactly for manufactured states
  (a pin for the discrete oracle, P:195-209 method of manufactured solutions).
* ``windowed.py``  — exact single-point evaluation of k time steps on a
  periodic window (the oracle run on a sub-box), for full-size sampled parity.
"""
from .core import (  # noqa: F401
    OracleParams,
    build,
    weights_exact,
    derivative,
    residual,
    step,
    diagnostics,
    run_series,
    scalar_residual,
    scalar_step,
)
