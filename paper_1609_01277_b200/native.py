"""ctypes binding of include/osbli.h (argument marshalling only)."""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
# OSBLI_LIB selects an alternative in-tree build (kernel-variant experiments)
_LIB_PATH = os.environ.get("OSBLI_LIB") or os.path.join(_HERE, "libosbli.so")
_lib = None

OSBLI_EULER = 0
OSBLI_RK3 = 1
OSBLI_RK3_2R = 2
OSBLI_BC_PERIODIC = 0
OSBLI_BC_SYMMETRY = 1
OSBLI_VISC_CONSTANT = 0
OSBLI_VISC_SUTHERLAND = 1
OSBLI_ENERGY_EXPANDED = 0
OSBLI_ENERGY_CONSERVATIVE = 1
OSBLI_SLAB_PLAIN = 0
OSBLI_SLAB_ZSPLIT = 1
OSBLI_SLAB_XYSPLIT = 2
_STATUS = {0: "OK", -1: "E_INVAL", -2: "E_UNSUPPORTED", -3: "E_NOMEM", -4: "E_CUDA",
           -5: "E_COMM", -6: "E_NONFINITE", -7: "E_STATE"}


class OsbliError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"osbli {_STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = _STATUS.get(code, str(code))


def lib_path() -> str:
    return _LIB_PATH


def build() -> str:
    """Compile libosbli.so for sm_100a in-tree (nvcc; no GPU needed)."""
    subprocess.check_call(["make", "-s", "-C", _ROOT, "paper_1609_01277_b200/libosbli.so"])
    return _LIB_PATH


class _Diag(ctypes.Structure):
    _fields_ = [("t", ctypes.c_double), ("step", ctypes.c_longlong),
                ("kinetic_energy", ctypes.c_double), ("enstrophy", ctypes.c_double),
                ("dissipation", ctypes.c_double)]


def load():
    """Load libosbli.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `make` (or __graft_entry__.build())")
    L = ctypes.CDLL(_LIB_PATH)
    c_int, c_double, vp = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
    H = ctypes.c_void_p
    L.osbli_create.argtypes = [c_int, c_int, c_int, c_int, c_double, c_double, c_double, c_double,
                               c_double, c_double, c_int, ctypes.POINTER(H)]
    L.osbli_create_dist.argtypes = [c_int, c_int, c_int, c_int, c_double, c_double, c_double,
                                    c_double, c_double, c_double, c_int, c_int, c_int, vp,
                                    ctypes.POINTER(H)]
    L.osbli_nccl_unique_id.argtypes = [vp]
    L.osbli_local_box.argtypes = [H, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]
    L.osbli_set_stream.argtypes = [H, vp]
    L.osbli_set_state.argtypes = [H, vp, c_int]
    L.osbli_get_state.argtypes = [H, vp, c_int]
    L.osbli_step.argtypes = [H, c_int]
    L.osbli_diagnostics.argtypes = [H, ctypes.POINTER(_Diag)]
    L.osbli_step_diag.argtypes = [H, c_int, ctypes.POINTER(_Diag)]
    L.osbli_residual.argtypes = [H, vp, c_int]
    L.osbli_sync.argtypes = [H]
    L.osbli_set_kernel_timing.argtypes = [H, c_int]
    L.osbli_kernel_timing.argtypes = [H, ctypes.POINTER(c_double), ctypes.POINTER(c_double),
                                      ctypes.POINTER(ctypes.c_longlong),
                                      ctypes.POINTER(ctypes.c_longlong)]
    ip = ctypes.POINTER(c_int)
    L.osbli_slab_bounds.argtypes = [c_int, c_int, c_int, ip, ip]
    L.osbli_ghost_plan.argtypes = [c_int, c_int, c_int, c_int, ip]
    L.osbli_ghost_plan_sym.argtypes = [c_int, c_int, c_int, c_int, c_int, ip]
    L.osbli_create_loopback.argtypes = [c_int, c_int, c_int, c_int, c_double, c_double, c_double,
                                        c_double, c_double, c_double, c_int, c_int,
                                        ctypes.POINTER(H)]
    L.osbli_loopback_step.argtypes = [ctypes.POINTER(H), c_int, c_int]
    L.osbli_set_source.argtypes = [H, vp, c_int]
    L.osbli_set_boundary.argtypes = [H, c_int, c_int]
    L.osbli_set_slab_schedule.argtypes = [H, c_int]
    L.osbli_set_state_async.argtypes = [H, vp, c_int]
    L.osbli_get_state_async.argtypes = [H, vp, c_int]
    L.osbli_set_viscosity.argtypes = [H, c_int, ctypes.c_double]
    L.osbli_set_energy_form.argtypes = [H, c_int]
    L.osbli_scalar_create.argtypes = [c_int, c_int, c_int, c_int, c_double, c_double, c_double,
                                      c_double, c_double, c_double, c_int, ctypes.POINTER(H)]
    for fn in ("osbli_scalar_set_state", "osbli_scalar_set_source", "osbli_scalar_get_state",
               "osbli_scalar_residual"):
        getattr(L, fn).argtypes = [H, vp, c_int]
    L.osbli_scalar_step.argtypes = [H, c_int]
    L.osbli_scalar_set_stream.argtypes = [H, vp]
    L.osbli_scalar_sync.argtypes = [H]
    L.osbli_scalar_last_error.argtypes = [H]
    L.osbli_scalar_last_error.restype = ctypes.c_char_p
    L.osbli_scalar_destroy.argtypes = [H]
    L.osbli_scalar_destroy.restype = None
    L.osbli_kernel_launches.argtypes = [H]
    L.osbli_kernel_launches.restype = ctypes.c_longlong
    L.osbli_last_error.argtypes = [H]
    L.osbli_last_error.restype = ctypes.c_char_p
    L.osbli_version.restype = ctypes.c_char_p
    L.osbli_destroy.argtypes = [H]
    L.osbli_destroy.restype = None
    _lib = L
    return L


def version() -> str:
    return load().osbli_version().decode()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load().osbli_nccl_unique_id(buf)
    if rc != 0:
        raise OsbliError(rc, load().osbli_last_error(None).decode())
    return buf.raw


def slab_bounds(nz: int, nranks: int, rank: int):
    """(z0, nz_local) from the library's partition rule (host-only, no GPU)."""
    z0, nzl = ctypes.c_int(), ctypes.c_int()
    rc = load().osbli_slab_bounds(nz, nranks, rank, ctypes.byref(z0), ctypes.byref(nzl))
    if rc != 0:
        raise OsbliError(rc, "invalid slab arguments")
    return z0.value, nzl.value


def ghost_plan(rank: int, nranks: int, nz_local: int, m: int, symz: bool = False):
    """The library's ghost-exchange plan: [(send_peer, send_plane, recv_peer, recv_plane)] x 2;
    with symmetry in z the transfers across the periodic wrap have peer -1."""
    plan = (ctypes.c_int * 8)()
    rc = load().osbli_ghost_plan_sym(rank, nranks, nz_local, m, int(symz), plan)
    if rc != 0:
        raise OsbliError(rc, "invalid ghost-plan arguments")
    return [tuple(plan[4 * t:4 * t + 4]) for t in range(2)]


def _ptr(a):
    """(pointer, on_device) for a numpy array or a contiguous fp64 torch tensor."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
            raise ValueError("state arrays must be C-contiguous float64")
        return a.ctypes.data, 0
    import torch  # torch only for device memory
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("state tensors must be contiguous float64")
        return a.data_ptr(), 1 if a.is_cuda else 0
    raise TypeError(f"unsupported array type {type(a)}")


@dataclass
class Diagnostics:
    t: float
    step: int
    kinetic_energy: float
    enstrophy: float
    dissipation: float


class Solver:
    """One handle of the C ABI (osbli_create / osbli_create_dist)."""

    def __init__(self, nx, ny, nz, order, dx, dt, Re=1600.0, Pr=0.71, Minf=0.1, gamma=1.4,
                 scheme=OSBLI_RK3, rank=0, nranks=1, unique_id: bytes | None = None):
        L = load()
        self._L = L
        self._h = ctypes.c_void_p()
        if nranks == 1 and unique_id is None:
            rc = L.osbli_create(nx, ny, nz, order, dx, dt, Re, Pr, Minf, gamma, scheme,
                                ctypes.byref(self._h))
        else:
            uid = ctypes.create_string_buffer(unique_id, 128) if unique_id else None
            rc = L.osbli_create_dist(nx, ny, nz, order, dx, dt, Re, Pr, Minf, gamma, scheme,
                                     rank, nranks, uid, ctypes.byref(self._h))
        if rc != 0:
            raise OsbliError(rc, L.osbli_last_error(None).decode())
        self.nx, self.ny, self.nz_global, self.order = nx, ny, nz, order
        z0, nzl = ctypes.c_int(), ctypes.c_int()
        L.osbli_local_box(self._h, ctypes.byref(z0), ctypes.byref(nzl))
        self.z0, self.nz = z0.value, nzl.value
        self.shape = (5, self.nz, ny, nx)

    def _check(self, rc):
        if rc != 0:
            raise OsbliError(rc, self._L.osbli_last_error(self._h).decode())

    def set_stream(self, stream_handle: int | None):
        self._check(self._L.osbli_set_stream(self._h, ctypes.c_void_p(stream_handle or 0)))

    def set_state(self, q):
        if tuple(q.shape) != self.shape:
            raise ValueError(f"state shape {tuple(q.shape)} != {self.shape}")
        p, dev = _ptr(q)
        self._check(self._L.osbli_set_state(self._h, ctypes.c_void_p(p), dev))

    def get_state(self, out=None):
        if out is None:
            out = np.empty(self.shape, dtype=np.float64)
        p, dev = _ptr(out)
        self._check(self._L.osbli_get_state(self._h, ctypes.c_void_p(p), dev))
        return out

    def set_state_async(self, q):
        """Stream-ordered set_state (q: pinned host or device tensor, kept alive by the caller)."""
        if tuple(q.shape) != self.shape:
            raise ValueError(f"state shape {tuple(q.shape)} != {self.shape}")
        p, dev = _ptr(q)
        self._check(self._L.osbli_set_state_async(self._h, ctypes.c_void_p(p), dev))

    def get_state_async(self, out):
        """Stream-ordered get_state into out (pinned host or device tensor)."""
        if tuple(out.shape) != self.shape:
            raise ValueError(f"state shape {tuple(out.shape)} != {self.shape}")
        p, dev = _ptr(out)
        self._check(self._L.osbli_get_state_async(self._h, ctypes.c_void_p(p), dev))
        return out

    def step(self, n: int = 1):
        self._check(self._L.osbli_step(self._h, int(n)))

    def residual(self, out=None):
        if out is None:
            out = np.empty(self.shape, dtype=np.float64)
        p, dev = _ptr(out)
        self._check(self._L.osbli_residual(self._h, ctypes.c_void_p(p), dev))
        return out

    def diagnostics(self) -> Diagnostics:
        d = _Diag()
        self._check(self._L.osbli_diagnostics(self._h, ctypes.byref(d)))
        return Diagnostics(d.t, d.step, d.kinetic_energy, d.enstrophy, d.dissipation)

    def step_diag(self, n: int = 1):
        """Advance n steps; the diagnostics of each step's input state (fused into
        the step's first xy-pass), as a list of n Diagnostics."""
        arr = (_Diag * max(int(n), 1))()
        self._check(self._L.osbli_step_diag(self._h, int(n), arr))
        return [Diagnostics(d.t, d.step, d.kinetic_energy, d.enstrophy, d.dissipation)
                for d in arr[:int(n)]]

    def sync(self):
        self._check(self._L.osbli_sync(self._h))

    def set_slab_schedule(self, schedule: int):
        """Slab handles: OSBLI_SLAB_PLAIN (0), _ZSPLIT (1) or _XYSPLIT (2)."""
        self._check(self._L.osbli_set_slab_schedule(self._h, int(schedule)))

    def set_boundary(self, direction: int, bc: int):
        """OSBLI_BC_PERIODIC or OSBLI_BC_SYMMETRY for direction 0/1/2."""
        self._check(self._L.osbli_set_boundary(self._h, int(direction), int(bc)))

    def set_viscosity(self, law: int, suth: float = 0.0):
        """OSBLI_VISC_CONSTANT (mu = 1) or OSBLI_VISC_SUTHERLAND with suth = S/T_ref."""
        self._check(self._L.osbli_set_viscosity(self._h, int(law), float(suth)))

    def set_energy_form(self, form: int):
        """OSBLI_ENERGY_EXPANDED or OSBLI_ENERGY_CONSERVATIVE viscous work."""
        self._check(self._L.osbli_set_energy_form(self._h, int(form)))

    def set_source(self, S):
        """Steady source: dQ/dt = R(Q) + S (None removes it)."""
        if S is None:
            self._check(self._L.osbli_set_source(self._h, None, 0))
            return
        if tuple(S.shape) != self.shape:
            raise ValueError(f"source shape {tuple(S.shape)} != {self.shape}")
        p, dev = _ptr(S)
        self._check(self._L.osbli_set_source(self._h, ctypes.c_void_p(p), dev))

    def set_kernel_timing(self, enable: bool):
        self._check(self._L.osbli_set_kernel_timing(self._h, 1 if enable else 0))

    def kernel_timing(self):
        """(zpass_ms_total, xypass_ms_total, n_zpass, n_xypass) since the last call."""
        z, x = ctypes.c_double(), ctypes.c_double()
        nz, nx = ctypes.c_longlong(), ctypes.c_longlong()
        self._check(self._L.osbli_kernel_timing(self._h, ctypes.byref(z), ctypes.byref(x),
                                                ctypes.byref(nz), ctypes.byref(nx)))
        return z.value, x.value, nz.value, nx.value

    @property
    def kernel_launches(self) -> int:
        return int(self._L.osbli_kernel_launches(self._h))

    @classmethod
    def _wrap(cls, L, h, nx, ny, nz_global, order):
        self = cls.__new__(cls)
        self._L, self._h = L, h
        self.nx, self.ny, self.nz_global, self.order = nx, ny, nz_global, order
        z0, nzl = ctypes.c_int(), ctypes.c_int()
        L.osbli_local_box(self._h, ctypes.byref(z0), ctypes.byref(nzl))
        self.z0, self.nz = z0.value, nzl.value
        self.shape = (5, self.nz, ny, nx)
        return self

    def close(self):
        if self._h:
            self._L.osbli_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class ScalarSolver:
    """Scalar advection-diffusion of the paper's verification cases (osbli_scalar_*):
    d phi/dt + d/dx_j [phi u_j - kappa d phi/dx_j] + S = 0, phi [nz][ny][nx]."""

    def __init__(self, nx, ny, nz, order, dx, dt, u=(0.0, 0.0, 0.0), kappa=0.0,
                 scheme=OSBLI_RK3):
        L = load()
        self._L = L
        self._h = ctypes.c_void_p()
        rc = L.osbli_scalar_create(nx, ny, nz, order, dx, dt, float(u[0]), float(u[1]),
                                   float(u[2]), float(kappa), scheme, ctypes.byref(self._h))
        if rc != 0:
            raise OsbliError(rc, L.osbli_scalar_last_error(None).decode())
        self.shape = (nz, ny, nx)

    def _check(self, rc):
        if rc != 0:
            raise OsbliError(rc, self._L.osbli_scalar_last_error(self._h).decode())

    def _io(self, fn, a):
        if tuple(a.shape) != self.shape:
            raise ValueError(f"shape {tuple(a.shape)} != {self.shape}")
        p, dev = _ptr(a)
        self._check(fn(self._h, ctypes.c_void_p(p), dev))
        return a

    def set_stream(self, stream_handle):
        self._check(self._L.osbli_scalar_set_stream(self._h, ctypes.c_void_p(stream_handle or 0)))

    def set_state(self, phi):
        self._io(self._L.osbli_scalar_set_state, phi)

    def set_source(self, S):
        if S is None:
            self._check(self._L.osbli_scalar_set_source(self._h, None, 0))
        else:
            self._io(self._L.osbli_scalar_set_source, S)

    def get_state(self, out=None):
        return self._io(self._L.osbli_scalar_get_state,
                        np.empty(self.shape) if out is None else out)

    def residual(self, out=None):
        return self._io(self._L.osbli_scalar_residual,
                        np.empty(self.shape) if out is None else out)

    def step(self, n=1):
        self._check(self._L.osbli_scalar_step(self._h, int(n)))

    def sync(self):
        self._check(self._L.osbli_scalar_sync(self._h))

    def close(self):
        if self._h:
            self._L.osbli_scalar_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """nslabs z-slab handles on one GPU exchanging ghost planes by device copies
    (osbli_create_loopback): the distributed kernel path without NCCL."""

    def __init__(self, nx, ny, nz, order, dx, dt, nslabs, Re=1600.0, Pr=0.71, Minf=0.1,
                 gamma=1.4, scheme=OSBLI_RK3):
        L = load()
        arr = (ctypes.c_void_p * nslabs)()
        rc = L.osbli_create_loopback(nx, ny, nz, order, dx, dt, Re, Pr, Minf, gamma, scheme,
                                     nslabs, arr)
        if rc != 0:
            raise OsbliError(rc, L.osbli_last_error(None).decode())
        self._L, self._arr = L, arr
        self.slabs = [Solver._wrap(L, ctypes.c_void_p(arr[i]), nx, ny, nz, order)
                      for i in range(nslabs)]

    def set_state(self, q):
        for s in self.slabs:
            s.set_state(np.ascontiguousarray(q[:, s.z0:s.z0 + s.nz]))

    def get_state(self):
        return np.concatenate([s.get_state() for s in self.slabs], axis=1)

    def step(self, n=1):
        rc = self._L.osbli_loopback_step(self._arr, len(self.slabs), int(n))
        if rc != 0:
            raise OsbliError(rc, self._L.osbli_last_error(self.slabs[0]._h).decode())

    def close(self):
        for s in self.slabs:
            s.close()


def inviscid() -> float:
    return math.inf
