"""B200-native OpenSBLI hot path: thin Python binding over libosbli.so (C ABI).

Every step of the path runs in the library's sm_100a kernels; this module only
marshals arguments (ctypes).  There is no CPU fallback: importing the binding
without a built ``libosbli.so`` raises immediately, and any call on a machine
without a CUDA device fails with the library's CUDA error.

PyTorch is used only for device memory and streams (torch tensors are passed
as device pointers) and process groups (``init_distributed``).
"""
from .native import (  # noqa: F401
    OSBLI_BC_PERIODIC,
    OSBLI_BC_SYMMETRY,
    OSBLI_ENERGY_CONSERVATIVE,
    OSBLI_ENERGY_EXPANDED,
    OSBLI_VISC_CONSTANT,
    OSBLI_VISC_SUTHERLAND,
    OSBLI_EULER,
    OSBLI_RK3,
    OSBLI_RK3_2R,
    OSBLI_SLAB_PLAIN,
    OSBLI_SLAB_XYSPLIT,
    OSBLI_SLAB_ZSPLIT,
    LoopbackGroup,
    OsbliError,
    ScalarSolver,
    Solver,
    ghost_plan,
    slab_bounds,
    build,
    lib_path,
    load,
    nccl_unique_id,
    version,
)
from .distributed import exchange_ghosts_torch, init_distributed  # noqa: F401
