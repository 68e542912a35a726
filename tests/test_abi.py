"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/osbli.h declares, and validates arguments before touching the device."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "osbli.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(osbli_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1609_01277_b200 import native
    if not os.path.exists(native.lib_path()):
        native.build()
    return native.load()


def test_library_exports_every_declared_symbol(lib):
    syms = _declared_symbols()
    assert len(syms) >= 14
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a(lib):
    from paper_1609_01277_b200 import native
    out = os.popen(f"cuobjdump --list-elf {native.lib_path()} 2>/dev/null").read()
    assert "sm_100a" in out


def test_version_string(lib):
    assert b"sm_100a" in lib.osbli_version()


@pytest.mark.parametrize("args,code", [
    ((0, 8, 8, 4, 0.1, 0.01, 1600.0, 0.71, 0.1, 1.4, 1), -1),    # nx < 1
    ((8, 8, 8, 3, 0.1, 0.01, 1600.0, 0.71, 0.1, 1.4, 1), -1),    # odd order
    ((8, 8, 8, 0, 0.1, 0.01, 1600.0, 0.71, 0.1, 1.4, 1), -1),    # order 0
    ((8, 8, 8, 14, 0.1, 0.01, 1600.0, 0.71, 0.1, 1.4, 1), -2),   # not built
    ((8, 8, 8, 4, -0.1, 0.01, 1600.0, 0.71, 0.1, 1.4, 1), -1),   # dx <= 0
    ((8, 8, 8, 4, 0.1, math.nan, 1600.0, 0.71, 0.1, 1.4, 1), -1),  # dt nan
    ((8, 8, 8, 4, 0.1, 0.01, 0.0, 0.71, 0.1, 1.4, 1), -1),       # Re <= 0
    ((8, 8, 8, 4, 0.1, 0.01, 1600.0, 0.71, 0.1, 1.0, 1), -1),    # gamma <= 1
    ((8, 8, 8, 4, 0.1, 0.01, 1600.0, 0.71, 0.1, 1.4, 7), -1),    # scheme
])
def test_create_validates_arguments(lib, args, code):
    h = ctypes.c_void_p()
    rc = lib.osbli_create(*args, ctypes.byref(h))
    assert rc == code
    assert not h.value
    assert lib.osbli_last_error(None)


def test_null_handle_calls_are_rejected(lib):
    assert lib.osbli_step(None, 1) == -1
    assert lib.osbli_sync(None) == -1
    assert lib.osbli_kernel_launches(None) == -1
    lib.osbli_destroy(None)


def test_product_package_does_not_import_oracle():
    """The product path never routes through oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1609_01277_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.lower().replace("no cpu fallback", ""), f
