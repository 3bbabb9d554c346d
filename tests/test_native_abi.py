"""The C-ABI library loads without a GPU, exports every symbol that
include/sliceprop_b200.h declares, and was compiled for sm_100a."""

import os
import re
import subprocess

import pytest

from paper_2108_07126_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sliceprop_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "sp_equiprop" in names and "sp_make_plan" in names
    assert set(names) == set(_native.HEADER_SYMBOLS), "binding table out of sync with header"


def test_every_declared_symbol_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (sp_[a-z_0-9]+)", out))
    missing = set(declared_functions()) - exported
    assert not missing, missing
    for name in declared_functions():
        assert hasattr(_native.lib, name)


def test_library_is_sm_100a():
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_tensor_core_kernels_use_dmma():
    """The tensor-core lane kernels really issue FP64 MMA (SASS DMMA)."""
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", _native.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA.8x8x4" in sass


def test_version_and_device_count_without_gpu():
    assert _native.lib.sp_version().decode().startswith("sliceprop_b200")
    import ctypes
    n = ctypes.c_int(-1)
    assert _native.lib.sp_device_count(ctypes.byref(n)) == 0
    assert n.value >= 0
