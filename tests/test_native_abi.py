"""CPU checks of the C-ABI boundary: the in-tree library loads and exports exactly the
symbols declared in include/bilevel_b200.h (no compute without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2212_02224_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    with open(os.path.join(ROOT, "include", "bilevel_b200.h")) as fh:
        src = fh.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bd_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2212_02224_b200.build import build
    build()
    return _native.load()


def test_header_matches_binding_table():
    assert header_functions() == sorted(_native.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name


def test_abi_version(lib):
    assert lib.bd_abi_version() == 4


def test_struct_layouts():
    assert ctypes.sizeof(_native.Limits) == 9 * 8
    # 5 ints, pad, 4 doubles, u64, 3 ints + pad, 2 pointers (numpy stream state / positions)
    assert ctypes.sizeof(_native.CemConfig) == 5 * 4 + 4 + 4 * 8 + 8 + 16 + 16


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _native.Context(0)


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
