"""The C-ABI library loads and exports every symbol include/mknn_b200.h
declares (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_1412_6170_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mknn_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mknn_[a-z_]+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "mknn_tick" in syms and "mknn_create" in syms and len(syms) == 23
    assert set(syms) == set(_native.SIGNATURES), "ctypes table out of sync with the header"


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_abi_version():
    assert _native.lib().mknn_abi_version() == 1


def test_create_rejects_bad_config_without_touching_the_gpu():
    cfg = _native.Config(k=0, th_quad=4, l_max=10, rebuild_window=3, rebuild_factor=1.5,
                         x_lo=0.0, y_lo=0.0, x_hi=1.0, y_hi=1.0)
    h = ctypes.c_void_p()
    assert _native.lib().mknn_create(ctypes.byref(cfg), ctypes.byref(h)) == _native.EINVAL
    cfg.k = 4
    cfg.l_max = 11
    assert _native.lib().mknn_create(ctypes.byref(cfg), ctypes.byref(h)) == _native.EINVAL


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1412_6170_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f
