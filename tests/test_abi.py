"""The C-ABI library loads on a GPU-less host and exports every symbol the
header declares (no compute calls here)."""

import re
from pathlib import Path

import pytest

from paper_2507_01522_b200 import _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "voltyard_b200.h"


def declared():
    src = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(vy_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_abi():
    names = declared()
    assert "vy_step" in names and "vy_create" in names and len(names) >= 12


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.vy_abi_version() == 1


def test_binding_signatures_cover_header():
    assert set(_native.exported_symbols()) == set(declared())


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(_native.NativeError):
        _native.lib()


def test_null_arguments_are_rejected_without_a_gpu():
    import ctypes as C

    lib = _native.lib()
    assert lib.vy_create(None, 4, 0, None) == _native.VY_ERR_ARG
    assert b"null" in lib.vy_last_error()
    assert lib.vy_step(None, None, 0, 0, 0, 0, None, None) == _native.VY_ERR_STATE
    out = C.c_void_p()
    assert lib.vy_destroy(out) == 0
