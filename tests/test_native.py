"""The C-ABI library loads and exports every symbol include/efg.h declares (no GPU needed)."""
import ctypes
import re
import subprocess
from pathlib import Path

from paper_2306_00606_b200 import _native

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "efg.h").read_text()
    return sorted(set(re.findall(r"EFG_API\s+[\w\s\*]*?\b(efg_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (efg_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_abi_version_and_error_string():
    lib = _native.lib()
    assert lib.efg_abi_version() == 1
    assert isinstance(lib.efg_last_error(), bytes)


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_context_is_an_argument_error():
    lib = _native.lib()
    rc = lib.efg_synchronize(None)
    assert rc == 1
    assert b"null" in lib.efg_last_error()
