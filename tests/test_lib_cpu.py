"""CPU-side checks of the native boundary: the library builds/loads and
exports every entry point include/hpez_b200.h declares (no GPU calls)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "hpez_b200.h")).read()
    return sorted(set(re.findall(r"\b(hpez_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2311_12133_b200 import _lib
    lib = _lib.lib()
    names = _declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    import subprocess
    from paper_2311_12133_b200 import _lib
    _lib.lib()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_build_info():
    from paper_2311_12133_b200 import _lib
    assert b"sm_100a" in _lib.lib().hpez_build_info()
