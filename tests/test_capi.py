"""CPU tests of the drop-in boundary: the sm_100a library builds/loads and
exports every symbol include/bfpmg_b200.h declares (no compute calls without a
GPU); the Python mirror raises loudly instead of falling back."""
import ctypes
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "bfpmg_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bfp_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "bfp_stencil_gemv" in syms and "bfp_mg_solve" in syms and len(syms) >= 35


def test_library_exports_every_declared_symbol():
    import paper_2307_00124_b200 as B
    if not os.path.exists(B.LIB_PATH):
        B.build()
    L = ctypes.CDLL(B.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB_PATH], capture_output=True,
                         text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s
    assert set(B.EXPORTS) == set(declared_symbols())


def test_library_is_sm100a():
    import paper_2307_00124_b200 as B
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_without_gpu():
    import paper_2307_00124_b200 as B
    assert B.lib().bfp_status_string(2).decode() == "exact row exceeds 127 bits"


def test_missing_library_fails_loudly(monkeypatch):
    import paper_2307_00124_b200 as B
    monkeypatch.setattr(B, "_lib", None)
    monkeypatch.setattr(B, "LIB_PATH", "/nonexistent/libbfpmg_b200.so")
    with pytest.raises(RuntimeError):
        B.lib()
