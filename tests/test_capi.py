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


def test_ctypes_structs_match_the_c_header(tmp_path):
    """The Python mirror's ctypes structs have the C layout of include/bfpmg_b200.h."""
    import paper_2307_00124_b200 as B
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "bfpmg_b200.h"\n'
                   "int main(void) { printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(bfp_mg_config_t),"
                   " offsetof(bfp_mg_config_t, ref_mode), offsetof(bfp_mg_config_t, ref_c1d),"
                   " sizeof(bfp_xf_t), sizeof(bfp_trace_rec_t)); return 0; }\n")
    exe = tmp_path / "sz"
    subprocess.run(["/usr/bin/gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(B.MgConfig), B.MgConfig.ref_mode.offset, B.MgConfig.ref_c1d.offset,
            ctypes.sizeof(B.XfC), ctypes.sizeof(B.TraceRec)]
    assert got == want


def test_refmode_host_scalars_match_the_restatement():
    """The product's host setup of the reference mode (Chebyshev scalars) equals the
    oracle's independent derivation."""
    from fractions import Fraction

    from oracle import pyref_refmode as R
    from paper_2307_00124_b200 import refmode
    for rho, eta in ((2.02, 0.3), (2.0, 0.0), (1.98765, 0.15), (3.1, 0.77)):
        wdot = [0] + [w for w in range(3, 34)]
        c1, kres, c1d, c2d = refmode.chebyshev_scalars(rho, eta, 400, wdot)
        rc1, rc2 = R.chebyshev(Fraction(rho), R.eta_rational(eta))
        c1x = R._round(rc1, 400, False)
        c2x = -R._round(-rc2, 400, False)
        hi, lo, e, st = c1
        top = Fraction((hi << 64) | lo) * Fraction(2) ** e
        assert top <= c1x < top + Fraction(2) ** (e + 1) and (st == 1) == (top != c1x)
        for l in range(1, 32):
            a = R.quantize_scalar_floor(c1x, wdot[l])
            b = R.quantize_scalar_floor(c2x, wdot[l])
            assert c1d[l] == (a.m[0], wdot[l], a.e) and c2d[l] == (b.m[0], wdot[l], b.e)


def test_cpp_facade_compiles():
    """include/bfpmg_b200.hpp (the reference-named C++ facade) builds against the C-ABI
    with g++ alone (no CUDA headers in the facade)."""
    import __graft_entry__ as g
    g.build_facade_test()
    assert os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "tests", "cpp", "_build", "facade_test"))
