"""The compiled C++ facade (include/bfpmg_b200.hpp: the reference's qaxpby / qsub / qspmv /
qgemv / nnq* / normalize / quantize / inf_norm_upper / dump_block names, QcompResult and the
exception types of P/include/bfpmg/blas.hpp:98-146) run on the GPU from a C++ program and
checked against the Python big-int restatement."""
import json
import os
import subprocess

import pytest

from oracle import pyref as P

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "facade_test")


def _blk(b, fl=None):
    d = {"q": b.q, "e": b.e, "m": list(b.m)}
    if fl is not None:
        d["flags"] = [int(fl.overflow), int(fl.underflow), int(fl.recomputed)]
    return d


def test_cpp_facade_vs_pyref():
    if not os.path.exists(EXE):
        import __graft_entry__ as g
        g.build_facade_test()
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2307_00124_b200", "_lib") +
               ":" + os.environ.get("LD_LIBRARY_PATH", ""))
    out = subprocess.run([EXE], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    got = {r["name"]: r for r in map(json.loads, out.stdout.strip().splitlines())}
    x = P.Block([5, -3, 7, 0, 2, -8, 1, 6], 5, -2)
    y = P.Block([1, 4, -2, 3, -7, 0, 5, -1], 4, 1)
    a, b = P.Block.scalar(3, 3, 0), P.Block.scalar(-2, 3, -1)
    g = lambda e: P.Block.scalar(1 << 14, 16, e)  # noqa: E731
    rows, cols, m, rp = 8, [], [], [0]
    for i in range(8):
        for j, v in ((i - 1, -1), (i, 2), (i + 1, -1)):
            if 0 <= j < 8:
                cols.append(j)
                m.append(v)
        rp.append(len(cols))
    A = P.Csr(rows, 8, rp, cols, m, 3, 2)
    eye = P.Csr(8, 8, list(range(9)), list(range(8)), [1] * 8, 2, 0)
    want = {
        "qaxpby": P.qcomp(P.EaxpbyKernel(x, y, a, b), 8, 12, g(-6)),
        "qaxpby_forced": P.qcomp(P.EaxpbyKernel(x, y, a, b), 8, 12, g(-6), force_recompute=True),
        "qaxpby_overflow": P.qcomp(P.EaxpbyKernel(x, y, a, b), 8, 12, g(-20)),
        "nnqaxpby": P.nnqcomp(P.EaxpbyKernel(x, y, a, b), 6, g(-9)),
        "qsub_xx": P.qcomp(P.EaxpbyKernel(x, x, P.bfp_one(), P.bfp_minus_one()), 8, 12, g(-6)),
        "qspmv_I": P.qcomp(P.EspmvKernel(eye, x), 5, 9, g(-11)),
        "qgemv": P.qcomp(P.EgemvKernel(A, x, y, P.bfp_minus_one(), P.bfp_one()), 10, 14, g(-7)),
        "nnqgemv": P.nnqcomp(P.EgemvKernel(A, x, y, P.bfp_minus_one(), P.bfp_one()), 7, g(-7)),
    }
    for name, (blk, fl) in want.items():
        w = _blk(blk, fl)
        r = got[name]
        assert (r["q"], r["e"], r["m"]) == (w["q"], w["e"], w["m"]), name
        assert r["flags"] == w["flags"], name
    assert got["qaxpby_forced"]["flags"][2] == 1 and got["qaxpby_overflow"]["flags"][0] == 1
    assert got["qsub_xx"]["m"] == [0] * 8
    nz = P.normalize(x)
    assert (got["normalize"]["q"], got["normalize"]["e"], got["normalize"]["m"]) == (nz.q, nz.e, list(nz.m))
    assert got["qspmv_I"]["m"] == list(nz.m) and got["qspmv_I"]["e"] == nz.e
    q3 = P.quantize(x, 3)
    assert (got["quantize3"]["q"], got["quantize3"]["e"], got["quantize3"]["m"]) == (q3.q, q3.e, list(q3.m))
    nu = P.inf_norm_upper(x, 16)
    assert (got["inf_norm_upper"]["m"], got["inf_norm_upper"]["q"], got["inf_norm_upper"]["e"]) == \
        (nu.m[0], nu.q, nu.e)
    assert got["dump_roundtrip"]["ok"] == 1
    assert got["exceptions"] == {"name": "exceptions", "domain": 1, "invalid": 1, "invalid2": 1}
