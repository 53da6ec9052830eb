"""Generate the committed golden fixtures under tests/golden/.

1. reference_known_answers.json -- the hand-derived known answers of the
   reference's own unit tests (paths relative to /root/reference/proj), as
   literal inputs/expected outputs with their file:line.  The script asserts
   the Python big-int restatement (oracle/pyref.py) reproduces every one.
2. mg_small.json -- driver-level golden vectors (final iterate, exponent,
   residual history, trace) of small configs of the DESIGN.md section 3
   driver, minted by pyref and cross-checked against the C oracle.

Run:  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import pyref as P  # noqa: E402

KA = [
    # wideint (tests/test_wideint.cpp)
    {"op": "msb", "v": 23, "want": 6, "ref": "tests/test_wideint.cpp:85"},
    {"op": "msb", "v": -8, "want": 4, "ref": "tests/test_wideint.cpp:86"},
    {"op": "msb", "v": -1, "want": 1, "ref": "tests/test_wideint.cpp:87"},
    {"op": "msb", "v": 0, "want": 1, "ref": "tests/test_wideint.cpp:88"},
    {"op": "ashr", "v": -3, "s": 1, "want": -2, "ref": "tests/test_wideint.cpp:45"},
    {"op": "ashr", "v": 5, "s": 1, "want": 2, "ref": "tests/test_wideint.cpp:46"},
] + [{"op": "ashr", "v": -1, "s": k, "want": -1, "ref": "tests/test_wideint.cpp:47"} for k in range(8)] + [
    {"op": "wrap", "v": 5, "w": 3, "want": -3, "ref": "tests/test_wideint.cpp:71 decr(1,5[w4])"},
    {"op": "clamp", "v": 11, "lo": -8, "hi": 7, "want": 7, "ref": "tests/test_wideint.cpp:101"},
    {"op": "clamp", "v": -9, "lo": -8, "hi": 7, "want": -8, "ref": "tests/test_wideint.cpp:102"},
    {"op": "clamp", "v": 3, "lo": -8, "hi": 7, "want": 3, "ref": "tests/test_wideint.cpp:103"},
    {"op": "dump_wideint", "v": -3, "w": 3, "want": "-3 w=3 0x5", "ref": "tests/test_wideint.cpp:108"},
    {"op": "dump_wideint", "v": 5, "w": 4, "want": "5 w=4 0x5", "ref": "tests/test_wideint.cpp:109"},
    {"op": "dump_wideint", "v": -1, "w": 8, "want": "-1 w=8 0xff", "ref": "tests/test_wideint.cpp:110"},
    # bfp (tests/test_bfp.cpp)
    {"op": "normalize", "m": [12, -4], "q": 8, "e": 0, "want": {"m": [96, -32], "e": -3},
     "ref": "tests/test_bfp.cpp:14-20"},
    {"op": "normalize", "m": [0, 0], "q": 6, "e": 5, "want": {"m": [0, 0], "e": 0},
     "ref": "tests/test_bfp.cpp:24-26"},
    {"op": "quantize", "m": [23, -5], "q": 8, "e": 0, "w": 4, "want": {"m": [5, -2], "e": 2},
     "ref": "tests/test_bfp.cpp:40-47"},
    {"op": "quantize", "m": [0, 0, 0], "q": 9, "e": 0, "w": 4, "want": {"m": [0, 0, 0], "e": 0},
     "ref": "tests/test_bfp.cpp:54-56"},
    {"op": "inf_norm_upper", "m": [23, -5], "q": 8, "e": 0, "qg": 16, "want_value": [23, 0],
     "ref": "tests/test_bfp.cpp:84-85"},
    {"op": "inf_norm_upper", "m": [23, -5], "q": 8, "e": 0, "qg": 3, "want_value": [24, 0],
     "ref": "tests/test_bfp.cpp:86-87"},
    {"op": "inf_norm_upper", "m": [-8], "q": 4, "e": 1, "qg": 16, "want_value": [16, 0],
     "ref": "tests/test_bfp.cpp:88-89"},
    {"op": "quantize_exact", "z": [1, -1], "k": [0, -1], "w": 3, "want": {"m": [2, -1], "e": -1},
     "ref": "tests/test_bfp.cpp:119-124 (from_extfloat [1,-0.5] w3)"},
    # blas (tests/test_blas.cpp)
    {"op": "qcomp_rows", "rows": [23, -5], "tq": 8, "te": 0, "w_out": 4, "w_tmp": 5,
     "gamma": [23, 6, 0], "want": {"m": [5, -2], "e": 2, "q": 4, "flags": [0, 0, 0]},
     "ref": "tests/test_blas.cpp:56-66"},
    {"op": "qcomp_rows", "rows": [23, -5], "tq": 8, "te": 0, "w_out": 4, "w_tmp": 5,
     "gamma": [8, 5, 0], "want": {"m": [5, -2], "e": 2, "q": 4, "flags": [1, 0, 1]},
     "ref": "tests/test_blas.cpp:68-71"},
    {"op": "qcomp_rows", "rows": [23, -5], "tq": 8, "te": 0, "w_out": 4, "w_tmp": 5,
     "gamma": [184, 9, 0], "want": {"m": [5, -2], "e": 2, "q": 4, "flags": [0, 1, 1]},
     "ref": "tests/test_blas.cpp:73-76"},
    {"op": "qcomp_rows", "rows": [23, -5], "tq": 8, "te": 0, "w_out": 4, "w_tmp": 4,
     "gamma": [23, 6, 0], "nn": True, "want": {"m": [5, -2], "e": 2, "q": 4},
     "ref": "tests/test_blas.cpp:86-90 (gamma-exact nnqcomp == qcomp)"},
    {"op": "qcomp_rows", "rows": [23], "tq": 8, "te": 0, "w_out": 4, "w_tmp": 4,
     "gamma": [8, 5, 0], "nn": True, "want": {"m": [7], "e": 1, "q": 4},
     "ref": "tests/test_blas.cpp:92-95 (saturates: value 14)"},
    {"op": "qcomp_rows", "rows": [3], "tq": 8, "te": 0, "w_out": 4, "w_tmp": 4,
     "gamma": [64, 8, 0], "nn": True, "want": {"m": [0], "e": 4, "q": 4},
     "ref": "tests/test_blas.cpp:97-100 (bits lost silently)"},
    {"op": "qcomp_rows", "rows": [0, 0], "tq": 9, "te": -3, "w_out": 4, "w_tmp": 6,
     "gamma": [9, 5, 2], "want": {"m": [0, 0], "e": -6, "q": 4},
     "ref": "tests/test_blas.cpp:363-368 (zero result anchor e*+1-w_out)"},
    {"op": "qcomp_error", "rows": [1], "tq": 4, "te": 0, "w_out": 5, "w_tmp": 4, "gamma": [1, 2, 0],
     "ref": "tests/test_blas.cpp:81"},
    {"op": "qcomp_error", "rows": [1], "tq": 4, "te": 0, "w_out": 2, "w_tmp": 4, "gamma": [-1, 2, 0],
     "ref": "tests/test_blas.cpp:82"},
    {"op": "qcomp_error", "rows": [1], "tq": 4, "te": 0, "w_out": 2, "w_tmp": 2, "gamma": [0, 2, 0],
     "nn": True, "ref": "tests/test_blas.cpp:83"},
    {"op": "axpby_tmpl", "x": [[1, 2], 8, 0], "y": [[1, 2], 8, 0], "alpha": [5, 4, 0],
     "beta": [-3, 4, 0], "want": {"d": 0, "q": 13, "e": 0}, "ref": "tests/test_blas.cpp:115-118"},
    {"op": "axpby_tmpl", "x": [[1, 2], 8, 0], "y": [[1, 2], 8, 3], "alpha": [5, 4, 0],
     "beta": [-3, 4, 0], "want": {"d": -3, "q": 16, "e": 0}, "ref": "tests/test_blas.cpp:120-124"},
    {"op": "spmv_tmpl", "qa": 4, "qx": 4, "m_a": 3, "want_q": 10, "ref": "tests/test_blas.cpp:141"},
    {"op": "spmv_tmpl", "qa": 4, "qx": 4, "m_a": 1, "want_q": 8, "ref": "tests/test_blas.cpp:142"},
    {"op": "spmv_tmpl", "qa": 8, "qx": 8, "m_a": 256, "want_q": 24, "ref": "tests/test_blas.cpp:143"},
    {"op": "axpby_row", "x": [[5, -3], 4, 0], "y": [[5, -3], 4, 0], "alpha": [1, 2, 0],
     "beta": [-1, 1, 0], "want_values": [[0, 0], [0, 0]], "ref": "tests/test_blas.cpp:184-191"},
    {"op": "axpby_row", "x": [[5], 4, 0], "y": [[-1], 1, 1], "alpha": [1, 2, 1], "beta": [3, 3, 0],
     "want_values": [[4, 0]], "ref": "tests/test_blas.cpp:192-198 (2*5 + 3*(-2) = 4)"},
    {"op": "spmv_row", "a": {"rows": 1, "cols": 3, "rowptr": [0, 3], "col": [0, 1, 2],
                             "m": [1, -2, 1], "q": 3, "e": 0},
     "x": [[7, 7, 7], 4, 2], "want_rows": [0], "ref": "tests/test_blas.cpp:201-209"},
    {"op": "spmv_error", "a": {"rows": 1, "cols": 3, "rowptr": [0, 3], "col": [0, 1, 2],
                               "m": [1, -2, 1], "q": 3, "e": 0},
     "x": [[7, 7, 7], 4, 2], "m_a": 2, "ref": "tests/test_blas.cpp:211"},
]

# driver-level configs, small enough for pure Python
MG_CASES = [
    dict(name="c1_small", d=1, l_fine=7, cycles=4, x0_random=True, rhs_kind=0, p=16),
    dict(name="c2_small", d=2, l_fine=5, cycles=3, rhs_kind=1, p=20),
    dict(name="c3_small", d=2, l_fine=6, l_coarse=3, cycles=1, rhs_kind=1, fmg=True,
         nonnormalized=True, p=[0, 0, 0] + [4 + 2 * (l - 3) for l in range(3, 32)][:29]),
    dict(name="c4_small", d=3, l_fine=4, cycles=1, rhs_kind=1, fmg=True, p=24),
    dict(name="c5_small", d=3, l_fine=4, cycles=2, x0_random=True, rhs_kind=2, p=48),
    # three-width PrecisionSchedule (w / wdot / wcheck) with a w_add cap (config 1 style)
    dict(name="c1_sched", d=1, l_fine=9, cycles=4, x0_random=True, rhs_kind=0, p=16,
         pd=[28] * 32, pc=[16] * 32, w_add_cap=4),
    # NormMode::hybrid (src/multigrid.cpp:406-408): qcomp only for IR residuals 1, 2
    dict(name="c2_hybrid", d=2, l_fine=5, cycles=4, rhs_kind=1, nonnormalized=2, p=20),
    dict(name="c3_hybrid", d=2, l_fine=6, l_coarse=3, cycles=3, rhs_kind=1, fmg=True,
         nonnormalized=2, p=[0, 0, 0] + [6 + 2 * (l - 3) for l in range(3, 32)][:29]),
]


def check_known_answers():
    for c in KA:
        op = c["op"]
        if op == "msb":
            assert P.msb(c["v"]) == c["want"], c
        elif op == "ashr":
            assert P.shift_floor(c["v"], c["s"]) == c["want"], c
        elif op == "wrap":
            assert P.truncate_to_width(c["v"], c["w"]) == c["want"], c
        elif op == "clamp":
            assert P.clamp(c["v"], c["lo"], c["hi"]) == c["want"], c
        elif op == "dump_wideint":
            assert P.dump_wideint(c["v"], c["w"]) == c["want"], c
        elif op in ("normalize", "quantize"):
            b = P.Block(c["m"], c["q"], c["e"])
            r = P.normalize(b) if op == "normalize" else P.quantize(b, c["w"])
            assert r.m == c["want"]["m"] and r.e == c["want"]["e"], (c, r)
        elif op == "inf_norm_upper":
            g = P.inf_norm_upper(P.Block(c["m"], c["q"], c["e"]), c["qg"])
            num, den = c["want_value"][0], 1
            assert g.values()[0] == num, (c, g)
        elif op == "quantize_exact":
            r = P.quantize_exact(c["z"], c["k"], c["w"])
            assert r.m == c["want"]["m"] and r.e == c["want"]["e"], (c, r)
        elif op == "qcomp_rows":
            k = P.FixedKernel(c["rows"], c["tq"], c["te"])
            g = P.Block.scalar(*c["gamma"])
            if c.get("nn"):
                r, fl = P.nnqcomp(k, c["w_out"], g)
            else:
                r, fl = P.qcomp(k, c["w_out"], c["w_tmp"], g)
                if "flags" in c["want"]:
                    assert [int(fl.overflow), int(fl.underflow), int(fl.recomputed)] == c["want"]["flags"]
            assert r.m == c["want"]["m"] and r.e == c["want"]["e"] and r.q == c["want"]["q"], (c, r)
        elif op == "qcomp_error":
            k = P.FixedKernel(c["rows"], c["tq"], c["te"])
            g = P.Block.scalar(*c["gamma"]) if c["gamma"][0] > 0 else P.Block([c["gamma"][0]], 8, 0, "scalar", 1, 1)
            try:
                if c.get("nn"):
                    P.nnqcomp(k, c["w_out"], g)
                else:
                    P.qcomp(k, c["w_out"], c["w_tmp"], g)
                raise AssertionError(f"no error: {c}")
            except ValueError:
                pass
        elif op == "axpby_tmpl":
            x, y = P.Block(*c["x"]), P.Block(*c["y"])
            k = P.EaxpbyKernel(x, y, P.Block.scalar(*c["alpha"]), P.Block.scalar(*c["beta"]))
            assert (k.d, k.tmpl.q, k.tmpl.e) == (c["want"]["d"], c["want"]["q"], c["want"]["e"]), c
        elif op == "spmv_tmpl":
            a = P.Csr(1, c["m_a"], [0, c["m_a"]], list(range(c["m_a"])), [1] * c["m_a"], c["qa"], 0)
            x = P.Block([0] * c["m_a"], c["qx"], 0)
            assert P.EspmvKernel(a, x, c["m_a"]).tmpl.q == c["want_q"], c
        elif op == "axpby_row":
            x, y = P.Block(*c["x"]), P.Block(*c["y"])
            k = P.EaxpbyKernel(x, y, P.Block.scalar(*c["alpha"]), P.Block.scalar(*c["beta"]))
            from fractions import Fraction
            for i, (num, _) in enumerate(c["want_values"]):
                assert Fraction(k.row(i)) * Fraction(2) ** k.tmpl.e == num, c
        elif op == "spmv_row":
            a = c["a"]
            A = P.Csr(a["rows"], a["cols"], a["rowptr"], a["col"], a["m"], a["q"], a["e"])
            k = P.EspmvKernel(A, P.Block(*c["x"]))
            assert [k.row(i) for i in range(A.rows)] == c["want_rows"], c
        elif op == "spmv_error":
            a = c["a"]
            A = P.Csr(a["rows"], a["cols"], a["rowptr"], a["col"], a["m"], a["q"], a["e"])
            try:
                P.EspmvKernel(A, P.Block(*c["x"]), c["m_a"])
                raise AssertionError("no error")
            except ValueError:
                pass
        else:
            raise KeyError(op)


def mg_case_cfg(case):
    kw = {k: v for k, v in case.items() if k not in ("name", "p")}
    p = case["p"]
    p = p + [0] * (32 - len(p)) if isinstance(p, list) else [p] * 32
    return kw, p


def mint_mg():
    from oracle import ob
    out = []
    for case in MG_CASES:
        kw, p = mg_case_cfg(case)
        res = P.Mg(P.MgConfig(**kw, p=p)).run()
        x, h, tr = ob.mg_run(ob.mg_config(**kw, p=p))
        assert x.m.tolist() == res.x.m and x.e == res.x.e, case["name"]
        assert h == res.history and tr == res.trace, case["name"]
        digest = hashlib.sha256(",".join(map(str, res.x.m)).encode()).hexdigest()
        out.append({"name": case["name"], "config": {**kw, "p": p}, "x_q": res.x.q, "x_e": res.x.e,
                    "x_sha256": digest, "x_head": res.x.m[:64], "history": res.history,
                    "trace": res.trace})
    return out


if __name__ == "__main__":
    check_known_answers()
    with open(os.path.join(HERE, "reference_known_answers.json"), "w") as f:
        json.dump({"source": "hand-derived known answers of the reference unit tests "
                             "(/root/reference/proj/tests), verified against oracle/pyref.py",
                   "cases": KA}, f, indent=1)
    mg = mint_mg()
    with open(os.path.join(HERE, "mg_small.json"), "w") as f:
        json.dump({"source": "oracle/pyref.py driver (DESIGN.md section 3), cross-checked "
                             "bit-exactly against oracle/bfp_oracle.c", "cases": mg}, f)
    print("ok", len(KA), "known answers;", len(mg), "driver cases")
