"""GPU parity: every call goes through the C-ABI of libbfpmg_b200.so on the
B200 and is compared bit-exactly (mantissas, exponents, flags, histories,
traces) with the CPU oracle on the same seeded inputs."""
import hashlib
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import ob
from oracle import pyref as P
from tests.cases import Rng, rational_axpby, rational_spmv

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def B():
    import paper_2307_00124_b200 as B
    B.lib()
    return B


def gflat(B, blk: P.Block, mb=8):
    return B.BfpVec.from_mantissas(blk.m, blk.q, blk.e, mant_bytes=mb)


def ggrid(B, d, l, m, q, e, mb=4):
    return B.BfpVec.from_mantissas(list(map(int, m)), q, e, dim=d, level=l, mant_bytes=mb)


def gcsr(B, A: P.Csr):
    return B.BfpCsr(A.rows, A.cols, A.rowptr, A.col, A.m, A.q, A.e)


def S(b: P.Block):
    import paper_2307_00124_b200 as B
    return B.Scalar(b.m[0], b.q, b.e)


def same(gv, want_m, want_e, want_q=None):
    m, q, e = gv.download()
    assert m.tolist() == list(want_m), (m.tolist()[:8], list(want_m)[:8])
    assert e == want_e
    if want_q is not None:
        assert q == want_q


# ---------------------------------------------------------------------------
# known answers of the reference unit tests, through the GPU


def test_known_answers_gpu(B):
    with open(os.path.join(GOLD, "reference_known_answers.json")) as f:
        cases = json.load(f)["cases"]
    n_checked = 0
    for c in cases:
        op = c["op"]
        if op == "qcomp_rows":
            g = B.Scalar(*c["gamma"])
            res = B.qcomp_rows(c["rows"], c["tq"], c["te"], c["w_out"], c["w_tmp"], g,
                               nn=bool(c.get("nn")))
            same(res.z, c["want"]["m"], c["want"]["e"], c["want"]["q"])
            if "flags" in c["want"]:
                assert [int(res.overflow), int(res.underflow), int(res.recomputed)] == c["want"]["flags"]
        elif op == "qcomp_error":
            with pytest.raises(B.InvalidArgument):
                B.qcomp_rows(c["rows"], c["tq"], c["te"], c["w_out"], c["w_tmp"],
                             B.Scalar(*c["gamma"]), nn=bool(c.get("nn")))
        elif op in ("normalize", "quantize"):
            x = B.BfpVec.from_mantissas(c["m"], c["q"], c["e"])
            r = B.normalize(x) if op == "normalize" else B.quantize(x, c["w"])
            same(r, c["want"]["m"], c["want"]["e"])
        elif op == "inf_norm_upper":
            x = B.BfpVec.from_mantissas(c["m"], c["q"], c["e"])
            g = B.inf_norm_upper(x, c["qg"])
            assert Fraction(g.m) * Fraction(2) ** g.e == c["want_value"][0]
        elif op == "spmv_row":
            a = c["a"]
            A = B.BfpCsr(a["rows"], a["cols"], a["rowptr"], a["col"], a["m"], a["q"], a["e"])
            res = B.qspmv(A, B.BfpVec.from_mantissas(*c["x"]), 8, 8, B.Scalar(1, 2, 0))
            assert res.z.mantissas().tolist() == c["want_rows"]
        elif op == "spmv_error":
            a = c["a"]
            A = B.BfpCsr(a["rows"], a["cols"], a["rowptr"], a["col"], a["m"], a["q"], a["e"])
            with pytest.raises(B.InvalidArgument):
                B.qspmv(A, B.BfpVec.from_mantissas(*c["x"]), 8, 8, B.Scalar(1, 2, 0), m_a=c["m_a"])
        elif op == "quantize_exact":  # from_extfloat [1, -0.5] w3
            r = B.quantize_exact(c["z"], c["k"], c["w"])
            same(r, c["want"]["m"], c["want"]["e"], c["w"])
            vals = [float(Fraction(z) * Fraction(2) ** k) for z, k in zip(c["z"], c["k"])]
            same(B.from_doubles(vals, c["w"]), c["want"]["m"], c["want"]["e"], c["w"])
        elif op == "axpby_row":
            x = B.BfpVec.from_mantissas(*c["x"])
            y = B.BfpVec.from_mantissas(*c["y"])
            res = B.qaxpby(x, y, B.Scalar(*c["alpha"]), B.Scalar(*c["beta"]), 60, 60,
                           B.Scalar(1, 2, 100))
            m, q, e = res.z.download()
            assert [Fraction(int(v)) * Fraction(2) ** e for v in m] == [w[0] for w in c["want_values"]]
        else:
            continue
        n_checked += 1
    assert n_checked >= 15


@pytest.mark.parametrize("mb", [4, 8])
def test_quantize_exact_gpu_vs_pyref(B, mb):
    """quantize_exact / from_extfloat on the device vs the big-int restatement (random
    signs, magnitudes, exponents and widths, zero entries and all-zero blocks)."""
    import math
    r = Rng(77 + mb)
    for it in range(60):
        n = r.uniform(0, 40)
        w = r.uniform(1, 31 if mb == 4 else 62)
        z = [0 if r.uniform(0, 4) == 0 else r.uniform(-(1 << 62), 1 << 62) >> r.uniform(0, 60)
             for _ in range(n)]
        if it % 10 == 0:
            z = [0] * n
        k = [r.uniform(-80, 80) for _ in range(n)]
        want = P.quantize_exact(z, k, w)
        same(B.quantize_exact(z, k, w, mant_bytes=mb), want.m, want.e, w)
        # doubles: z with at most 53 significant bits
        zd = [v >> max(0, v.bit_length() - 53) if v > 0 else -((-v) >> max(0, (-v).bit_length() - 53))
              for v in z]
        vals = [math.ldexp(float(a), b) for a, b in zip(zd, k)]
        want = P.quantize_exact(zd, k, w)
        same(B.from_doubles(vals, w, mant_bytes=mb), want.m, want.e, w)
    with pytest.raises(B.InvalidArgument):
        B.from_doubles([float("nan")], 4)


def test_domain_error_on_upload(B):
    with pytest.raises(B.DomainError):  # check_fits, src/bfp.cpp:11-14
        B.BfpVec.from_mantissas([8], 4, 0)


def test_dump_parse_roundtrip_gpu(B):
    r = Rng(25)
    for _ in range(30):
        v = r.random_vec(r.uniform(1, 9), r.uniform(1, 60), -40, 40, False)
        g = gflat(B, v)
        text = B.dump_block(g)
        assert text == P.dump_block(v)
        back = B.parse_block(text)
        same(back, v.m, v.e, v.q)


# ---------------------------------------------------------------------------
# generic CSR / axpby path vs the rational oracle and pyref


def test_qcomp_gemv_random_gpu(B):
    """tests/test_blas.cpp:239-261 and 263-306 replayed through the GPU."""
    r = Rng(35)
    for it in range(150):
        n = r.uniform(1, 16)
        w_out = r.uniform(2, 16)
        w_tmp = w_out + r.uniform(0, 6)
        x = r.random_vec(n, r.uniform(2, 16))
        y = r.random_vec(n, r.uniform(2, 16))
        A = r.random_csr(n, n, r.uniform(1, 8), r.uniform(2, 16))
        a = P.Block.scalar(r.in_width(6), 6, r.uniform(-3, 3))
        b = P.Block.scalar(r.in_width(6), 6, r.uniform(-3, 3))
        k = P.EgemvKernel(A, x, y, a, b)
        gamma = r.gamma_with_binade(k.tmpl.e + r.uniform(-2, k.tmpl.q + 2))
        want, fl = P.qcomp(k, w_out, w_tmp, gamma)
        rows = rational_axpby(a, rational_spmv(A, x.values()), b, y.values())
        wm, we = P.window_truncate(rows, k.tmpl.e, w_out)
        assert want.m == wm and want.e == we
        gx, gy, gA = gflat(B, x), gflat(B, y), gcsr(B, A)
        res = B.qgemv(gA, gx, gy, S(a), S(b), w_out, w_tmp, S(gamma), force=(it % 7 == 0))
        same(res.z, wm, we, w_out)
        if it % 7:
            assert (res.overflow, res.underflow) == (fl.overflow, fl.underflow)
        nn, _ = P.nnqcomp(k, w_out, gamma)
        res2 = B.nnqgemv(gA, gx, gy, S(a), S(b), w_out, S(gamma))
        same(res2.z, nn.m, nn.e, w_out)
        ks = P.EspmvKernel(A, x)
        want3, _ = P.qcomp(ks, w_out, w_tmp, gamma)
        same(B.qspmv(gA, gx, w_out, w_tmp, S(gamma)).z, want3.m, want3.e)
        # int32 storage path
        if w_tmp <= 32:
            gx4, gy4 = gflat(B, x, 4), gflat(B, y, 4)
            res4 = B.qaxpby(gx4, gy4, S(a), S(b), w_out, w_tmp, S(gamma))
            want4, _ = P.qcomp(P.EaxpbyKernel(x, y, a, b), w_out, w_tmp, gamma)
            same(res4.z, want4.m, want4.e)


def test_saturation_and_order_gpu(B):
    r = Rng(38)
    for _ in range(100):
        n = r.uniform(1, 12)
        w = r.uniform(2, 10)
        x = r.random_vec(n, r.uniform(2, 14))
        y = r.random_vec(n, r.uniform(2, 14))
        a3, m3 = P.Block.scalar(3, 3, 0), P.Block.scalar(-3, 3, 0)
        k = P.EaxpbyKernel(x, y, a3, m3)
        gamma = r.gamma_with_binade(k.tmpl.e + r.uniform(-4, k.tmpl.q + 4))
        want, _ = P.nnqcomp(k, w, gamma)
        res = B.nnqaxpby(gflat(B, x), gflat(B, y), S(a3), S(m3), w, S(gamma))
        same(res.z, want.m, want.e)
        hi = (1 << (w - 1)) - 1
        assert all(-hi - 1 <= v <= hi for v in res.z.mantissas().tolist())
    x = Rng(40).random_vec(6, 9)
    g = gflat(B, x)
    assert B.qsub(g, g, 5, 7, B.inf_norm_upper(g)).z.is_zero()
    eye = B.BfpCsr(6, 6, list(range(7)), list(range(6)), [1] * 6, 2, 0)
    nx = P.normalize(x)
    same(B.qspmv(eye, g, x.q, x.q + 2, B.inf_norm_upper(g)).z, nx.m, nx.e)


def test_dot_exact_gpu(B):
    r = Rng(77)
    for mb in (4, 8):
        n = 1000
        x = r.random_vec(n, 30 if mb == 4 else 60)
        y = r.random_vec(n, 30 if mb == 4 else 60)
        v, e = B.dot_exact(gflat(B, x, mb), gflat(B, y, mb))
        assert v == sum(a * b for a, b in zip(x.m, y.m)) and e == x.e + y.e


# ---------------------------------------------------------------------------
# grid operators vs the C oracle (chained so pending shifts are consumed)


def _oblock(g):
    m, q, e = g.download()
    return ob.OBlock(m, q, e)


@pytest.mark.parametrize("d,l,mb", [(1, 2, 4), (1, 9, 4), (1, 9, 8), (2, 2, 4), (2, 6, 4),
                                    (2, 6, 8), (3, 2, 4), (3, 4, 4), (3, 4, 8),
                                    # pipelined transfer kernels (3-D l >= 7, 2-D l >= 10)
                                    (1, 12, 4), (2, 9, 4), (2, 10, 4), (3, 7, 4),
                                    # 3-D transfer marches (coarse l >= 7), int32 and int64
                                    (3, 8, 4), (3, 8, 8)])
def test_grid_ops_gpu_vs_oracle(B, d, l, mb):
    r = Rng(1000 + 100 * d + 10 * l + mb)
    for it in range(3):
        p = r.uniform(6, 24 if mb == 4 else 44)
        gx = B.gen_uniform(B.BfpVec.grid(d, l, mb), p, it + 1, 1)
        gb = B.gen_uniform(B.BfpVec.grid(d, l, mb), p, it + 1, 2)
        ox, obb = ob.gen_uniform(d, l, p, it + 1, 1), ob.gen_uniform(d, l, p, it + 1, 2)
        same(gx, ox.m.tolist(), ox.e)
        if it == 2:
            gx.zero(p)
            ox = ob.OBlock(np.zeros(len(ox.m), np.int64), p, 0)
        w_out = r.uniform(3, min(p, 30 if mb == 4 else 60))
        w_tmp = w_out + r.uniform(0, 2)
        for mode in ("q", "nn"):
            nn = mode == "nn"
            g = r.gamma_with_binade(r.uniform(-10, 40))
            Sg = S(g)
            # residual r = b - A x, then feed the (possibly deferred-shift) result onward
            res = B.residual(gx, gb, w_out, w_tmp, Sg, nn=nn)
            want, wfl = ob.stencil_gemv(d, l, ox, obb, (-1, 1, 0), (1, 2, 0), mode, w_out, w_tmp,
                                        g.m[0], g.e)
            same(res.z, want.m.tolist(), want.e, w_out)
            if not nn:
                assert (res.overflow, res.underflow, res.recomputed) == tuple(map(bool, wfl))
            c = B.jacobi_coeff(d, l, 16)
            g2 = r.gamma_with_binade(r.uniform(-10, 40))
            j = B.jacobi(gx, res.z, c, w_out, w_tmp, S(g2), nn=nn)
            wj, _ = ob.jacobi(d, l, ox, want, (c.m, c.q, c.e), mode, w_out, w_tmp, g2.m[0], g2.e)
            same(j.z, wj.m.tolist(), wj.e)
            sc = B.scal(j.z, c, w_out, w_tmp, S(g2), nn=nn)
            ws, _ = ob.scal(wj, (c.m, c.q, c.e), mode, w_out, w_tmp, g2.m[0], g2.e)
            same(sc.z, ws.m.tolist(), ws.e)
            ax = B.qaxpby(j.z, sc.z, B.bfp_one(), B.bfp_minus_one(), w_out, w_tmp, S(g), nn=nn)
            wa, _ = ob.axpby(wj, ws, (1, 2, 0), (-1, 1, 0), mode, w_out, w_tmp, g.m[0], g.e)
            same(ax.z, wa.m.tolist(), wa.e)
            if l >= 3:
                rs = B.restrict_fw(res.z, w_out, w_tmp, S(g2), nn=nn)
                wr, _ = ob.restrict(d, l, want, mode, w_out, w_tmp, g2.m[0], g2.e)
                same(rs.z, wr.m.tolist(), wr.e)
                pr = B.prolong(rs.z, w_out, w_tmp, S(g), nn=nn)
                wp, _ = ob.prolong(d, l, wr, mode, w_out, w_tmp, g.m[0], g.e)
                same(pr.z, wp.m.tolist(), wp.e)
                pc = B.prolong_correct(rs.z, j.z, w_out, w_tmp, S(g2), nn=nn)
                wpc, _ = ob.prolong_correct(d, l, wr, wj, mode, w_out, w_tmp, g2.m[0], g2.e)
                same(pc.z, wpc.m.tolist(), wpc.e)


@pytest.mark.parametrize("d,l,p", [(1, 10, 16), (2, 6, 20), (3, 4, 24), (2, 5, 4), (3, 3, 48)])
def test_generators_gpu_vs_oracle(B, d, l, p):
    mb = 8 if p > 30 else 4
    g = B.gen_sine(B.BfpVec.grid(d, l, mb), p)
    o = ob.gen_sine(d, l, p)
    same(g, o.m.tolist(), o.e, p)
    g = B.gen_uniform(B.BfpVec.grid(d, l, mb), p, 5, 9)
    o = ob.gen_uniform(d, l, p, 5, 9)
    same(g, o.m.tolist(), o.e, p)


# ---------------------------------------------------------------------------
# solver: golden fixtures, larger configs vs the C oracle, graph replay


def _mg_gpu(B, cfgkw, p, graph=False):
    mg = B.Multigrid(B.mg_config(**cfgkw, p=p))
    mg.solve(use_graph=graph)
    return mg.result()


def _sha(m):
    return hashlib.sha256(",".join(map(str, list(m))).encode()).hexdigest()


def test_mg_golden_gpu(B):
    with open(os.path.join(GOLD, "mg_small.json")) as f:
        cases = json.load(f)["cases"]
    for case in cases:
        cfg = dict(case["config"])
        p = cfg.pop("p")
        for graph in (False, True):
            x, q, e, hist, tr = _mg_gpu(B, cfg, p, graph)
            assert e == case["x_e"] and q == case["x_q"], case["name"]
            assert _sha(x.tolist()) == case["x_sha256"], case["name"]
            assert hist == case["history"], case["name"]
            assert [list(t) for t in tr] == case["trace"], case["name"]


@pytest.mark.parametrize("name,cfgkw,p", [
    ("c1", dict(d=1, l_fine=14, cycles=10, x0_random=True, rhs_kind=0, pd=[28] * 32,
                w_add_cap=4), 16),
    ("c1_flat16", dict(d=1, l_fine=12, cycles=6, x0_random=True, rhs_kind=0), 16),
    ("c2", dict(d=2, l_fine=8, cycles=15, rhs_kind=1), 20),
    ("c3", dict(d=2, l_fine=9, l_coarse=3, cycles=1, rhs_kind=1, fmg=True, nonnormalized=True),
     [0, 0, 0] + [4 + 2 * (l - 3) for l in range(3, 32)][:29]),
    ("c2_hybrid", dict(d=2, l_fine=8, cycles=6, rhs_kind=1, nonnormalized="hybrid"), 20),
    ("c4", dict(d=3, l_fine=6, cycles=1, rhs_kind=1, fmg=True), 24),
    ("c5", dict(d=3, l_fine=5, cycles=3, x0_random=True, rhs_kind=2), 48),
    # the V(nu1, nu2) x n_ir variants of the FMG time-to-accuracy sweep (tools/fmg_sweep.py)
    ("c4_v21_n2", dict(d=3, l_fine=6, cycles=2, rhs_kind=1, fmg=True, nu2=1), 24),
    ("c4_v10_n3_nc4", dict(d=3, l_fine=5, cycles=3, rhs_kind=1, fmg=True, nu1=1, nu2=0,
                           n_coarse=4), 24),
    ("c2_v12", dict(d=2, l_fine=7, cycles=3, rhs_kind=1, nu1=1, nu2=2), 20),
])
def test_mg_gpu_vs_oracle(B, name, cfgkw, p):
    ox, oh, otr = ob.mg_run(ob.mg_config(**cfgkw, p=p))
    for fuse in (0, 4096):  # per-op launches, and the shared-memory fused bottom levels
        x, q, e, hist, tr = _mg_gpu(B, dict(cfgkw, fuse_points=fuse), p, graph=True)
        assert e == ox.e and q == ox.q, fuse
        assert x.tolist() == ox.m.tolist(), fuse
        assert hist == oh, fuse
        assert [tuple(t) for t in tr] == [tuple(t) for t in otr], fuse
    x, q, e, hist, tr = _mg_gpu(B, cfgkw, p, graph=True)
    assert e == ox.e and q == ox.q
    assert x.tolist() == ox.m.tolist()
    assert hist == oh
    assert [tuple(t) for t in tr] == [tuple(t) for t in otr]


# ---------------------------------------------------------------------------
# full-size (BASELINE.json config 2) residual: bit-exact against the oracle


def test_full_size_residual_c2(B):
    d, l, p = 2, 12, 20
    gx = B.gen_uniform(B.BfpVec.grid(d, l, 4), p, 1, 1)
    gb = B.gen_sine(B.BfpVec.grid(d, l, 4), p)
    ox, obb = ob.gen_uniform(d, l, p, 1, 1), ob.gen_sine(d, l, p)
    for g in (B.Scalar(1 << 14, 16, 20), B.Scalar(1 << 14, 16, 30), B.Scalar(1 << 14, 16, 0)):
        res = B.residual(gx, gb, p, p + 5, g)
        want, fl = ob.stencil_gemv(d, l, ox, obb, (-1, 1, 0), (1, 2, 0), "q", p, p + 5, g.m, g.e)
        m, q, e = res.z.download()
        assert e == want.e and np.array_equal(m, want.m)
        assert (res.overflow, res.underflow) == (bool(fl[0]), bool(fl[1]))


@pytest.mark.parametrize("d,l,mb,p", [(2, 10, 4, 20), (2, 11, 4, 20), (3, 7, 4, 20),
                                      (3, 8, 4, 20), (3, 7, 8, 40), (3, 7, 8, 52)])
def test_stencil_paths_agree_with_oracle(B, d, l, mb, p):
    """Stencil ops through the bulk-async pipelines (2-D N >= 1024, 3-D N >= 128, int32
    and int64 storage, int64 / int128 rows) and through the register march / generic
    grid kernel are both bit-exact vs the oracle (qcomp fast / recompute, nnqcomp)."""
    ox, ob_ = ob.gen_uniform(d, l, p, 3, 1), ob.gen_sine(d, l, p)
    c = B.jacobi_coeff(d, l, 16)
    try:
        for bulk in (True, False):
            B.set_kernel_path(bulk)
            gx = B.gen_uniform(B.BfpVec.grid(d, l, mb), p, 3, 1)
            gb = B.gen_sine(B.BfpVec.grid(d, l, mb), p)
            for g, nn in ((B.Scalar(1 << 14, 16, 2 * l + 2), False), (B.Scalar(1 << 14, 16, 0), False),
                          (B.Scalar(1 << 14, 16, 2 * l + 2), True)):
                mode = "nn" if nn else "q"
                res = B.residual(gx, gb, p, p + 5, g, nn=nn)
                want, fl = ob.stencil_gemv(d, l, ox, ob_, (-1, 1, 0), (1, 2, 0), mode, p, p + 5,
                                           g.m, g.e)
                m, q, e = res.z.download()
                assert e == want.e and np.array_equal(m, want.m), (bulk, g, nn)
                j = B.jacobi(gx, res.z, c, p, p + 5, g, nn=nn)
                wj, _ = ob.jacobi(d, l, ox, want, (c.m, c.q, c.e), mode, p, p + 5, g.m, g.e)
                m, q, e = j.z.download()
                assert e == wj.e and np.array_equal(m, wj.m), (bulk, "jacobi", g, nn)
    finally:
        B.set_kernel_path(True)


@pytest.mark.parametrize("p", [40, 48, 52])
def test_int64_residual_windows_vs_oracle(B, p):
    """3-D int64 residuals through the bulk pipeline over the window regimes of the
    split-window path (SplitWin, bfp_kernels.cuh): alignment d of both signs (X/Y swap),
    window shift rs above and below |d|, rows all in {0, -1} (mu* from the low words),
    rs >= 64 / left-shift windows (the two-word fallback), overflow and underflow."""
    d, l = 3, 7
    ox, obb = ob.gen_uniform(d, l, p, 5, 1), ob.gen_sine(d, l, p)
    gx = ggrid(B, d, l, ox.m, ox.q, ox.e, mb=8)
    for off in (-40, -12, 0, 9, 30):
        bo = ob.OBlock(obb.m, obb.q, obb.e + off)
        gb = ggrid(B, d, l, bo.m, bo.q, bo.e, mb=8)
        for ge in range(-70, 80, 9):
            g = B.Scalar(1 << 14, 16, ge)
            res = B.residual(gx, gb, p, p + 5, g)
            want, fl = ob.stencil_gemv(d, l, ox, bo, (-1, 1, 0), (1, 2, 0), "q", p, p + 5,
                                       g.m, g.e)
            m, q, e = res.z.download()
            assert e == want.e and np.array_equal(m, want.m), (off, ge)
            assert (res.overflow, res.underflow) == (bool(fl[0]), bool(fl[1])), (off, ge)


@pytest.mark.parametrize("p", [32, 40, 48, 52])
def test_int64_jacobi_windows_vs_oracle(B, p):
    """3-D int64 Jacobi updates through the bulk pipeline over the regimes of the
    three-limb split window (JacobiOp::point_sp, bfp_ops.cuh): b ahead of and behind the
    stencil term (d1 of both signs, beyond +-31 for the two-word fallback), x aligned above
    and below limb 1 (d2 around 32), window shift rs around 32, coefficients of 8..30 bits,
    overflow and underflow flags."""
    d, l = 3, 7
    ox, obb = ob.gen_uniform(d, l, p, 5, 1), ob.gen_sine(d, l, p)
    gx = ggrid(B, d, l, ox.m, ox.q, ox.e, mb=8)
    done = 0
    for off in (-45, -20, -6, 0, 7, 25, 40):
        bo = ob.OBlock(obb.m, obb.q, obb.e + off)
        gb = ggrid(B, d, l, bo.m, bo.q, bo.e, mb=8)
        for qc, ge in ((8, 4), (16, -30), (16, 0), (16, 12), (24, 5), (30, 20), (16, 60)):
            c = B.jacobi_coeff(d, l, qc)
            g = B.Scalar(1 << 14, 16, ge)
            try:
                j = B.jacobi(gx, gb, c, p, p + 3, g)
            except B.WidthError:  # exact row beyond 127 bits: outside the product's range
                assert p >= 40 and abs(off) >= 25, (off, qc, ge)
                continue
            done += 1
            wj, fl = ob.jacobi(d, l, ox, bo, (c.m, c.q, c.e), "q", p, p + 3, g.m, g.e)
            m, q, e = j.z.download()
            assert e == wj.e and np.array_equal(m, wj.m), (off, qc, ge)
            assert (j.overflow, j.underflow) == (bool(fl[0]), bool(fl[1])), (off, qc, ge)
    assert done >= 30


@pytest.mark.parametrize("l", [18, 20, 24])
def test_1d_wide_alignment_residual_vs_oracle(B, l):
    """1-D residuals at config-1 scale and beyond: h^-2 = 2^{2l} puts A x ~2l bits above
    b (alignment d = 2l + e_x - e_b >= 31), the 32-bit-operand path with a 64-bit
    alignment shift (GemvOp::wsh); uniform x and b (config 1), window regimes from
    underflow to overflow, and the swapped alignment (b scaled far above A x)."""
    d, p = 1, 16
    ox, obu = ob.gen_uniform(d, l, p, 1, 1), ob.gen_uniform(d, l, p, 1, 2)
    gx = ggrid(B, d, l, ox.m, ox.q, ox.e)
    for off in (0, 2 * l + 40):
        bo = ob.OBlock(obu.m, obu.q, obu.e + off)
        gb = ggrid(B, d, l, bo.m, bo.q, bo.e)
        for ge in (2 * l + off - 12, 2 * l + off + 2, 2 * l + off + 20, 0):
            g = B.Scalar(1 << 14, 16, ge)
            res = B.residual(gx, gb, p, p + 5, g)
            want, fl = ob.stencil_gemv(d, l, ox, bo, (-1, 1, 0), (1, 2, 0), "q", p, p + 5,
                                       g.m, g.e)
            m, q, e = res.z.download()
            assert e == want.e and np.array_equal(m, want.m), (off, ge)
            assert (res.overflow, res.underflow) == (bool(fl[0]), bool(fl[1])), (off, ge)
            nn = B.residual(gx, gb, p, p + 5, g, nn=True)
            wn, _ = ob.stencil_gemv(d, l, ox, bo, (-1, 1, 0), (1, 2, 0), "nn", p, p + 5, g.m, g.e)
            m, q, e = nn.z.download()
            assert e == wn.e and np.array_equal(m, wn.m), ("nn", off, ge)


def test_c1_solve_full_size_vs_oracle(B):
    """BASELINE config 1 at its full size (2^20 - 1 points, 10 IR-V(2,2) cycles, the
    frozen wdot = 28 schedule): iterate, residual history and trace bit-exact."""
    kw = dict(d=1, l_fine=20, cycles=10, x0_random=True, rhs_kind=0, w_add_cap=4)
    ox, oh, otr = ob.mg_run(ob.mg_config(**kw, p=16, pd=28))
    mg = B.Multigrid(B.mg_config(**kw, p=16, pd=[28] * 32))
    mg.solve(use_graph=True)
    x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
    assert e == ox.e and x.tolist() == ox.m.tolist()
    assert hist == oh
    assert [tuple(t) for t in tr] == [tuple(t) for t in otr]
