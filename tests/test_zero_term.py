"""All-zero eaxpby terms (axpby_setup_z in oracle/bfp_oracle.c and csrc/bfp_ops.cuh).

When one term of an eaxpby/egemv template is zero on every row, the C oracle and the
device drop it together with its alignment shift: the rows become the reference rows
/ 2^zd and qcomp/nnqcomp run in those shifted coordinates.  That keeps the rows within
the 127-bit accumulators where the reference's mpz rows are merely long (a zero
right-hand side at e = 0 next to a diverging iterate: BASELINE config 5 at p = 4).
Checked here against pyref, which keeps the reference templates and unbounded
integers: random far-apart exponents, the all-zero qcomp anchor (mu* = 1 in the
reference's coordinates, P/src/blas.cpp:153, tests/test_blas.cpp:363-368) through a
singular operator, and diverging solves whose exponents pass 127 bits."""
import numpy as np
import pytest

from oracle import ob
from oracle import pyref as P
from tests.cases import Rng


def ob_block(b: P.Block) -> ob.OBlock:
    return ob.OBlock(np.array(b.m, dtype=np.int64), b.q, b.e)


def ob_csr(A: P.Csr) -> ob.OCsr:
    return ob.OCsr(A.rows, A.cols, A.rowptr, A.col, A.m, A.q, A.e)


def second_difference(n: int) -> P.Csr:
    """[1, -2, 1] rows (tests/test_blas.cpp:201-212): A * const = 0 on interior rows."""
    rowptr, col, m = [0], [], []
    for i in range(n):
        for c, v in ((i - 1, 1), (i, -2), (i + 1, 1)):
            if 0 <= c < n:
                col.append(c)
                m.append(v)
        rowptr.append(len(col))
    return P.Csr(n, n, rowptr, col, m, 3, 0)


def cases(seed=71, count=120):
    """(A, x, y, alpha, beta, w_out, w_tmp, gamma): one term all-zero, exponents far apart."""
    r = Rng(seed)
    for it in range(count):
        n = r.uniform(1, 12)
        w_out = r.uniform(2, 16)
        w_tmp = w_out + r.uniform(0, 6)
        far = r.uniform(-300, 300)
        a = P.Block.scalar(r.in_width(6) or 1, 6, r.uniform(-3, 3))
        b = P.Block.scalar(r.in_width(6) or 1, 6, r.uniform(-3, 3))
        kind = it % 4
        if kind == 3:  # singular A on a constant x: every interior row is exactly zero
            n = r.uniform(3, 12)
            A = second_difference(n)
            A = P.Csr(A.rows, A.cols, A.rowptr, A.col, A.m, A.q, r.uniform(-8, 8))
            # boundary rows are nonzero unless they are dropped: keep only interior rows
            rows = list(range(1, n - 1))
            rowptr, col, m = [0], [], []
            for i in rows:
                col += A.col[A.rowptr[i]:A.rowptr[i + 1]]
                m += A.m[A.rowptr[i]:A.rowptr[i + 1]]
                rowptr.append(len(col))
            A = P.Csr(len(rows), n, rowptr, col, m, A.q, A.e)
            c = r.in_width(8) or 3
            x = P.Block([c] * n, 8, r.uniform(-8, 8))
            y = P.Block([0] * len(rows), r.uniform(2, 12), far)
        else:
            A = r.random_csr(n, n, r.uniform(1, 6), r.uniform(2, 12))
            x = r.random_vec(n, r.uniform(2, 12))
            y = P.Block([0] * n, r.uniform(2, 12), far)
            if kind == 1:  # the zero term is alpha*A*x instead
                x, y = P.Block([0] * n, r.uniform(2, 12), far), r.random_vec(n, r.uniform(2, 12))
            if kind == 2:  # alpha = 0 with a nonzero x
                a = P.Block.scalar(0, 6, r.uniform(-3, 3))
                y = r.random_vec(n, r.uniform(2, 12), e_lo=far - 4, e_hi=far + 4)
        k = P.EgemvKernel(A, x, y, a, b)
        gamma = r.gamma_with_binade(k.tmpl.e + r.uniform(-4, k.tmpl.q + 4))
        yield it, A, x, y, a, b, w_out, w_tmp, gamma, k


def sc(s: P.Block):
    return (s.m[0], s.q, s.e)


def test_zero_term_oracle_vs_pyref():
    """The oracle's shifted-coordinate windows equal pyref's reference-template windows
    (mantissas, exponent, flags), for qcomp, forced qcomp and nnqcomp."""
    anchors = 0
    for it, A, x, y, a, b, w_out, w_tmp, gamma, k in cases():
        for force in (False, True):
            want, fl = P.qcomp(k, w_out, w_tmp, gamma, force_recompute=force)
            got, gfl = ob.gemv(ob_csr(A), ob_block(x), ob_block(y), sc(a), sc(b), "q", w_out,
                               w_tmp, gamma.m[0], gamma.e, force=force)
            assert got.m.tolist() == want.m and got.e == want.e, (it, force)
            assert gfl[:2] == (fl.overflow, fl.underflow), (it, force)
        anchors += all(v == 0 for v in want.m)
        nn, _ = P.nnqcomp(k, w_out, gamma)
        got, _ = ob.gemv(ob_csr(A), ob_block(x), ob_block(y), sc(a), sc(b), "nn", w_out, w_out,
                         gamma.m[0], gamma.e)
        assert got.m.tolist() == nn.m and got.e == nn.e, it
    assert anchors >= 20  # the all-zero anchor is exercised


@pytest.mark.parametrize("d,l,cycles", [(1, 10, 30), (2, 6, 30)])
def test_diverging_solve_past_127_bits_oracle_vs_pyref(d, l, cycles):
    """BASELINE config 5's flat p = 4 schedule diverges; the iterate's
    exponent passes 127 bits (1-D: e = 454) and the oracle still follows pyref exactly:
    iterate, residual history and every trace record."""
    cfg = P.MgConfig(d=d, l_fine=l, cycles=cycles, x0_random=True, rhs_kind=2, p=[4] * 32)
    want = P.Mg(cfg).run()
    x, hist, tr = ob.mg_run(ob.mg_config(d, l, cycles=cycles, x0_random=True, rhs_kind=2, p=4))
    assert x.e == want.x.e and x.m.tolist() == list(want.x.m)
    assert hist == want.history
    assert [tuple(t) for t in tr] == [tuple(t) for t in want.trace]
    assert x.e + 2 * l > 127  # the unelided residual template would need > 127 bits


# ---------------------------------------------------------------------------
# the device path


@pytest.fixture(scope="module")
def B():
    import paper_2307_00124_b200 as B
    B.lib()
    return B


@pytest.mark.gpu
def test_zero_term_gpu_vs_pyref(B):
    def S(s):
        return B.Scalar(s.m[0], s.q, s.e)

    def gv(blk, mb=8):
        return B.BfpVec.from_mantissas(blk.m, blk.q, blk.e, mant_bytes=mb)

    for it, A, x, y, a, b, w_out, w_tmp, gamma, k in cases():
        gA = B.BfpCsr(A.rows, A.cols, A.rowptr, A.col, A.m, A.q, A.e)
        want, fl = P.qcomp(k, w_out, w_tmp, gamma)
        res = B.qgemv(gA, gv(x), gv(y), S(a), S(b), w_out, w_tmp, S(gamma))
        m, q, e = res.z.download()
        assert m.tolist() == want.m and e == want.e, it
        assert (res.overflow, res.underflow) == (fl.overflow, fl.underflow), it
        nn, _ = P.nnqcomp(k, w_out, gamma)
        m, q, e = B.nnqgemv(gA, gv(x), gv(y), S(a), S(b), w_out, S(gamma)).z.download()
        assert m.tolist() == nn.m and e == nn.e, it
        if A.rows == x.rows and x.rows == y.rows and w_tmp <= 32:  # pointwise, int32 storage
            kx = P.EaxpbyKernel(x, y, a, b)
            want4, fl4 = P.qcomp(kx, w_out, w_tmp, gamma)
            r4 = B.qaxpby(gv(x, 4), gv(y, 4), S(a), S(b), w_out, w_tmp, S(gamma))
            m, q, e = r4.z.download()
            assert m.tolist() == want4.m and e == want4.e, it


@pytest.mark.gpu
@pytest.mark.parametrize("d,l,cycles,p", [(1, 10, 30, 4), (2, 6, 30, 4), (3, 6, 10, 4),
                                          (3, 5, 10, 8)])
def test_diverging_solve_gpu_vs_oracle(B, d, l, cycles, p):
    """The flat-p config-5 schedule on the device (graph replay), bit-exact with the
    oracle while the exponents run past 127 bits."""
    kw = dict(d=d, l_fine=l, cycles=cycles, x0_random=True, rhs_kind=2)
    ox, oh, otr = ob.mg_run(ob.mg_config(**kw, p=p))
    mg = B.Multigrid(B.mg_config(**kw, p=p))
    mg.solve(use_graph=True)
    x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
    assert e == ox.e and x.tolist() == ox.m.tolist()
    assert hist == oh
    assert [tuple(t) for t in tr] == [tuple(t) for t in otr]
