"""Sharded (z-slab) stencil ops on one GPU: P slabs run sequentially in one process
(LocalComm: device halo copies, local MAX of the partials), bit-exact against the
unsharded GPU op and the oracle.  Exercises the slab kernels, the partial window
and the finalize kernel of the multi-rank path."""
import numpy as np
import pytest

from oracle import ob

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import paper_2307_00124_b200 as B
    B.lib()
    return B


def _gather(slabs):
    parts, e0 = [], None
    for s in slabs:
        m, q, e = s.vec.download()
        parts.append(m)
        assert e0 is None or e == e0, "exponent differs between slabs"
        e0 = e
    return np.concatenate(parts), e0


def _scatter(B, D, full, d, l, ranges):
    """Slabs holding the planes of a full vector (generators normalise globally)."""
    m, q, e = full.download()
    n = (1 << l) - 1
    per_plane = n ** (d - 1)
    out = []
    for r, (lo, hi) in enumerate(ranges):
        v = B.BfpVec.slab(d, l, lo, hi)
        v.upload(m[lo * per_plane: min(hi, n) * per_plane], q, e)
        out.append(D.Slab(r, v))
    return out


@pytest.mark.parametrize("d,l,P", [(2, 11, 2), (2, 11, 4), (2, 10, 8), (3, 7, 2), (3, 7, 4),
                                   (2, 7, 4), (3, 7, 64)])
def test_sharded_stencil_matches_unsharded(B, d, l, P):
    from paper_2307_00124_b200 import dist as D
    p = 20
    be = D.GpuBackend()
    comm = D.LocalComm(be, P)
    ds = D.DistStencil(comm, be, n_local=P)
    ranges = D.slab_ranges(l, P)
    gx = B.gen_uniform(B.BfpVec.grid(d, l), p, 5, 1)
    gb = B.gen_sine(B.BfpVec.grid(d, l), p)
    xs = _scatter(B, D, gx, d, l, ranges)
    bs = _scatter(B, D, gb, d, l, ranges)
    assert np.array_equal(_gather(xs)[0], gx.download()[0])

    ox, obb = ob.gen_uniform(d, l, p, 5, 1), ob.gen_sine(d, l, p)
    c = B.jacobi_coeff(d, l, 16)
    g_exact = B.inf_norm_upper(B.residual(gx, gb, p, p + 5, B.Scalar(1 << 14, 16, 0)).z)
    for g, nn in ((g_exact, False),                            # exact binade: qcomp fast path
                  (B.Scalar(1 << 14, 16, 2 * l + 2), False),   # overestimate: underflow
                  (B.Scalar(1 << 14, 16, 0), False),           # overflow -> recompute stage
                  (B.Scalar(1 << 14, 16, 2 * l + 2), True)):   # nnqcomp
        outs = [D.Slab(r, B.BfpVec.slab(d, l, lo, hi)) for r, (lo, hi) in enumerate(ranges)]
        ds.gemv(xs, bs, B.bfp_minus_one(), B.bfp_one(), p, p + 5, g, outs, nn=nn)
        got, e = _gather(outs)
        ref = B.residual(gx, gb, p, p + 5, g, nn=nn)
        m, q, er = ref.z.download()
        assert e == er and np.array_equal(got, m), (d, l, P, g, nn)
        flags = {s.vec.flags for s in outs}
        assert flags == {ref.z.flags}
        if g is g_exact:
            assert not (ref.z.flags & B.FLAG_RECOMPUTED)  # the fast path really ran
        want, _ = ob.stencil_gemv(d, l, ox, obb, (-1, 1, 0), (1, 2, 0), "nn" if nn else "q", p,
                                  p + 5, g.m, g.e)
        assert e == want.e and np.array_equal(got, want.m)
        # a Jacobi sweep from the sharded residual
        js = [D.Slab(r, B.BfpVec.slab(d, l, lo, hi)) for r, (lo, hi) in enumerate(ranges)]
        ds.jacobi(xs, outs, c, p, p + 5, g, js, nn=nn)
        got, e = _gather(js)
        jref = B.jacobi(gx, ref.z, c, p, p + 5, g, nn=nn)
        m, q, er = jref.z.download()
        assert e == er and np.array_equal(got, m), ("jacobi", d, l, P, g, nn)


def test_slab_ranges():
    from paper_2307_00124_b200 import dist as D
    assert D.slab_ranges(9, 8) == [(64 * r, 64 * (r + 1)) for r in range(8)]
    with pytest.raises(ValueError):
        D.slab_ranges(3, 8)


@pytest.mark.parametrize("d,l,P", [(2, 11, 4), (3, 7, 2), (3, 7, 8), (3, 7, 64),
                                   (3, 8, 2), (3, 8, 4)])  # l = 8: slabs through the tiled-TMA march
def test_native_dist_ops_match_unsharded(B, d, l, P):
    """The native sharded ops (bfp_dist_*: halo, partial windows, MAX all-reduce and
    finalize enqueued in C++) equal the unsharded ops bit-exactly."""
    from paper_2307_00124_b200 import dist as D
    p = 20
    ranges = D.slab_ranges(l, P)
    gx = B.gen_uniform(B.BfpVec.grid(d, l), p, 5, 1)
    gb = B.gen_sine(B.BfpVec.grid(d, l), p)
    xs = [s.vec for s in _scatter(B, D, gx, d, l, ranges)]
    bs = [s.vec for s in _scatter(B, D, gb, d, l, ranges)]
    ops = B.DistOps(P)
    c = B.jacobi_coeff(d, l, 16)
    g_exact = B.inf_norm_upper(B.residual(gx, gb, p, p + 5, B.Scalar(1 << 14, 16, 0)).z)
    for g, nn in ((g_exact, False), (B.Scalar(1 << 14, 16, 2 * l + 2), False),
                  (B.Scalar(1 << 14, 16, 0), False), (B.Scalar(1 << 14, 16, 2 * l + 2), True)):
        outs = [B.BfpVec.slab(d, l, lo, hi) for (lo, hi) in ranges]
        ops.gemv(xs, bs, B.bfp_minus_one(), B.bfp_one(), p, p + 5, g, outs, nn=nn)
        got, e = _gather([D.Slab(r, v) for r, v in enumerate(outs)])
        ref = B.residual(gx, gb, p, p + 5, g, nn=nn)
        m, q, er = ref.z.download()
        assert e == er and np.array_equal(got, m), (d, l, P, g, nn)
        assert {v.flags for v in outs} == {ref.z.flags}
        js = [B.BfpVec.slab(d, l, lo, hi) for (lo, hi) in ranges]
        ops.jacobi(xs, outs, c, p, p + 5, g, js, nn=nn)
        got, e = _gather([D.Slab(r, v) for r, v in enumerate(js)])
        m, q, er = B.jacobi(gx, ref.z, c, p, p + 5, g, nn=nn).z.download()
        assert e == er and np.array_equal(got, m), ("jacobi", d, l, P, g, nn)


@pytest.mark.parametrize("P", [2, 4])
def test_native_dist_ops_int64_l8(B, P):
    """int64 storage (p = 40) at 3-D l = 8: the slabs (plane offset z0 > 0) run the tiled-TMA
    march with the split windows (residual: SplitWin, Jacobi: three limbs) and the 32-bit pad
    predicates; equal to the unsharded ops bit for bit."""
    from paper_2307_00124_b200 import dist as D
    d, l, p = 3, 8, 40
    ranges = D.slab_ranges(l, P)
    n = (1 << l) - 1
    per = n * n
    gx = B.gen_uniform(B.BfpVec.grid(d, l, 8), p, 5, 1)
    gb = B.gen_sine(B.BfpVec.grid(d, l, 8), p)

    def scatter(full):
        m, q, e = full.download()
        out = []
        for lo, hi in ranges:
            v = B.BfpVec.slab(d, l, lo, hi, 8)
            v.upload(m[lo * per: min(hi, n) * per], q, e)
            out.append(v)
        return out
    xs, bs = scatter(gx), scatter(gb)
    ops = B.DistOps(P)
    c = B.jacobi_coeff(d, l, 16)
    g_exact = B.inf_norm_upper(B.residual(gx, gb, p, p + 5, B.Scalar(1 << 14, 16, 0)).z)
    for g in (g_exact, B.Scalar(1 << 14, 16, 0)):
        outs = [B.BfpVec.slab(d, l, lo, hi, 8) for (lo, hi) in ranges]
        ops.gemv(xs, bs, B.bfp_minus_one(), B.bfp_one(), p, p + 5, g, outs)
        got, e = _gather([D.Slab(r, v) for r, v in enumerate(outs)])
        ref = B.residual(gx, gb, p, p + 5, g)
        m, q, er = ref.z.download()
        assert e == er and np.array_equal(got, m), (P, g)
        js = [B.BfpVec.slab(d, l, lo, hi, 8) for (lo, hi) in ranges]
        ops.jacobi(xs, outs, c, p, p + 3, g, js)
        got, e = _gather([D.Slab(r, v) for r, v in enumerate(js)])
        m, q, er = B.jacobi(gx, ref.z, c, p, p + 3, g).z.download()
        assert e == er and np.array_equal(got, m), ("jacobi", P, g)
