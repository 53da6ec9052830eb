"""Exact BFP dot product <x, y> (csrc/op_dot.cu, config 5's 128-bit
exact dot): the device's 192-bit accumulation against exact Python integers.

* random int64 mantissas (p = 62) on a 511^3 grid, both signs;
* same-sign near-maximal mantissas: n >= 64 products of 62-bit values leave 128 bits
  (bfp_dot_exact raises WidthError, the 192-bit entry point is exact), and the 1023^3
  grid at the largest int64 mantissa (the config-5 extreme, ~2^154);
* the stream-ordered entry point inside a captured CUDA graph;
* the sharded dot (in-process rank group over z-slabs, int64 limb SUM) equals the
  unsharded one for P = 2, 4, 8.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def exact_dot_np(a, b):
    """sum_i a_i b_i exactly for int64 arrays (21-bit pieces, int64 chunk sums)."""
    a = np.asarray(a, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    M = (1 << 21) - 1
    pa = [a & M, (a >> 21) & M, a >> 42]
    pb = [b & M, (b >> 21) & M, b >> 42]
    total = 0
    CH = 1 << 18
    for i in range(3):
        for j in range(3):
            s = 0
            for c in range(0, len(a), CH):
                s += int(np.sum(pa[i][c:c + CH] * pb[j][c:c + CH], dtype=np.int64))
            total += s << (21 * (i + j))
    return total


def test_dot_random_int64_511(gpu):
    B = gpu
    x = B.gen_uniform(B.BfpVec.grid(3, 9, 8), 62, 11, 1)
    y = B.gen_uniform(B.BfpVec.grid(3, 9, 8), 62, 12, 1)
    mx, _, ex = x.download()
    my, _, ey = y.download()
    want = exact_dot_np(mx, my)
    v, e = B.dot_exact(x, y)
    assert v == want and e == ex + ey
    if -(1 << 127) <= want < (1 << 127):
        assert B.dot_exact128(x, y)[0] == want
    else:
        with pytest.raises(B.WidthError):
            B.dot_exact128(x, y)


@pytest.mark.parametrize("n", [64, 100, 4096])
def test_dot_same_sign_beyond_128_bits(gpu, n):
    """same-sign 62-bit mantissas; n >= 64 such products exceed 2^127."""
    B = gpu
    m = (1 << 62) - 1 - np.arange(n, dtype=np.int64) * 7
    x = B.BfpVec.from_mantissas(m.tolist(), 63, -3)
    y = B.BfpVec.from_mantissas((-m).tolist(), 63, 5)
    want = -sum(int(v) * int(v) for v in m)
    v, e = B.dot_exact(x, y)
    assert v == want and e == 2
    assert want < -(1 << 127)
    with pytest.raises(B.WidthError):
        B.dot_exact128(x, y)
    # below the boundary the 128-bit entry point is exact
    k = 8
    xs = B.BfpVec.from_mantissas(m[:k].tolist(), 63, 0)
    ys = B.BfpVec.from_mantissas(m[:k].tolist(), 63, 0)
    assert B.dot_exact128(xs, ys)[0] == sum(int(v) * int(v) for v in m[:k])


def test_dot_1023_extreme(gpu):
    """Config 5's grid (1023^3) at the largest int64 mantissa: n (2^62 - 1)^2 ~ 2^154."""
    B = gpu
    n = 1023 ** 3
    mval = (1 << 62) - 1
    x = B.BfpVec.grid(3, 10, 8)
    x.upload(np.full(n, mval, dtype=np.int64), 63, 0)
    v, e = B.dot_exact(x, x)
    assert v == n * mval * mval and e == 0
    with pytest.raises(B.WidthError):
        B.dot_exact128(x, x)
    del x


def test_dot_async_in_graph(gpu):
    import torch
    B = gpu
    x = B.gen_uniform(B.BfpVec.grid(3, 7, 8), 60, 3, 1)
    y = B.gen_uniform(B.BfpVec.grid(3, 7, 8), 60, 4, 1)
    mx, _, ex = x.download()
    my, _, ey = y.download()
    want = exact_dot_np(mx, my)
    acc = torch.zeros(8, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            B.set_stream(s.cuda_stream)
            B.dot_exact_async(x, y, acc.data_ptr())
    finally:
        B.set_stream(None)
    for _ in range(3):
        acc.fill_(12345)
        g.replay()
        torch.cuda.synchronize()
        a = acc.cpu().tolist()
        assert B.dot_value(a) == want and a[4] == ex + ey


@pytest.mark.parametrize("P", [2, 4, 8])
def test_dist_dot_equals_unsharded(gpu, P):
    import torch
    B = gpu
    from paper_2307_00124_b200 import dist as Dm
    d, l = 3, 7
    x = B.gen_uniform(B.BfpVec.grid(d, l, 8), 61, 5, 1)
    y = B.gen_uniform(B.BfpVec.grid(d, l, 8), 61, 6, 1)
    want, e = B.dot_exact(x, y)
    n = (1 << l) - 1
    per = n * n
    mx, qx, ex = x.download()
    my, qy, ey = y.download()
    ops = B.DistOps(P)
    xs, ys = [], []
    for lo, hi in Dm.slab_ranges(l, P):
        a = B.BfpVec.slab(d, l, lo, hi, 8)
        a.upload(mx[lo * per: min(hi, n) * per], qx, ex)
        b = B.BfpVec.slab(d, l, lo, hi, 8)
        b.upload(my[lo * per: min(hi, n) * per], qy, ey)
        xs.append(a)
        ys.append(b)
    accs = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(P)]
    ops.dot(xs, ys, [a.data_ptr() for a in accs])
    torch.cuda.synchronize()
    for a in accs:
        v = a.cpu().tolist()
        assert B.dot_value(v) == want and v[4] == e
