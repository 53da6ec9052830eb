"""FEM load vectors of the reference-algorithm mode: the oracle's
restatement of the reference's quadrature (oracle/pyref_refmode.py: fem_rhs) against the
closed form of the hat-function integrals, and the product's host code
(paper_2307_00124_b200/refmode.py: fem_rhs, 62-bit dyadics for bfp_quantize_exact) against
the oracle after quantisation.  Host only."""
import math

import pytest

mp = pytest.importorskip("mpmath")

from oracle import pyref as P  # noqa: E402
from oracle import pyref_refmode as R  # noqa: E402
from paper_2307_00124_b200 import refmode as H  # noqa: E402


@pytest.mark.parametrize("level,k", [(3, 3), (5, 2), (6, 3), (8, 3)])
def test_gauss_load_close_to_closed_form(level, k):
    """integral sin(k pi x) phi_i = 2 (1 - cos(k pi h)) / (k^2 pi^2 h) sin(k pi x_i) exactly;
    the 2-point Gauss rule per element is off by O((k pi h)^4) relative."""
    n = 1 << level
    h = 1.0 / n
    got = R._fem_load_1d(level, k, 200)
    assert len(got) == n - 1
    amp = 2 * (1 - math.cos(k * math.pi * h)) / (k * k * math.pi ** 2 * h)
    tol = (k * math.pi * h) ** 4 / 100 * amp + 1e-30
    for i, v in enumerate(got, start=1):
        assert abs(float(v) - amp * math.sin(k * math.pi * i * h)) <= tol, (i, float(v))


def test_two_point_rule_is_not_the_exact_integral():
    """The restatement follows the reference's quadrature, not the analytic load."""
    level, k = 3, 3
    h = 1.0 / (1 << level)
    got = float(R._fem_load_1d(level, k, 200)[0])
    exact = 2 * (1 - math.cos(k * math.pi * h)) / (k * k * math.pi ** 2 * h) * math.sin(k * math.pi * h)
    assert abs(got - exact) > 1e-6 * abs(exact)


@pytest.mark.parametrize("d,level,w", [(1, 4, 12), (1, 7, 24), (1, 9, 44), (1, 6, 62),
                                       (2, 3, 16), (2, 5, 24), (2, 4, 60)])
def test_host_dyadics_quantise_to_the_oracle_block(d, level, w):
    want = R.fem_rhs(d, level, w)
    z, k = H.fem_rhs(d, level)
    assert all(abs(v) < 1 << 62 for v in z)
    got = P.quantize_exact(z, k, w)
    assert (got.q, got.e) == (want.q, want.e)
    assert got.m == want.m
    n = ((1 << level) - 1) ** d
    assert len(got.m) == n and max(abs(v) for v in got.m) >= 1 << (w - 2)


def test_symmetric_zeros_are_exact_zeros():
    """sin(2 pi x) phi_i vanishes at x_i = 1/2 by symmetry: the row i1 = n/2 of the 2-D load
    (all of level 1) is exactly zero, not 2^-prec rounding noise with an exponent of -500."""
    assert R.fem_rhs(2, 1, 24).m == [0] and R.fem_rhs(2, 1, 24).e == 0
    z, k = H.fem_rhs(2, 1)
    assert z == [0]
    level = 3
    n = (1 << level) - 1
    blk = R.fem_rhs(2, level, 24)
    mid = n // 2
    assert all(blk.m[mid * n + i2] == 0 for i2 in range(n))
    assert any(blk.m[(mid - 1) * n + i2] != 0 for i2 in range(n))


def test_precision_insensitive():
    """440 vs 600 bits of working precision give the same blocks (the reference's 400-bit
    roundings are far below every quantisation boundary met here)."""
    for d, level, w in ((1, 6, 40), (2, 4, 30)):
        a, b = R.fem_rhs(d, level, w, prec=440), R.fem_rhs(d, level, w, prec=600)
        assert (a.e, a.m) == (b.e, b.m)


def test_2d_load_is_the_outer_product_slow_index_first():
    """b[i1 n + i2] = 13 pi^2 l2[i1] l3[i2] / (8/3): the slow index carries sin(2 pi .)."""
    level, w = 4, 30
    n = (1 << level) - 1
    blk = R.fem_rhs(2, level, w)
    v = [m * 2.0 ** blk.e for m in blk.m]
    h = 1.0 / (1 << level)
    i1, i2 = 3, 5
    ratio = v[i1 * n + i2] / v[(i1 + 1) * n + i2]
    assert abs(ratio - math.sin(2 * math.pi * (i1 + 1) * h) / math.sin(2 * math.pi * (i1 + 2) * h)) < 1e-3
