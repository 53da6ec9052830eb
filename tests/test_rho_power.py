"""rho by power iteration (Hierarchy::setup_scaling): the oracle's exact-rational restatement
(oracle/pyref_refmode.py: power_rho) against the product's host code (refmode.estimate_rho,
mpmath) -- both correctly rounded, so bit-identical -- and against the true lambda_max."""
import math
from fractions import Fraction

import pytest

pytest.importorskip("mpmath")

from oracle import pyref_refmode as R  # noqa: E402
from paper_2307_00124_b200 import refmode as H  # noqa: E402


@pytest.mark.parametrize("d,l_est,iters", [(1, 3, 400), (1, 5, 400), (2, 2, 400), (2, 3, 60)])
def test_host_rho_equals_oracle(d, l_est, iters):
    want = R.power_rho(d, l_est, max_iter=iters)
    got = H.estimate_rho(d, l_est, max_iter=iters)
    assert isinstance(got, Fraction) and got == want
    assert got.numerator.bit_length() <= 400  # a 400-bit value


def test_rho_brackets_lambda_max_1d():
    """lambda_max(D^-1 A) = 1 + cos(pi h); after 400 iterations the Rayleigh quotient is
    within 1% below it, so rho = 1.01 lambda_400 lands within [0.995, 1.01] lambda_max."""
    for l in (3, 5):
        lmax = 1 + math.cos(math.pi / (1 << l))
        rho = float(H.estimate_rho(1, l))
        assert 0.995 * lmax <= rho <= 1.01 * lmax + 1e-12, (l, rho, lmax)


def test_early_stop_on_tiny_level():
    """Level 1 (one unknown): the quotient is exact at once and the relative-change stop
    fires at it = 3 -- rho = 1.01 rounded up."""
    rho = H.estimate_rho(1, 1)
    assert rho == R.power_rho(1, 1)
    assert abs(float(rho) - 1.01) < 1e-15
