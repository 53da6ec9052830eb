"""Host-side setup of the reference-algorithm mode (the scalars the reference's
Hierarchy::set_eta / apply_schedule derive, P/src/multigrid.cpp:183-193, 313-361):
Chebyshev coefficients from rho and eta in exact rational arithmetic, rounded to the
hierarchy precision like ExtFloat::from_mpq (round to nearest, P/src/extfloat.cpp:21-25),
the V-residual gamma factor add_up(2 c1, 1) / 4 (round up, :131-135), and c1 / c2
floor-quantised at each level's wdot (quantize_scalar_floor, :233-241)."""
from __future__ import annotations

from fractions import Fraction
from typing import List, Tuple


def _round(v: Fraction, prec: int, up: bool) -> Fraction:
    """|v| rounded to prec significant bits (up: toward +inf for v > 0; else nearest-even)."""
    if v == 0:
        return v
    neg = v < 0
    a = -v if neg else v
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    s = prec - 1 - e
    scaled = a * Fraction(2) ** s
    fl = scaled.numerator // scaled.denominator
    rem = scaled - fl
    if up:
        q = fl + (1 if rem > 0 else 0)
    else:
        q = fl + (1 if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl & 1) else 0)
    r = Fraction(q) / Fraction(2) ** s
    return -r if neg else r


def _zk(v: Fraction) -> Tuple[int, int]:
    den = v.denominator
    k = -(den.bit_length() - 1)
    assert den == 1 << (-k)
    return v.numerator, k


def _top128(v: Fraction) -> Tuple[int, int, int, int]:
    """(hi, lo, e, sticky): the top 128 bits of a positive dyadic value."""
    z, k = _zk(v)
    assert z > 0
    b = z.bit_length()
    sticky = 0
    if b > 128:
        s = b - 128
        sticky = int(z & ((1 << s) - 1) != 0)
        z >>= s
        k += s
    return z >> 64, z & ((1 << 64) - 1), k, sticky


def _floor_scalar(v: Fraction, w: int) -> Tuple[int, int, int]:
    """quantize_scalar_floor: m = floor(z 2^(k - e)), e = msb(z) + k - w."""
    z, k = _zk(v)
    if z == 0:
        return 0, w, 0
    mz = z.bit_length() + 1 if z > 0 else (-z - 1).bit_length() + 1
    e = mz + k - w
    s = e - k
    m = z >> s if s >= 0 else z << (-s)
    return m, w, e


def eta_rational(eta: float) -> Fraction:
    num = round(eta * 100.0)
    if abs(eta - num / 100.0) < 1e-12:
        return Fraction(num, 100)
    return Fraction(eta)


def chebyshev_scalars(rho: float, eta: float, prec: int, wdot: List[int]):
    r, et = Fraction(rho), eta_rational(eta)
    alpha = (1 + et) * r / 2
    c = (1 - et) * r / 2
    beta = alpha - c * c / (2 * alpha)
    c1 = _round(2 / beta, prec, False)
    c2 = _round(Fraction(-1) / (alpha * beta), prec, False)
    kres = _round(2 * c1 + 1, prec, True) / 4
    c1d = [_floor_scalar(c1, w) if w else (0, 1, 0) for w in wdot]
    c2d = [_floor_scalar(c2, w) if w else (0, 1, 0) for w in wdot]
    return _top128(c1), _top128(kres), c1d, c2d
