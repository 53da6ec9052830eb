"""Host-side mirror of the reference API (no GPU): PrecisionSchedule (P/src/multigrid.cpp:13-44),
TraceRecord::to_line / SolverTrace counters (:157-177), and the gamma text format of
ExtFloat::str(6) (mpfr "%.6Rg", P/src/extfloat.cpp:65-73)."""
from fractions import Fraction

import pytest

import paper_2307_00124_b200 as B


def test_precision_schedule_flat_affine_validate():
    s = B.PrecisionSchedule.flat(4, 24, 20, 16)
    assert s.levels() == 4 and s.w == [0, 20, 20, 20, 20] and s.wcheck[3] == 24 and s.wdot[1] == 16
    s.validate()
    a = B.PrecisionSchedule.affine(5, 1, 2, 6, 4, 3)
    # w_j = 2j + 4, wcheck_j = max(3j + 6, w_j), wdot_j = min(j + 3, w_j)  (:22-35)
    assert a.w == [0, 6, 8, 10, 12, 14]
    assert a.wcheck == [0, 9, 12, 15, 18, 21]
    assert a.wdot == [0, 4, 5, 6, 7, 8]
    a.validate()
    # the clamps keep the ordering even when the affine laws cross
    c = B.PrecisionSchedule.affine(3, 4, 1, -10, 2, 1)
    c.validate()
    assert all(c.wcheck[j] >= c.w[j] >= c.wdot[j] for j in range(1, 4))
    for bad in (B.PrecisionSchedule([0, 10], [0, 12], [0, 8]),   # wcheck < w
                B.PrecisionSchedule([0, 12], [0, 10], [0, 11]),  # wdot > w
                B.PrecisionSchedule([0, 12], [0, 10], [0, 0])):  # wdot < 1
        with pytest.raises(ValueError, match="level 1"):
            bad.validate()


def test_trace_record_to_line_and_counters():
    t = B.TraceRecord(5, 4, 28, 32, 30877, -11, 0, 1, 1, 1)
    assert t.to_line() == ("v-restrict level=4 w_out=28 w_tmp=32 gamma=15.0767 overflow=0 "
                           "underflow=1 recompute=1 normalized=1")
    tr = B.SolverTrace([(0, 3, 16, 21, 1 << 14, -3, 0, 0, 0, 1), (3, 3, 16, 18, 20000, -9, 1, 0, 1, 1),
                        (3, 2, 16, 18, 20000, -9, 0, 1, 1, 1), tuple(t.__dict__.values())])
    assert tr.calls_at_level(3) == 2 and tr.recomputes_at_level(3) == 1
    assert tr.calls_at_level(2) == 1 and tr.recomputes_at_level(2) == 1
    assert tr.calls_at_level(7) == 0
    assert tr.lines()[0].startswith("ir-residual level=3 w_out=16 w_tmp=21 gamma=2048 ")
    assert {r.step_name() for r in tr.records} <= B.REF_STEP_NAMES


@pytest.mark.parametrize("gm,ge,want", [
    (1 << 14, -14, "1"), (3, 0, "3"), (32767, -5, "1023.97"), (1 << 14, -414, "3.87259e-121"),
    (30877, -11, "15.0767"), (1 << 14, 6, "1.04858e+06"), (12345, 0, "12345"),
    (1 << 14, 2000, "1.8811e+606"), (25000, -1100, "1.84054e-327"),
])
def test_gamma_str_matches_percent_g(gm, ge, want):
    assert B.gamma_str(gm, ge) == want
    v = Fraction(gm) * Fraction(2) ** ge
    try:
        f = float(v)
    except OverflowError:
        return
    if f != 0.0 and Fraction(f) == v:
        assert B.gamma_str(gm, ge) == "%.6g" % f
