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


def _stiffness(level: int, d: int):
    """The level's stiffness up to a constant (the generalised eigenproblem is scale-free):
    1-D tridiag(-1, 2, -1); 2-D the 9-point (8, -1 x 8) of A1 (x) M1 + M1 (x) A1."""
    import numpy as np
    n = (1 << level) - 1
    t = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    if d == 1:
        return t
    m = 4.0 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)  # 6/h M1
    return np.kron(t, m) + np.kron(m, t)                    # 6 (A1 (x) M1 + M1 (x) A1)


def conv_rate_vcycle(level: int, rho: float, eta: float, w, wdot=None, wcheck=None,
                     ext_prec: int = 400, streams: int = 4, d: int = 1):
    """conv_rate_vcycle (P/src/multigrid.cpp:572-601) in the reference mode (d = 1 or 2):
    one IR-V error-propagation step (b = 0) from every unit vector e_i (from_extfloat at
    wdot) gives the columns (I - B A) e_i; the columns run as independent solves spread
    over `streams` CUDA streams (each a replayed graph), and rho_V = sqrt(lambda_max) of
    the generalised problem (M^T A M, A) with the level's stiffness A (rho_v_of_columns,
    :533-568; here in float64 -- the columns are exact).
    Returns (rho_V, columns as (mantissas, e) per unit vector)."""
    import ctypes as C

    import numpy as np
    import scipy.linalg

    from . import BfpVec, Multigrid, _raise, lib, mg_config_ref, set_stream

    n = ((1 << level) - 1) ** d
    cfg = mg_config_ref(level, rho, eta, w=w, wdot=wdot, wcheck=wcheck, cycles=1, fmg=False,
                        rhs_kind=2, ext_prec=ext_prec, d=d)
    cfg.x0_random = 2  # the caller's iterate
    wd = cfg.pd[level] or cfg.p[level]
    L = lib()
    import torch
    strs = [torch.cuda.Stream() for _ in range(max(1, streams))]
    mgs = [Multigrid(cfg) for _ in strs]
    xs, outs = [], []
    for mg in mgs:
        xh, _, _ = mg.vectors()
        xs.append(BfpVec._view(xh.value, d, level, 8, mg))
        outs.append(mg.rank_result(0)[0])  # the final iterate (x_final)
    cols = [None] * n
    try:
        for base in range(0, n, len(strs)):
            batch = list(range(base, min(n, base + len(strs))))
            for k, i in enumerate(batch):  # enqueue: upload e_i, replay the solve graph
                set_stream(strs[k].cuda_stream)
                unit = np.zeros(n, dtype=np.int64)
                unit[i] = 1 << (wd - 2)  # from_extfloat(e_i, wdot): m = 2^(w-2), e = 2 - w
                _raise(L.bfp_vec_upload(xs[k].h, unit.ctypes.data_as(C.c_void_p), wd, 2 - wd,
                                        C.c_void_p(strs[k].cuda_stream)), "upload e_i")
                mgs[k].solve(use_graph=True)
            for k, i in enumerate(batch):
                set_stream(strs[k].cuda_stream)
                x, q, e = outs[k].download()
                cols[i] = (x.copy(), e)
    finally:
        set_stream(None)
    M = np.stack([np.ldexp(c[0].astype(np.float64), c[1]) for c in cols], axis=1)
    A = _stiffness(level, d)
    lam = scipy.linalg.eigh(M.T @ A @ M, A, eigvals_only=True)
    return float(np.sqrt(max(lam.max(), 0.0))), cols


def recompute_table(level: int, rho: float, eta: float, w, wdot=None, wcheck=None, n_ir: int = 1,
                    caps=(-1, 4, 2, 0), rhs_kind: int = 1, d: int = 1, ext_prec: int = 400):
    """The reference's recompute table (cmd_recompute_table, P/src/experiments.cpp:556-600):
    the FMG solve of the reference-algorithm mode under GammaPolicy::w_add_cap = inf, 4, 2, 0,
    and for each cap the recomputations and calls at the finest level
    (SolverTrace::recomputes_at_level / calls_at_level, P/src/multigrid.cpp:165-177).
    Returns rows (cap, recomputes, calls) -- cap -1 is the table's "inf"."""
    from . import Multigrid, mg_config_ref

    rows = []
    for cap in caps:
        cfg = mg_config_ref(level, rho, eta, w=w, wdot=wdot, wcheck=wcheck, cycles=n_ir, fmg=True,
                            rhs_kind=rhs_kind, ext_prec=ext_prec, w_add_cap=cap, d=d)
        mg = Multigrid(cfg)
        mg.solve(use_graph=True)
        tr = mg.trace()
        rows.append((cap, tr.recomputes_at_level(level), tr.calls_at_level(level)))
    return rows


# ---------------------------------------------------------------------------
# FEM load vector of the reference's manufactured problems (rhs_kind 3)

def fem_load_1d(level: int, k: int, prec: int = 480):
    """integral of sin(k pi x) phi_i(x) over (0, 1), i = 1 .. 2^level - 1, for the p = 1 hat
    basis by the reference's element rule: Gauss-Legendre with degree + 1 = 2 points per
    element, weights on [-1, 1] times the Jacobian h / 2 (assemble_1d_full and ElementRule,
    P/src/fem.cpp:286-296, 316-336).  The reference evaluates in 400-bit MPFR; here mpmath
    at `prec` >= 440 bits, which floor-quantises to the same block unless an entry lies
    within 2^-380 (relative) of a quantisation boundary.  Returns mpmath values."""
    import mpmath as mp
    n = 1 << level
    with mp.workprec(prec):
        h = mp.ldexp(mp.mpf(1), -level)
        g = 1 / mp.sqrt(3)
        nodes = [(1 - g) / 2, (1 + g) / 2]
        kpi = k * mp.pi
        s = [[mp.sin(kpi * ((el + nq) * h)) for nq in nodes] for el in range(n)]
        half = h / 2
        # phi_i = xi on element i - 1, 1 - xi on element i (xi the element-local coordinate)
        load = [half * (s[i - 1][0] * nodes[0] + s[i - 1][1] * nodes[1] +
                        s[i][0] * (1 - nodes[0]) + s[i][1] * (1 - nodes[1]))
                for i in range(1, n)]
        # entries that vanish by symmetry (sin(2 pi x) at x_i = 1/2) are rounding noise, here
        # and in the reference's MPFR evaluation alike; they are taken as exactly 0
        cut = mp.ldexp(h * h, -(prec // 2))  # against the entries' natural size ~ k pi h^2
        return [mp.mpf(0) if abs(v) <= cut else v for v in load]


def _zk62(v) -> Tuple[int, int]:
    """An mpmath value as z 2^k with |z| < 2^62, floored: exact under a later floor
    quantisation at w <= 62 (nested floors with 2^k dividing 2^e_out)."""
    sign, man, exp, bc = v._mpf_
    z = -int(man) if sign else int(man)
    s = max(0, bc - 62)
    return z >> s, exp + s


def fem_rhs(d: int, level: int, prec: int = 480):
    """The D^-1-scaled load vector of level `level` (Hierarchy::setup_scaling,
    P/src/multigrid.cpp:286-289: b / diag(A)) of the reference's Poisson problems as (z, k)
    lists for quantize_exact, x fastest:
      1-D  f = 9 pi^2 sin(3 pi x)  (Manufactured::f, P/src/fem.cpp:99-103), D = 2 / h;
      2-D  f = 13 pi^2 sin(2 pi x1) sin(3 pi x2) as the outer product of two 1-D loads,
           b[i1 n + i2] = 13 pi^2 l2[i1] l3[i2]  (assemble, P/src/fem.cpp:441-456), D = 8/3."""
    import mpmath as mp
    if d not in (1, 2):
        raise ValueError("fem_rhs: d = 1 or 2")
    with mp.workprec(prec):
        pi2 = mp.pi * mp.pi
        l3 = fem_load_1d(level, 3, prec)
        if d == 1:
            c = 9 * pi2 * mp.ldexp(mp.mpf(1), -level) / 2
            vals = [c * v for v in l3]
        else:
            l2 = fem_load_1d(level, 2, prec)
            c = 13 * pi2 * 3 / 8
            vals = [(c * a) * b for a in l2 for b in l3]
        zk = [_zk62(v) for v in vals]
    return [z for z, _ in zk], [k for _, k in zk]


def set_fem_rhs(mg, prec: int = 480):
    """Write the FEM load vectors into a rhs_kind = 3 solver (every level of an FMG
    hierarchy, else the finest), floor-quantised at each level's wcheck on the device
    (bfp_quantize_exact into the handles of bfp_mg_level_rhs)."""
    from . import quantize_exact
    cfg = mg.cfg
    lo = (1 if cfg.ref_mode else cfg.l_coarse) if cfg.fmg else cfg.l_fine
    for l in range(lo, cfg.l_fine + 1):
        z, k = fem_rhs(cfg.d, l, prec)
        w = cfg.pc[l] or cfg.p[l]
        quantize_exact(z, k, w, out=mg.level_rhs(l))


# ---------------------------------------------------------------------------
# rho by power iteration (Hierarchy::setup_scaling)

_RHO_CACHE = {}


def estimate_rho(d: int, l_est: int = 5, prec: int = 400, max_iter: int = 400,
                 rel_tol: float = 1e-12) -> Fraction:
    """rho as the reference's Hierarchy::setup_scaling derives it
    (P/src/multigrid.cpp:277-280): max_gen_eig_upper = 1.01 (rounded up) times the power
    iteration power_max_gen of D^-1 A on level l_est (P/src/linalg.cpp:272-295; the drivers
    pass l_est = min(5, levels)), in correctly rounded prec-bit arithmetic (mpmath: exact
    products added with one rounding = mpfr_fma).  The operator is the p = 1 stiffness up
    to its power-of-two 1/h: 1-D tridiag(-1, 2, -1), 2-D (8/3, -1/3 x 8).  Returns the exact
    value of the prec-bit result; pass it as `rho` to mg_config_ref."""
    key = (d, l_est, prec, max_iter, rel_tol)
    if key in _RHO_CACHE:
        return _RHO_CACHE[key]
    import mpmath as mp
    if d not in (1, 2):
        raise ValueError("estimate_rho: d = 1 or 2")
    n1 = (1 << l_est) - 1
    with mp.workprec(prec):
        if d == 1:
            n = n1
            cen, off = mp.mpf(2), mp.mpf(-1)
            nbr = [[j for j in (i - 1, i, i + 1) if 0 <= j < n] for i in range(n)]
        else:
            n = n1 * n1
            cen, off = mp.mpf(8) / 3, mp.mpf(-1) / 3
            nbr = [[j1 * n1 + j2 for j1 in (i1 - 1, i1, i1 + 1) for j2 in (i2 - 1, i2, i2 + 1)
                    if 0 <= j1 < n1 and 0 <= j2 < n1] for i1 in range(n1) for i2 in range(n1)]
        fma = lambda acc, a, b: mp.fadd(mp.fmul(a, b, exact=True), acc)  # noqa: E731
        x = [mp.mpf(8 + (i % 7)) / 8 for i in range(n)]
        tol = mp.mpf(rel_tol)
        lam = lam_prev = mp.mpf(0)
        for it in range(max_iter):
            ax = []
            for i in range(n):
                y = mp.mpf(0)
                for j in nbr[i]:
                    y = fma(y, cen if j == i else off, x[j])
                ax.append(y)
            num = den = mp.mpf(0)
            for xi, yi in zip(x, ax):
                num = fma(num, xi, yi)
            for xi in x:
                den = fma(den, cen * xi, xi)
            lam = num / den
            if it > 2 and abs(lam - lam_prev) <= tol * abs(lam):
                break
            lam_prev = lam
            x = [yi / cen for yi in ax]
            nrm = max(abs(v) for v in x)
            x = [v / nrm for v in x]
        rho = mp.fmul(lam, mp.mpf(101) / 100, rounding="u")
        sign, man, exp, _ = rho._mpf_
    out = Fraction(int(man)) * Fraction(2) ** int(exp)
    _RHO_CACHE[key] = -out if sign else out
    return _RHO_CACHE[key]
