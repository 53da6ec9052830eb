"""Reference-algorithm parity mode: a big-int restatement of the
reference solver P/src/multigrid.cpp:430-518 -- Chebyshev V(1,0) cycles, IR and FMG
with the Table-1 gamma chain (:121-155) -- on the reference's own p = 1 operators
after the D = I scaling (P/src/multigrid.cpp:278-306):

  1-D  A_j = tridiag(-1/2, 1, -1/2)   P_j = [1/2, 1, 1/2] (linear interpolation)
       R_j = D_c^-1 P^T D_f = 2 P^T   (D = 2/h, so D_f / D_c = 2)
  2-D  A_j = A1 (x) M1 + M1 (x) A1 (P/src/fem.cpp:426-457): centre 8/3, eight
       neighbours -1/3 at every level, so D = 8/3 and D^-1 A = (1, -1/8 x 8);
       P_j = P1 (x) P1 (P/src/fem.cpp:542-543), R_j = P^T (D_f = D_c)

Vectors are in lexicographic order, x fastest (kron row index = iy * n + ix).

Operators are quantised with quantize_csr (:216-229) at wcheck / wdot / w, the
Chebyshev coefficients with chebyshev_coeffs_q (:183-193) from rho and eta (rho injected
or power_rho below: max_gen_eig_upper by power iteration), rounded to nearest at the
hierarchy precision (ExtFloat::from_mpq, P/src/extfloat.cpp:21-25) and floor-quantised
at wdot (quantize_scalar_floor, :233-241).  The right-hand side is injected per level
(fem_rhs below: the reference's FEM load vector).

The gamma chain follows gamma_policy_eval (:121-155) with ExtFloat semantics:
mul_up / add_up round up at the operands' maximal precision (P/src/extfloat.cpp:131-140),
exact_norm_ext (:109-117) is exact, scalar_up (:84-105) ceils to q_gamma = 16.

TEST INFRASTRUCTURE ONLY (the checker of the GPU's ref mode), never the product.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, List, Optional, Sequence

from . import pyref as P

Q_GAMMA = 16


# ---------------------------------------------------------------------------
# ExtFloat values: (exact rational, precision in bits)

@dataclass(frozen=True)
class XF:
    v: Fraction
    prec: int


def _round(v: Fraction, prec: int, up: bool) -> Fraction:
    """v >= 0 rounded to prec significant bits: upward (MPFR_RNDU) or to nearest, ties
    to even (MPFR_RNDN)."""
    if v == 0:
        return v
    assert v > 0
    e = v.numerator.bit_length() - v.denominator.bit_length()
    if Fraction(2) ** e > v:
        e -= 1
    s = prec - 1 - e  # v 2^s in [2^(prec-1), 2^prec)
    scaled = v * (Fraction(2) ** s)
    fl = scaled.numerator // scaled.denominator
    rem = scaled - fl
    if up:
        q = fl + (1 if rem > 0 else 0)
    else:
        q = fl + (1 if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl & 1) else 0)
    return Fraction(q) / (Fraction(2) ** s)


def _dyadic(v: Fraction):
    den = v.denominator
    k = -(den.bit_length() - 1)
    assert den == 1 << (-k), "dyadic value"
    return v.numerator, k


def xf_exact_norm(b: P.Block) -> XF:
    """exact_norm_ext (P/src/multigrid.cpp:109-117)."""
    mx = max((abs(v) for v in b.m), default=0)
    prec = max(64, P.msb(mx) + 8)
    return XF(Fraction(mx) * Fraction(2) ** b.e, prec)


def mul_up(a: XF, b: XF) -> XF:
    p = max(a.prec, b.prec)
    return XF(_round(a.v * b.v, p, True), p)


def add_up(a: XF, b: XF) -> XF:
    p = max(a.prec, b.prec)
    return XF(_round(a.v + b.v, p, True), p)


def scalar_up(v: XF, q_gamma: int = Q_GAMMA) -> P.Block:
    """scalar_up (P/src/multigrid.cpp:84-105): ceil to a q_gamma-bit scalar."""
    if v.v <= 0:
        return P.Block.scalar(1 << (q_gamma - 2), q_gamma, -400 - (q_gamma - 2))
    z, k = _dyadic(v.v)
    s = P.msb(z) - q_gamma
    if s <= 0:
        m = z << (-s)
    else:
        m = -((-z) >> s)  # cdiv_q_2exp
        if P.msb(m) > q_gamma:
            m >>= 1
            s += 1
    return P.Block.scalar(m, q_gamma, k + s)


# ---------------------------------------------------------------------------
# operators and scalars

def quantize_values(vals: Sequence[Fraction], w: int):
    """quantize_csr (P/src/multigrid.cpp:216-229) on dyadic values: (mantissas, e)."""
    zk = [(0, 0) if v == 0 else _dyadic(v) for v in vals]
    top = None
    for z, k in zk:
        if z:
            t = P.msb(z) + k
            top = t if top is None else max(top, t)
    if top is None:
        return [0] * len(zk), 0
    e = top - w
    return [P.shift_floor(z, e - k) for z, k in zk], e


def csr_from(rows: int, cols: int, entries: Dict[int, List[tuple]], w: int) -> P.Csr:
    rowptr, col, vals = [0], [], []
    for i in range(rows):
        for c, v in sorted(entries.get(i, [])):
            col.append(c)
            vals.append(v)
        rowptr.append(len(col))
    m, e = quantize_values(vals, w)
    return P.Csr(rows, cols, rowptr, col, m, w, e)


def _entries_a1(j: int):
    n = (1 << j) - 1
    return {i: [(c, Fraction(1) if c == i else Fraction(-1, 2)) for c in (i - 1, i, i + 1)
                if 0 <= c < n] for i in range(n)}


def _entries_p1(j: int):
    """Linear interpolation level j-1 -> j (fine row 2k+1 <- coarse k)."""
    nc = (1 << (j - 1)) - 1
    ent: Dict[int, List[tuple]] = {}
    for k in range(nc):
        for i, wgt in ((2 * k, Fraction(1, 2)), (2 * k + 1, Fraction(1)), (2 * k + 2, Fraction(1, 2))):
            ent.setdefault(i, []).append((k, wgt))
    return ent


def _transpose(ent, scale=Fraction(1)):
    out: Dict[int, List[tuple]] = {}
    for i, row in ent.items():
        for c, v in row:
            out.setdefault(c, []).append((i, v * scale))
    return out


def _kron(ea, eb, nb_rows: int, nb_cols: int):
    """kron(a, b): row ia * nb_rows + ib, column ca * nb_cols + cb (P/src/fem.cpp:364-424)."""
    out: Dict[int, List[tuple]] = {}
    for ia, ra in ea.items():
        for ib, rb in eb.items():
            out[ia * nb_rows + ib] = [(ca * nb_cols + cb, va * vb) for ca, va in ra for cb, vb in rb]
    return out


def _entries_a2(j: int):
    """D^-1 (A1 (x) M1 + M1 (x) A1): centre 1, eight neighbours -1/8."""
    n = (1 << j) - 1
    ent = {}
    for iy in range(n):
        for ix in range(n):
            row = []
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    y, x = iy + dy, ix + dx
                    if 0 <= y < n and 0 <= x < n:
                        row.append((y * n + x, Fraction(1) if dx == dy == 0 else Fraction(-1, 8)))
            ent[iy * n + ix] = row
    return ent


def op_a(j: int, w: int, d: int = 1) -> P.Csr:
    n = ((1 << j) - 1) ** d
    return csr_from(n, n, _entries_a1(j) if d == 1 else _entries_a2(j), w)


def op_p(j: int, w: int, d: int = 1) -> P.Csr:
    nf, nc = (1 << j) - 1, (1 << (j - 1)) - 1
    e1 = _entries_p1(j)
    if d == 1:
        return csr_from(nf, nc, e1, w)
    return csr_from(nf * nf, nc * nc, _kron(e1, e1, nf, nc), w)


def op_r(j: int, w: int, d: int = 1) -> P.Csr:
    """1-D: R = 2 P^T (coarse row k <- fine 2k, 2k+1, 2k+2 with weights 1, 2, 1);
    2-D: R = P^T = (P1 (x) P1)^T."""
    nf, nc = (1 << j) - 1, (1 << (j - 1)) - 1
    if d == 1:
        return csr_from(nc, nf, _transpose(_entries_p1(j), Fraction(2)), w)
    pt = _transpose(_entries_p1(j))
    return csr_from(nc * nc, nf * nf, _kron(pt, pt, nc, nf), w)


NORM_A_UP = Fraction(2)  # ||tridiag(-1/2, 1, -1/2)||_inf = ||(1, -1/8 x 8)||_inf
NORM_R_UP = Fraction(4)  # ||2 P1^T||_inf = ||(P1 (x) P1)^T||_inf


def chebyshev(rho: Fraction, eta: Fraction):
    """chebyshev_coeffs_q (P/src/multigrid.cpp:183-193)."""
    alpha = (1 + eta) * rho / 2
    c = (1 - eta) * rho / 2
    beta = alpha - c * c / (2 * alpha)
    return 2 / beta, Fraction(-1) / (alpha * beta)


def eta_rational(eta: float) -> Fraction:
    """Hierarchy::set_eta (P/src/multigrid.cpp:313-323): two-decimal etas are exact."""
    num = round(eta * 100.0)
    if abs(eta - num / 100.0) < 1e-12:
        return Fraction(num, 100)
    return Fraction(eta)


def quantize_scalar_floor(v: Fraction, w: int) -> P.Block:
    """quantize_scalar_floor (P/src/multigrid.cpp:233-241) of a dyadic value."""
    z, k = _dyadic(v)
    b = P.quantize_exact([z], [k], w)
    return P.Block.scalar(b.m[0], w, b.e)


# ---------------------------------------------------------------------------
# the solver

@dataclass
class RefConfig:
    l_fine: int
    w: List[int]        # per level (index = level), 1..l_fine
    wdot: List[int]
    wcheck: List[int]
    rho: float
    eta: float
    cycles: int = 1     # IR iterations (or n_ir per FMG level)
    fmg: bool = False
    ext_prec: int = 400  # Hierarchy precision (ExtFloat)
    x0: Optional[P.Block] = None
    d: int = 1          # 1 or 2
    w_add_cap: int = -1  # GammaPolicy::w_add_cap (P/src/multigrid.cpp:75-79); < 0: unlimited


@dataclass
class RefResult:
    x: P.Block = None
    history: List[float] = field(default_factory=list)
    trace: List[tuple] = field(default_factory=list)


STEP_IDS = {"ir-residual": 0, "ir-correction": 1, "v-relax": 3, "v-residual": 4,
            "v-restrict": 5, "v-correct": 6, "fmg-prolong": 7}
W_ADD = {"ir-correction": 0, "v-relax": 2, "v-residual": 4, "v-restrict": 6,
         "v-correct": 1, "fmg-prolong": 0}  # GammaPolicy::default_w_add (:62-73)


class RefMg:
    def __init__(self, cfg: RefConfig, rhs: Dict[int, P.Block]):
        self.cfg, self.res = cfg, RefResult()
        self.b = rhs
        self.last_res: Dict[int, XF] = {}
        rho = Fraction(cfg.rho)
        eta = eta_rational(cfg.eta)
        c1, c2 = chebyshev(rho, eta)
        self.c1x = XF(_round(c1, cfg.ext_prec, False), cfg.ext_prec)
        c2x = -_round(-c2, cfg.ext_prec, False)
        self.c1d = {j: quantize_scalar_floor(self.c1x.v, cfg.wdot[j]) for j in range(1, cfg.l_fine + 1)}
        self.c2d = {j: quantize_scalar_floor(c2x, cfg.wdot[j]) for j in range(1, cfg.l_fine + 1)}

    def step(self, name, level, k, w_out, g: XF, ir_iter=1):
        w_add = (5 if ir_iter == 1 else 4) if name == "ir-residual" else W_ADD[name]
        if self.cfg.w_add_cap >= 0:  # GammaPolicy::w_tmp_for
            w_add = min(w_add, self.cfg.w_add_cap)
        gam = scalar_up(g)
        out, fl = P.qcomp(k, w_out, w_out + w_add, gam)
        self.res.trace.append((STEP_IDS[name], level, w_out, w_out + w_add, gam.m[0], gam.e,
                               int(fl.overflow), int(fl.underflow), int(fl.recomputed), 1))
        return out

    def vcycle(self, lev: int, r: P.Block) -> P.Block:
        """P/src/multigrid.cpp:430-456."""
        cfg = self.cfg
        wd = cfg.wdot[lev]
        rn = xf_exact_norm(r)
        ad = op_a(lev, wd, cfg.d)
        y = self.step("v-relax", lev, P.EgemvKernel(ad, r, r, self.c2d[lev], self.c1d[lev]), wd,
                      mul_up(self.c1x, rn))
        if lev > 1:
            two_c1 = XF(self.c1x.v * 2, self.c1x.prec)
            g = mul_up(add_up(two_c1, XF(Fraction(1), self.c1x.prec)), rn)
            g = XF(g.v / 4, g.prec)
            rv = self.step("v-residual", lev, P.EgemvKernel(ad, y, r, P.bfp_one(), P.bfp_minus_one()),
                           wd, g)
            rc = self.step("v-restrict", lev, P.EspmvKernel(op_r(lev, wd, cfg.d), rv), wd,
                           mul_up(XF(NORM_R_UP, cfg.ext_prec), xf_exact_norm(rv)))
            d = self.vcycle(lev - 1, rc)
            y = self.step("v-correct", lev,
                          P.EgemvKernel(op_p(lev, wd, cfg.d), d, y, P.bfp_minus_one(), P.bfp_one()), wd,
                          add_up(xf_exact_norm(y), xf_exact_norm(d)))
        return y

    def ir(self, lev: int, x: P.Block, iters: int) -> P.Block:
        """P/src/multigrid.cpp:458-500 (tol < 0: exactly iters iterations)."""
        cfg = self.cfg
        b = self.b[lev]
        for i in range(1, iters + 1):
            if i > 1:
                g = self.last_res[lev]
            elif lev > 1 and (lev - 1) in self.last_res:
                g = self.last_res[lev - 1]
            else:
                g = add_up(mul_up(XF(NORM_A_UP, cfg.ext_prec), xf_exact_norm(x)), xf_exact_norm(b))
            r = self.step("ir-residual", lev,
                          P.EgemvKernel(op_a(lev, cfg.wcheck[lev], cfg.d), x, b, P.bfp_one(), P.bfp_minus_one()),
                          cfg.wdot[lev], g, ir_iter=i)
            self.last_res[lev] = xf_exact_norm(r)
            mx = max((abs(v) for v in r.m), default=0)
            self.res.history.append(float(Fraction(mx) * Fraction(2) ** r.e))
            y = self.vcycle(lev, r)
            x = self.step("ir-correction", lev, P.EaxpbyKernel(x, y, P.bfp_one(), P.bfp_minus_one()),
                          cfg.w[lev], add_up(xf_exact_norm(x), xf_exact_norm(y)))
        return x

    def fmg(self, lev: int) -> P.Block:
        """P/src/multigrid.cpp:502-518 (each IR iteration a fresh ir(..., 1, -1) call)."""
        cfg = self.cfg
        if lev == 1:
            x = P.zero_vec(1, cfg.w[1])
        else:
            xc = self.fmg(lev - 1)
            x = self.step("fmg-prolong", lev, P.EspmvKernel(op_p(lev, cfg.w[lev], cfg.d), xc), cfg.w[lev],
                          xf_exact_norm(xc))
        for _ in range(cfg.cycles):
            x = self.ir(lev, x, 1)
        return x

    def recomputes_at_level(self, level: int) -> int:
        """SolverTrace::recomputes_at_level (P/src/multigrid.cpp:165-170)."""
        return sum(1 for t in self.res.trace if t[1] == level and (t[6] or t[7]))

    def calls_at_level(self, level: int) -> int:
        """SolverTrace::calls_at_level (:172-177)."""
        return sum(1 for t in self.res.trace if t[1] == level)

    def run(self) -> RefResult:
        cfg = self.cfg
        if cfg.fmg:
            self.res.x = self.fmg(cfg.l_fine)
        else:
            l = cfg.l_fine
            x = cfg.x0 if cfg.x0 is not None else P.zero_vec(((1 << l) - 1) ** cfg.d, cfg.w[l])
            self.res.x = self.ir(l, x, cfg.cycles)
        return self.res


# ---------------------------------------------------------------------------
# FEM load vectors (the right-hand sides of the reference's Poisson problems)

def _fem_load_1d(level: int, k: int, prec: int):
    """assemble_1d_full's load against g(x) = sin(k pi x) for degree 1, m_order 1
    (P/src/fem.cpp:316-336), in the reference's loop order: elements, quadrature points
    (ElementRule(degree + 1): Gauss-Legendre nodes mapped to [0, 1], weights on [-1, 1],
    Jacobian h / 2, :286-296), local basis functions a = 0 (1 - xi) and a = 1 (xi);
    fma_acc into load[span - degree + a] with span = degree + el.  Index 0 and 2^level are
    the boundary functions; the interior is 1 .. 2^level - 1 (interior_offset = 1 for
    Dirichlet p = 1).  MPFR at 400 bits there, mpmath at `prec` here (see fem_rhs)."""
    import mpmath as mp
    n_el = 1 << level
    with mp.workprec(prec):
        h = mp.ldexp(mp.mpf(1), -level)
        jac = h / 2
        gn = [-1 / mp.sqrt(3), 1 / mp.sqrt(3)]      # gauss_legendre(2)
        gw = [mp.mpf(1), mp.mpf(1)]
        nodes01 = [(v + 1) / 2 for v in gn]
        load = [mp.mpf(0)] * (n_el + 1)
        for el in range(n_el):
            for q in range(2):
                xq = (el + nodes01[q]) * h
                xi = nodes01[q]
                ders0 = [1 - xi, xi]                 # hat functions on the element
                fq = mp.sin(k * mp.pi * xq) * (gw[q] * jac)
                for a in range(2):
                    load[el + a] = load[el + a] + fq * ders0[a]
        # An entry that vanishes by symmetry (sin(2 pi x) phi_i at x_i = 1/2: the two
        # elements' contributions cancel) is rounding noise of relative size 2^-prec, in
        # the reference as well (2^-400 there), and floor() of noise is 0 or -1 by the
        # sign of the noise.  The restatement takes the mathematical value 0 -- the one
        # documented deviation.
        cut = mp.ldexp(h * h, -(prec // 2))  # the entries' natural size is ~ k pi h^2
        return [mp.mpf(0) if abs(v) <= cut else v for v in load[1:n_el]]


def fem_rhs(d: int, level: int, w: int, prec: int = 600) -> P.Block:
    """Level `level`'s right-hand side as the reference quantises it: the FEM load vector
    (assemble, P/src/fem.cpp:426-457: 1-D f = Manufactured::f = 9 pi^2 sin(3 pi x), :99-103;
    2-D b[i1 n + i2] = 13 pi^2 load_sin2pi[i1] load_sin3pi[i2]) divided by the level's
    diagonal (Hierarchy::setup_scaling, P/src/multigrid.cpp:286-289; diag = 2 / h in 1-D,
    8 / 3 in 2-D) and floor-quantised at w = wcheck (quantize_vec = from_extfloat,
    P/src/multigrid.cpp:231, P/src/bfp.cpp:189-194).

    The reference rounds every ExtFloat operation to 400 bits; this restatement evaluates
    at `prec` >= 440 bits and floors the result, which gives the same block unless an
    entry lies within ~2^-380 (relative) of a quantisation boundary (the entries are
    transcendental; SURVEY 8(f)-1 asks for exactly this)."""
    import mpmath as mp
    with mp.workprec(prec):
        pi2 = mp.pi * mp.pi
        l3 = _fem_load_1d(level, 3, prec)
        if d == 1:
            diag = 2 / mp.ldexp(mp.mpf(1), -level)
            vals = [(9 * pi2) * v / diag for v in l3]
        else:
            l2 = _fem_load_1d(level, 2, prec)
            c = 13 * pi2
            diag = mp.mpf(8) / 3
            vals = [((c * a) * b) / diag for a in l2 for b in l3]
    z, k = [], []
    for v in vals:
        sign, man, exp, _ = v._mpf_
        z.append(-int(man) if sign else int(man))
        k.append(int(exp))
    return P.quantize_exact(z, k, w)


# ---------------------------------------------------------------------------
# rho by power iteration (Hierarchy::setup_scaling, P/src/multigrid.cpp:277-280)

def _rn(v: Fraction, prec: int) -> Fraction:
    """MPFR_RNDN at prec bits of a signed rational."""
    return -_round(-v, prec, False) if v < 0 else _round(v, prec, False)


def _fem_rows(d: int, level: int, prec: int):
    """a_sym of the p = 1 discretisation by rows (columns ascending, as band_to_csr_interior
    and kron_sum produce them, P/src/fem.cpp:426-431) and its diagonal, up to the common
    power of two 1/h that scales nothing in the iteration: 1-D tridiag(-1, 2, -1);
    2-D A1 (x) M1 + M1 (x) A1 = (8/3, -1/3 x 8), its non-dyadic entries rounded to nearest
    at prec (the reference's come out of the 400-bit quadrature within a few ulps of that)."""
    n = (1 << level) - 1
    rows = []
    if d == 1:
        for i in range(n):
            rows.append([(j, Fraction(2 if j == i else -1)) for j in (i - 1, i, i + 1) if 0 <= j < n])
        return rows, [Fraction(2)] * n
    c, o = _rn(Fraction(8, 3), prec), _rn(Fraction(-1, 3), prec)
    for i1 in range(n):
        for i2 in range(n):
            r = []
            for j1 in (i1 - 1, i1, i1 + 1):
                for j2 in (i2 - 1, i2, i2 + 1):
                    if 0 <= j1 < n and 0 <= j2 < n:
                        r.append((j1 * n + j2, c if (j1, j2) == (i1, i2) else o))
            rows.append(r)
    return rows, [c] * (n * n)


def power_rho(d: int, l_est: int, prec: int = 400, max_iter: int = 400,
              rel_tol: float = 1e-12) -> Fraction:
    """rho = max_gen_eig_upper(a_sym, diag) (P/src/multigrid.cpp:206-209) on level l_est:
    power_max_gen (P/src/linalg.cpp:272-295) -- start vector 1 + (i mod 7)/8, per iteration
    spmv (mpfr_fma accumulation per row, :30-39), the Rayleigh quotient in the D inner
    product (dot = fma chain, :47-51; den += (d_i x_i) x_i), the relative-change stop after
    it > 2, x <- D^-1 A x normalised by its inf-norm -- with every operation rounded to
    nearest at prec like MPFR_RNDN, then mul_up by from_mpq(101/100).  With the default
    400 iterations and 1e-12 the stop never triggers on these operators (the gap ratio at
    level 5 is 0.993): the value is the 400th Rayleigh quotient, ~1e-3 below lambda_max.
    Exact rationals rounded after each operation, so the restatement IS correctly rounded;
    what differs from the reference is only the last ulps of the 2-D matrix entries."""
    rows, diag = _fem_rows(d, l_est, prec)
    n = len(rows)
    x = [Fraction(8 + (i % 7), 8) for i in range(n)]
    tol = Fraction(rel_tol)
    lam = lam_prev = Fraction(0)
    for it in range(max_iter):
        ax = []
        for r in rows:
            y = Fraction(0)
            for j, a in r:
                y = _rn(y + a * x[j], prec)
            ax.append(y)
        num = Fraction(0)
        for xi, yi in zip(x, ax):
            num = _rn(num + xi * yi, prec)
        den = Fraction(0)
        for xi, di in zip(x, diag):
            den = _rn(den + _rn(di * xi, prec) * xi, prec)
        lam = _rn(num / den, prec)
        if it > 2 and abs(_rn(lam - lam_prev, prec)) <= _rn(tol * abs(lam), prec):
            break
        lam_prev = lam
        x = [_rn(yi / di, prec) for yi, di in zip(ax, diag)]
        nrm = max(abs(v) for v in x)
        x = [_rn(v / nrm, prec) for v in x]
    return _round(lam * _rn(Fraction(101, 100), prec), prec, True)
