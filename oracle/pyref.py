"""Python big-int restatement of the reference BFP hot path.

TEST INFRASTRUCTURE ONLY -- the second, independent oracle used to pin the C
restatement (oracle/bfp_oracle.c).  Python ints give exact mpz semantics:
``>>`` floors like ``mpz_fdiv_q_2exp``, ``& mask`` is ``mpz_fdiv_r_2exp`` and
``bit_length`` is ``mpz_sizeinbase(., 2)``.  Pure-Python loops: small cases only.

Reference sections restated (paths relative to /root/reference/proj):
  msb / shift_floor / truncate_to_width / clamp    src/wideint.cpp:15-25,74-79,94-107
  BfpBlock, normalize, quantize, inf_norm_upper     src/bfp.cpp:26-148
  quantize_exact                                    src/bfp.cpp:163-187
  dump_block / parse_block                          src/bfp.cpp:230-272
  EaxpbyKernel / EspmvKernel / EgemvKernel          src/blas.cpp:41-142
  qcomp / nnqcomp                                   src/blas.cpp:144-212
  rational oracle (window_truncate, binade)         tests/oracle.hpp:20-106
The grid operators and the multigrid driver restate DESIGN.md section 3.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Callable, List, Optional, Sequence, Tuple

# --------------------------------------------------------------------------
# wideint.cpp


def msb(v: int) -> int:
    """Minimal w >= 1 with v in T_w (src/wideint.cpp:15-25)."""
    if v == 0:
        return 1
    if v > 0:
        return v.bit_length() + 1
    t = -v - 1
    return 1 if t == 0 else t.bit_length() + 1


def fits_width(v: int, w: int) -> bool:
    if w < 1:
        return False
    hi = 1 << (w - 1)
    return -hi <= v < hi


def shift_floor(x: int, s: int) -> int:
    """floor(x / 2^s); s < 0 shifts left exactly (src/wideint.cpp:94-100)."""
    return x >> s if s >= 0 else x << (-s)


def truncate_to_width(x: int, w: int) -> int:
    """Low w bits as two's complement (src/wideint.cpp:102-107)."""
    r = x & ((1 << w) - 1)
    if (r >> (w - 1)) & 1:
        r -= 1 << w
    return r


def clamp(v: int, lo: int, hi: int) -> int:
    if lo > hi:
        raise ValueError("clamp: lo > hi")
    return lo if v < lo else (hi if v > hi else v)


def dump_wideint(v: int, w: int) -> str:
    """Debug dump "-3 w=3 0x5" (src/wideint.cpp:81-92)."""
    bits = v + (1 << w) if v < 0 else v
    hx = format(bits, "x")
    digits = (w + 3) // 4
    return f"{v} w={w} 0x{hx.rjust(digits, '0')}"


# --------------------------------------------------------------------------
# bfp.cpp


@dataclass
class Block:
    m: List[int]
    q: int
    e: int
    layout: str = "vector"  # scalar | vector | matrix
    rows: int = 0
    cols: int = 1

    def __post_init__(self):
        if self.layout == "vector" and self.rows == 0:
            self.rows = len(self.m)
        for v in self.m:
            if not fits_width(v, self.q):
                raise OverflowError("BfpBlock: mantissa does not fit T_q")  # domain_error

    @staticmethod
    def scalar(m: int, q: int, e: int) -> "Block":
        return Block([m], q, e, "scalar", 1, 1)

    def values(self) -> List[Fraction]:
        return [Fraction(v) * Fraction(2) ** self.e for v in self.m]

    def is_zero(self) -> bool:
        return all(v == 0 for v in self.m)

    def is_normalized(self) -> bool:
        return self.is_zero() or max_msb(self.m) == self.q


def max_msb(m: Sequence[int]) -> int:
    mu = 0
    for v in m:
        if v != 0:
            mu = max(mu, msb(v))
    return mu


def zero_vec(n: int, q: int) -> Block:
    return Block([0] * n, q, 0)


def normalize(x: Block) -> Block:
    """src/bfp.cpp:97-108."""
    if x.is_zero():
        return Block(list(x.m), x.q, 0, x.layout, x.rows, x.cols)
    shift = x.q - max_msb(x.m)
    return Block([shift_floor(v, -shift) for v in x.m], x.q, x.e - shift, x.layout, x.rows, x.cols)


def quantize(x: Block, w: int) -> Block:
    """src/bfp.cpp:110-122."""
    if w < 1:
        raise ValueError("quantize: width must be >= 1")
    if x.is_zero():
        return Block(list(x.m), w, 0, x.layout, x.rows, x.cols)
    s = max_msb(x.m) - w
    return Block([shift_floor(v, s) for v in x.m], w, x.e + s, x.layout, x.rows, x.cols)


def inf_norm_upper(x: Block, q_gamma: int = 16) -> Block:
    """src/bfp.cpp:124-148."""
    if q_gamma < 2:
        raise ValueError("inf_norm_upper: q_gamma must be >= 2")
    mx = max((abs(v) for v in x.m), default=0)
    if mx == 0:
        return Block.scalar(1 << (q_gamma - 2), q_gamma, x.e - (q_gamma - 2))
    s = msb(mx) - q_gamma
    if s <= 0:
        m = mx << (-s)
    else:
        m = -((-mx) >> s)  # mpz_cdiv_q_2exp
        if msb(m) > q_gamma:
            m >>= 1
            s += 1
    return Block.scalar(m, q_gamma, x.e + s)


def quantize_exact(z: Sequence[int], k: Sequence[int], w: int) -> Block:
    """src/bfp.cpp:163-187 (vector layout)."""
    top = None
    for zi, ki in zip(z, k):
        if zi != 0:
            t = msb(zi) + ki
            top = t if top is None else max(top, t)
    if top is None:
        return Block([0] * len(z), w, 0)
    e_out = top - w
    return Block([shift_floor(zi, e_out - ki) for zi, ki in zip(z, k)], w, e_out)


def dump_block(x: Block) -> str:
    """src/bfp.cpp:230-241."""
    if x.layout == "scalar":
        d = "scalar"
    elif x.layout == "vector":
        d = str(x.rows)
    else:
        d = f"{x.rows}x{x.cols}"
    return f"{x.q} {x.e} {d}\n" + "".join(f"{v}\n" for v in x.m)


def parse_block(text: str) -> Block:
    """src/bfp.cpp:243-272."""
    tok = text.split()
    if len(tok) < 3:
        raise ValueError("parse_block: bad header")
    q, e, d = int(tok[0]), int(tok[1]), tok[2]
    m = [int(t) for t in tok[3:]]
    if d == "scalar":
        if len(m) != 1:
            raise ValueError("parse_block: entry count mismatch")
        return Block.scalar(m[0], q, e)
    if "x" in d:
        r, c = (int(t) for t in d.split("x"))
        if len(m) != r * c:
            raise ValueError("parse_block: entry count mismatch")
        return Block(m, q, e, "matrix", r, c)
    if len(m) != int(d):
        raise ValueError("parse_block: entry count mismatch")
    return Block(m, q, e)


# --------------------------------------------------------------------------
# blas.cpp


def ceil_log2(m: int) -> int:
    r, v = 0, 1
    while v < m:
        v <<= 1
        r += 1
    return r


@dataclass
class Tmpl:
    q: int
    e: int


def _axpby_setup(qa: int, ea: int, qb: int, eb: int) -> Tuple[int, Tmpl]:
    d = ea - eb
    q = (max(qa, qb - d) if d < 0 else max(qb, qa + d)) + 1
    return d, Tmpl(q, min(ea, eb))


def _combine(am: int, a: int, bm: int, b: int, d: int) -> int:
    if d < 0:
        return ((bm * b) << (-d)) + am * a
    return ((am * a) << d) + bm * b


class ExactKernel:
    """Plug-in interface (include/bfpmg/blas.hpp:25-31)."""

    tmpl: Tmpl
    n: int

    def row(self, i: int) -> int:  # pragma: no cover - interface
        raise NotImplementedError


class FixedKernel(ExactKernel):
    def __init__(self, rows: Sequence[int], q: int, e: int):
        self.rows, self.tmpl, self.n = list(rows), Tmpl(q, e), len(rows)

    def row(self, i):
        return self.rows[i]


class EaxpbyKernel(ExactKernel):
    """src/blas.cpp:41-72."""

    def __init__(self, x: Block, y: Block, alpha: Block, beta: Block):
        if len(x.m) != len(y.m):
            raise ValueError("axpby: layout mismatch")
        self.x, self.y, self.a, self.b = x, y, alpha, beta
        self.n = len(x.m)
        self.qa, self.qb = alpha.q + x.q, beta.q + y.q
        self.d, self.tmpl = _axpby_setup(self.qa, alpha.e + x.e, self.qb, beta.e + y.e)

    def row(self, i):
        return _combine(self.a.m[0], self.x.m[i], self.b.m[0], self.y.m[i], self.d)


@dataclass
class Csr:
    rows: int
    cols: int
    rowptr: List[int]
    col: List[int]
    m: List[int]
    q: int
    e: int

    @property
    def max_row_nnz(self) -> int:
        return max((self.rowptr[i + 1] - self.rowptr[i] for i in range(self.rows)), default=0)


class EspmvKernel(ExactKernel):
    """src/blas.cpp:74-94."""

    def __init__(self, a: Csr, x: Block, m_a: int = 0):
        if a.cols != len(x.m):
            raise ValueError("spmv: dimension mismatch")
        if m_a == 0:
            m_a = a.max_row_nnz
        if m_a < a.max_row_nnz:
            raise ValueError("spmv: m_a below actual row nonzero count")
        self.a, self.x, self.n = a, x, a.rows
        self.tmpl = Tmpl(a.q + x.q + ceil_log2(max(m_a, 1)), a.e + x.e)

    def row(self, i):
        a = self.a
        return sum(a.m[k] * self.x.m[a.col[k]] for k in range(a.rowptr[i], a.rowptr[i + 1]))


class EgemvKernel(ExactKernel):
    """src/blas.cpp:96-142."""

    def __init__(self, a: Csr, x: Block, y: Block, alpha: Block, beta: Block, m_a: int = 0):
        if a.cols != len(x.m) or a.rows != len(y.m):
            raise ValueError("gemv: dimension mismatch")
        if m_a == 0:
            m_a = a.max_row_nnz
        if m_a < a.max_row_nnz:
            raise ValueError("gemv: m_a below actual row nonzero count")
        self.sp = EspmvKernel(a, x, m_a)
        self.y, self.al, self.be, self.n = y, alpha, beta, a.rows
        g = self.sp.tmpl
        self.d, self.tmpl = _axpby_setup(alpha.q + g.q, alpha.e + g.e, beta.q + y.q, beta.e + y.e)

    def row(self, i):
        return _combine(self.al.m[0], self.sp.row(i), self.be.m[0], self.y.m[i], self.d)


@dataclass
class Flags:
    overflow: bool = False
    underflow: bool = False
    recomputed: bool = False


def _gamma_window_msb(gamma: Block, e_ref: int) -> int:
    if gamma.m[0] <= 0:
        raise ValueError("gamma must be > 0")
    return msb(gamma.m[0]) + gamma.e - e_ref


def qcomp(k: ExactKernel, w_out: int, w_tmp: int, gamma: Block, force_recompute=False):
    """src/blas.cpp:144-187."""
    if w_out < 1 or w_out > w_tmp:
        raise ValueError("qcomp: need 0 < w_out <= w_tmp")
    t = k.tmpl
    mu_tmp = _gamma_window_msb(gamma, t.e)
    lam_tmp = mu_tmp - w_tmp
    tmp, mu_star = [], 1
    for i in range(k.n):
        z = k.row(i)
        if z != 0:
            mu_star = max(mu_star, msb(z))
        tmp.append(truncate_to_width(shift_floor(z, lam_tmp), w_tmp))
    lam_out = mu_star - w_out
    e_out = t.e + lam_out
    fl = Flags(mu_tmp < mu_star, lam_out < lam_tmp)
    if fl.overflow or fl.underflow or force_recompute:
        fl.recomputed = True
        out = [shift_floor(k.row(i), lam_out) for i in range(k.n)]
    else:
        s = lam_out - lam_tmp
        out = [truncate_to_width(shift_floor(v, s), w_out) for v in tmp]
    return Block(out, w_out, e_out), fl


def nnqcomp(k: ExactKernel, w_out: int, gamma: Block):
    """src/blas.cpp:189-212."""
    if w_out < 1:
        raise ValueError("nnqcomp: need 0 < w_out")
    t = k.tmpl
    lam_out = _gamma_window_msb(gamma, t.e) - w_out
    hi, lo = (1 << (w_out - 1)) - 1, -(1 << (w_out - 1))
    out = [clamp(shift_floor(k.row(i), lam_out), lo, hi) for i in range(k.n)]
    return Block(out, w_out, t.e + lam_out), Flags()


def bfp_one() -> Block:
    return Block.scalar(1, 2, 0)


def bfp_minus_one() -> Block:
    return Block.scalar(-1, 1, 0)


# --------------------------------------------------------------------------
# rational oracle (tests/oracle.hpp:20-106)


def binade(v: Fraction) -> int:
    k = v.denominator.bit_length() - 1
    return msb(v.numerator) - k


def floor_div_pow2(v: Fraction, e: int) -> int:
    return math.floor(v / (Fraction(2) ** e))


def window_truncate(rows: Sequence[Fraction], e_zstar: int, w_out: int):
    tops = [binade(v) for v in rows if v != 0]
    top = max(tops) if tops else e_zstar + 1
    e_out = top - w_out
    return [floor_div_pow2(v, e_out) for v in rows], e_out


# --------------------------------------------------------------------------
# grid operators and multigrid driver


def grid_n(l: int) -> int:
    return (1 << l) - 1


def stencil_desc(d: int, l: int) -> Tuple[int, int, int]:
    return msb(2 * d), 2 * l, 2 * d + 1


def _unravel(i: int, n: int, d: int) -> List[int]:
    c = []
    for _ in range(d):
        c.append(i % n)
        i //= n
    return c


def _stencil_row(d: int, n: int, x: Sequence[int], i: int) -> int:
    c = _unravel(i, n, d)
    acc = 2 * d * x[i]
    stride = 1
    for a in range(d):
        if c[a] > 0:
            acc -= x[i - stride]
        if c[a] < n - 1:
            acc -= x[i + stride]
        stride *= n
    return acc


class StencilGemv(ExactKernel):
    """EgemvKernel with A = 2^{2l} S_d as a matrix-free stencil."""

    def __init__(self, d, l, x: Block, y: Block, alpha: Block, beta: Block):
        qa, ea, ma = stencil_desc(d, l)
        self.d, self.nn, self.x, self.y, self.al, self.be = d, grid_n(l), x, y, alpha, beta
        self.n = len(x.m)
        gq, ge = qa + x.q + ceil_log2(ma), ea + x.e
        self.dd, self.tmpl = _axpby_setup(alpha.q + gq, alpha.e + ge, beta.q + y.q, beta.e + y.e)

    def row(self, i):
        g = _stencil_row(self.d, self.nn, self.x.m, i)
        return _combine(self.al.m[0], g, self.be.m[0], self.y.m[i], self.dd)


class Jacobi(ExactKernel):
    """z = x + c (b - A x): egemv(A,x,b,-1,1) composed with eaxpby(x,r,1,c)."""

    def __init__(self, d, l, x: Block, b: Block, c: Block):
        qa, ea, ma = stencil_desc(d, l)
        self.d, self.nn, self.x, self.b, self.c = d, grid_n(l), x, b, c
        self.n = len(x.m)
        gq, ge = qa + x.q + ceil_log2(ma), ea + x.e
        self.d1, tr = _axpby_setup(1 + gq, ge, 2 + b.q, b.e)
        self.d2, self.tmpl = _axpby_setup(2 + x.q, x.e, c.q + tr.q, c.e + tr.e)

    def row(self, i):
        g = _stencil_row(self.d, self.nn, self.x.m, i)
        r = _combine(-1, g, 1, self.b.m[i], self.d1)
        return _combine(1, self.x.m[i], self.c.m[0], r, self.d2)


class Scal(ExactKernel):
    def __init__(self, r: Block, c: Block):
        self.r, self.c, self.n = r, c, len(r.m)
        self.tmpl = Tmpl(c.q + r.q, c.e + r.e)

    def row(self, i):
        return self.c.m[0] * self.r.m[i]


class Restrict(ExactKernel):
    """Full weighting espmv: R = (1,2,1)^{(x)d} 2^{-2d}."""

    def __init__(self, d, lf, r: Block):
        self.d, self.nf, self.nc, self.r = d, grid_n(lf), grid_n(lf - 1), r
        self.n = self.nc ** d
        self.tmpl = Tmpl(d + 2 + r.q + ceil_log2(3 ** d), -2 * d + r.e)

    def row(self, ic):
        c = _unravel(ic, self.nc, self.d)
        acc = 0
        offs = [(dx, dy, dz) for dz in ((-1, 0, 1) if self.d >= 3 else (0,))
                for dy in ((-1, 0, 1) if self.d >= 2 else (0,)) for dx in (-1, 0, 1)]
        for o in offs:
            w, fi, stride = 1, 0, 1
            for a in range(self.d):
                w *= 2 - abs(o[a])
                fi += (2 * c[a] + 1 + o[a]) * stride
                stride *= self.nf
            acc += w * self.r.m[fi]
        return acc


def _prolong_row(d, nf, nc, xc, i):
    f = _unravel(i, nf, d)
    axes = []
    for a in range(d):
        if f[a] & 1:
            axes.append([((f[a] - 1) // 2, 2)])
        else:
            opts = []
            if f[a] // 2 - 1 >= 0:
                opts.append((f[a] // 2 - 1, 1))
            if f[a] // 2 < nc:
                opts.append((f[a] // 2, 1))
            axes.append(opts)
    acc = 0

    def rec(a, idx, w, stride):
        nonlocal acc
        if a == d:
            acc += w * xc[idx]
            return
        for ci, cw in axes[a]:
            rec(a + 1, idx + ci * stride, w * cw, stride * nc)

    rec(0, 0, 1, 1)
    return acc


class Prolong(ExactKernel):
    def __init__(self, d, lf, xc: Block):
        self.d, self.nf, self.nc, self.xc = d, grid_n(lf), grid_n(lf - 1), xc
        self.n = self.nf ** d
        self.tmpl = Tmpl(d + 2 + xc.q + d, -d + xc.e)

    def row(self, i):
        return _prolong_row(self.d, self.nf, self.nc, self.xc.m, i)


class ProlongCorrect(ExactKernel):
    def __init__(self, d, lf, ec: Block, y: Block):
        self.d, self.nf, self.nc, self.ec, self.y = d, grid_n(lf), grid_n(lf - 1), ec, y
        self.n = self.nf ** d
        gq, ge = d + 2 + ec.q + d, -d + ec.e
        self.dd, self.tmpl = _axpby_setup(2 + gq, ge, 2 + y.q, y.e)

    def row(self, i):
        g = _prolong_row(self.d, self.nf, self.nc, self.ec.m, i)
        return _combine(1, g, 1, self.y.m[i], self.dd)


def jacobi_coeff(d: int, l: int, qc: int) -> Block:
    v = Fraction(1, {1: 3, 2: 5, 3: 7}[d])
    top = math.floor(math.log2(v)) + 2
    m = math.floor(v * Fraction(2) ** (qc - top))
    return Block.scalar(m, qc, top - qc - 2 * l)


# gamma arithmetic: 15-bit round-up values


def g15_from(mag: int, e: int) -> Tuple[int, int]:
    if mag == 0:
        return (0, 0)
    b = mag.bit_length()
    if b <= 15:
        return (mag << (15 - b), e - (15 - b))
    s = b - 15
    m = -((-mag) >> s)
    if m == 1 << 15:
        m >>= 1
        s += 1
    return (m, e + s)


def g15_exact(v: Fraction) -> Tuple[int, int]:
    """Round a nonnegative dyadic rational up to 15 significant bits."""
    if v == 0:
        return (0, 0)
    k = v.denominator.bit_length() - 1
    return g15_from(v.numerator, -k)


def g15_val(g) -> Fraction:
    return Fraction(g[0]) * Fraction(2) ** g[1]


def g15_mul(a, b):
    if a[0] == 0 or b[0] == 0:
        return (0, 0)
    return g15_from(a[0] * b[0], a[1] + b[1])


def g15_add(a, b):
    if a[0] == 0:
        return b
    if b[0] == 0:
        return a
    return g15_exact(g15_val(a) + g15_val(b))


def g15_norm(x: Block):
    return g15_from(max((abs(v) for v in x.m), default=0), x.e)


def g15_gamma(g) -> Block:
    if g[0] == 0:
        return Block.scalar(1 << 14, 16, -400 - 14)
    return Block.scalar(g[0], 16, g[1])


# generators

M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def gen_uniform(d: int, l: int, p: int, seed: int, stream: int) -> Block:
    key = splitmix64(splitmix64(seed) ^ stream)
    n = grid_n(l) ** d
    m = [(splitmix64((key + i) & M64) >> (64 - p)) - (1 << (p - 1)) for i in range(n)]
    return normalize(Block(m, p, -(p - 1)))


def gen_sine(d: int, l: int, p: int) -> Block:
    n = grid_n(l)
    h = math.ldexp(1.0, -l)
    s = [math.sin(math.pi * ((i + 1) * h)) for i in range(n)]
    C = float(d) * (math.pi * math.pi)
    z, k = [], []
    for i in range(n ** d):
        c = _unravel(i, n, d)
        v = C * s[c[0]]
        for a in range(1, d):
            v = v * s[c[a]]
        fr, ex = math.frexp(v)
        z.append(int(math.ldexp(fr, 53)))
        k.append(ex - 53)
    return quantize_exact(z, k, p)


STEPS = ["ir-residual", "ir-correction", "v-relax0", "v-relax", "v-residual", "v-restrict",
         "v-correct", "fmg-prolong", "final-residual"]


@dataclass
class MgConfig:
    d: int
    l_fine: int
    l_coarse: int = 2
    nu1: int = 2
    nu2: int = 2
    n_coarse: int = 16
    cycles: int = 1
    fmg: bool = False
    nonnormalized: bool = False
    x0_random: bool = False
    rhs_kind: int = 1
    qc: int = 16
    seed: int = 1
    p: Optional[List[int]] = None   # w: iterate width, indexed by level
    pd: Optional[List[int]] = None  # wdot: residual / V-cycle width (0 / None = p)
    pc: Optional[List[int]] = None  # wcheck: right-hand-side width (0 / None = p)
    w_add_cap: int = -1             # GammaPolicy::w_add_cap (-1 = unlimited)


@dataclass
class MgResult:
    x: Block = None
    history: List[float] = field(default_factory=list)
    trace: List[tuple] = field(default_factory=list)


class Mg:
    """DESIGN.md section 3 driver: IR with correction-scheme Jacobi V-cycles, FMG."""

    def __init__(self, cfg: MgConfig):
        self.cfg, self.res = cfg, MgResult()
        self.prev = {}

    def w(self, l):
        return self.cfg.p[l]

    def wd(self, l):
        pd = self.cfg.pd
        return pd[l] if pd and pd[l] else self.cfg.p[l]

    def wc(self, l):
        pc = self.cfg.pc
        return pc[l] if pc and pc[l] else self.cfg.p[l]

    def step(self, name, level, k, w_out, g, w_add):
        # NormMode (src/multigrid.cpp:403-409): 0 / False normalized, 1 / True
        # nonnormalized, 2 hybrid (qcomp only for IR residuals of iterations <= 2)
        nm = int(self.cfg.nonnormalized)
        normalized = (nm == 0 or name == "final-residual" or
                      (nm == 2 and name == "ir-residual" and self.ir_iter <= 2))
        if self.cfg.w_add_cap >= 0:
            w_add = min(w_add, self.cfg.w_add_cap)
        gam = g15_gamma(g)
        if normalized:
            out, fl = qcomp(k, w_out, w_out + w_add, gam)
        else:
            out, fl = nnqcomp(k, w_out, gam)
        self.res.trace.append((STEPS.index(name), level, w_out,
                               w_out + w_add if normalized else w_out, gam.m[0], gam.e,
                               int(fl.overflow), int(fl.underflow), int(fl.recomputed),
                               int(normalized)))
        return out

    def vcycle(self, l, r):
        cfg = self.cfg
        d = cfg.d
        c = jacobi_coeff(d, l, cfg.qc)
        c15 = g15_from(c.m[0], c.e)
        e = self.step("v-relax0", l, Scal(r, c), self.wd(l), g15_mul(c15, g15_norm(r)), 2)
        sweeps = cfg.n_coarse if l == cfg.l_coarse else cfg.nu1
        for _ in range(1, sweeps):
            e = self.step("v-relax", l, Jacobi(d, l, e, r, c), self.wd(l),
                          g15_add(g15_norm(e), g15_mul(c15, g15_norm(r))), 3)
        if l == cfg.l_coarse:
            return e
        rv = self.step("v-residual", l, StencilGemv(d, l, e, r, bfp_minus_one(), bfp_one()),
                       self.wd(l), g15_norm(r), 4)
        rc = self.step("v-restrict", l, Restrict(d, l, rv), self.wd(l), g15_norm(rv), 6)
        ec = self.vcycle(l - 1, rc)
        e = self.step("v-correct", l, ProlongCorrect(d, l, ec, e), self.wd(l),
                      g15_add(g15_norm(e), g15_norm(ec)), 2)
        for _ in range(cfg.nu2):
            e = self.step("v-relax", l, Jacobi(d, l, e, r, c), self.wd(l),
                          g15_add(g15_norm(e), g15_mul(c15, g15_norm(r))), 3)
        return e

    def ir(self, l, x, b, iters):
        d = self.cfg.d
        self.prev.pop(l, None)
        for it in range(iters):
            self.ir_iter = it + 1
            first = l not in self.prev
            if first:  # ||b|| + ||A|| ulp(x)
                ulp = g15_from(1, x.e) if not x.is_zero() else (0, 0)
                g = g15_add(g15_norm(b), g15_mul(g15_from(4 * d, 2 * l), ulp))
            else:
                g = self.prev[l]
            r = self.step("ir-residual", l, StencilGemv(d, l, x, b, bfp_minus_one(), bfp_one()),
                          self.wd(l), g, 5 if first else 4)
            self.prev[l] = g15_norm(r)
            self.res.history.append(_norm_double(r))
            e = self.vcycle(l, r)
            x = self.step("ir-correction", l, EaxpbyKernel(x, e, bfp_one(), bfp_one()), self.w(l),
                          g15_add(g15_norm(x), g15_norm(e)), 1)
        return x

    def rhs(self, l):
        cfg = self.cfg
        if cfg.rhs_kind == 1:
            return gen_sine(cfg.d, l, self.wc(l))
        if cfg.rhs_kind == 0:
            return gen_uniform(cfg.d, l, self.wc(l), cfg.seed, 2)
        return zero_vec(grid_n(l) ** cfg.d, self.wc(l))

    def final(self, l, x, b):
        r = self.step("final-residual", l,
                      StencilGemv(self.cfg.d, l, x, b, bfp_minus_one(), bfp_one()), self.wd(l),
                      self.prev[l], 4)
        self.res.history.append(_norm_double(r))

    def fmg(self, l):
        cfg = self.cfg
        b = self.rhs(l)
        if l == cfg.l_coarse:
            x = zero_vec(grid_n(l) ** cfg.d, self.w(l))
        else:
            xc = self.fmg(l - 1)
            x = self.step("fmg-prolong", l, Prolong(cfg.d, l, xc), self.w(l), g15_norm(xc), 1)
        x = self.ir(l, x, b, cfg.cycles)
        if l == cfg.l_fine:
            self.final(l, x, b)
        return x

    def run(self) -> MgResult:
        cfg = self.cfg
        if cfg.fmg:
            self.res.x = self.fmg(cfg.l_fine)
        else:
            l = cfg.l_fine
            b = self.rhs(l)
            if cfg.x0_random:
                x = gen_uniform(cfg.d, l, cfg.p[l], cfg.seed, 1)
            else:
                x = zero_vec(grid_n(l) ** cfg.d, cfg.p[l])
            x = self.ir(l, x, b, cfg.cycles)
            self.final(l, x, b)
            self.res.x = x
        return self.res


def _norm_double(b: Block) -> float:
    mx = max((abs(v) for v in b.m), default=0)
    return math.ldexp(float(mx), b.e)
