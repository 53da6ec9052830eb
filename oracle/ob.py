"""ctypes binding of the C oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs; never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

STEP_NAMES = ["ir-residual", "ir-correction", "v-relax0", "v-relax", "v-residual", "v-restrict",
              "v-correct", "fmg-prolong", "final-residual"]


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


class Block(C.Structure):
    _fields_ = [("n", C.c_int64), ("q", C.c_int64), ("e", C.c_int64),
                ("m", C.POINTER(C.c_int64))]


class Flags(C.Structure):
    _fields_ = [("overflow", C.c_int), ("underflow", C.c_int), ("recomputed", C.c_int)]


class Kernel(C.Structure):
    _fields_ = [("q", C.c_int64), ("e", C.c_int64), ("n", C.c_int64), ("row", C.c_void_p),
                ("a", C.c_void_p), ("p", C.c_int64 * 24), ("ptr", C.c_void_p * 8),
                ("zd", C.c_int64)]


class Csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("q", C.c_int64), ("e", C.c_int64),
                ("max_row_nnz", C.c_int64), ("rowptr", C.POINTER(C.c_int64)),
                ("col", C.POINTER(C.c_int64)), ("m", C.POINTER(C.c_int64))]


class Grid(C.Structure):
    _fields_ = [("d", C.c_int), ("l", C.c_int)]


class G15(C.Structure):
    _fields_ = [("m", C.c_int64), ("e", C.c_int64)]


class TraceRec(C.Structure):
    _fields_ = [("step", C.c_int32), ("level", C.c_int32), ("w_out", C.c_int32),
                ("w_tmp", C.c_int32), ("gm", C.c_int64), ("ge", C.c_int64),
                ("overflow", C.c_int32), ("underflow", C.c_int32), ("recomputed", C.c_int32),
                ("normalized", C.c_int32)]


class MgConfig(C.Structure):
    _fields_ = [("d", C.c_int), ("l_fine", C.c_int), ("l_coarse", C.c_int), ("nu1", C.c_int),
                ("nu2", C.c_int), ("n_coarse", C.c_int), ("cycles", C.c_int), ("fmg", C.c_int),
                ("nonnormalized", C.c_int), ("x0_random", C.c_int), ("rhs_kind", C.c_int),
                ("qc", C.c_int), ("seed", C.c_uint64), ("p", C.c_int * 32), ("pd", C.c_int * 32),
                ("pc", C.c_int * 32), ("w_add_cap", C.c_int)]


class MgResult(C.Structure):
    _fields_ = [("x", Block), ("res_history", C.POINTER(C.c_double)), ("n_history", C.c_int),
                ("trace", C.POINTER(TraceRec)), ("trace_cap", C.c_int64),
                ("n_trace", C.c_int64), ("err", C.c_int)]


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        i64, pi64 = C.c_int64, C.POINTER(C.c_int64)
        L.ob_msb64.restype = i64
        L.ob_msb64.argtypes = [i64]
        L.ob_msb128.restype = i64
        L.ob_msb128.argtypes = [i64, C.c_uint64]
        L.ob_shift_floor64.restype = i64
        L.ob_shift_floor64.argtypes = [i64, i64, C.POINTER(C.c_int)]
        L.ob_wrap64.restype = i64
        L.ob_wrap64.argtypes = [i64, i64]
        for f in ("ob_normalize",):
            getattr(L, f).argtypes = [C.POINTER(Block), C.POINTER(Block)]
        L.ob_quantize.argtypes = [C.POINTER(Block), i64, C.POINTER(Block)]
        L.ob_inf_norm_upper.argtypes = [C.POINTER(Block), i64, pi64, pi64, pi64]
        L.ob_qcomp.argtypes = [C.POINTER(Kernel), i64, i64, i64, i64, C.c_int, C.POINTER(Block),
                               C.POINTER(Flags)]
        L.ob_nnqcomp.argtypes = [C.POINTER(Kernel), i64, i64, i64, C.POINTER(Block)]
        L.ob_make_axpby.argtypes = [C.POINTER(Kernel), C.POINTER(Block), C.POINTER(Block)] + [i64] * 6
        L.ob_make_spmv.argtypes = [C.POINTER(Kernel), C.POINTER(Csr), C.POINTER(Block), i64]
        L.ob_make_gemv.argtypes = [C.POINTER(Kernel), C.POINTER(Csr), C.POINTER(Block),
                                   C.POINTER(Block)] + [i64] * 7
        L.ob_make_rows.argtypes = [C.POINTER(Kernel), i64, pi64, C.POINTER(C.c_uint64), i64, i64]
        L.ob_kernel_row.argtypes = [C.POINTER(Kernel), i64, pi64, C.POINTER(C.c_uint64)]
        L.ob_grid_n.restype = i64
        L.ob_grid_n.argtypes = [Grid]
        L.ob_grid_size.restype = i64
        L.ob_grid_size.argtypes = [Grid]
        L.ob_stencil_desc.argtypes = [Grid, pi64, pi64, pi64]
        L.ob_make_stencil_gemv.argtypes = [C.POINTER(Kernel), Grid, C.POINTER(Block),
                                           C.POINTER(Block)] + [i64] * 6
        L.ob_make_jacobi.argtypes = [C.POINTER(Kernel), Grid, C.POINTER(Block), C.POINTER(Block),
                                     i64, i64, i64]
        L.ob_make_scal.argtypes = [C.POINTER(Kernel), C.POINTER(Block), i64, i64, i64]
        L.ob_make_restrict.argtypes = [C.POINTER(Kernel), Grid, C.POINTER(Block)]
        L.ob_make_prolong.argtypes = [C.POINTER(Kernel), Grid, C.POINTER(Block)]
        L.ob_make_prolong_correct.argtypes = [C.POINTER(Kernel), Grid, C.POINTER(Block),
                                              C.POINTER(Block)]
        L.ob_jacobi_coeff.argtypes = [Grid, i64, pi64, pi64]
        L.ob_g15_norm.restype = G15
        L.ob_g15_norm.argtypes = [C.POINTER(Block), i64]
        L.ob_g15_from.restype = G15
        L.ob_g15_from.argtypes = [C.c_uint64, i64]
        L.ob_g15_mul.restype = G15
        L.ob_g15_mul.argtypes = [G15, G15]
        L.ob_g15_add.restype = G15
        L.ob_g15_add.argtypes = [G15, G15]
        L.ob_splitmix64.restype = C.c_uint64
        L.ob_splitmix64.argtypes = [C.c_uint64]
        L.ob_gen_uniform.argtypes = [Grid, i64, C.c_uint64, C.c_uint64, C.POINTER(Block)]
        L.ob_gen_sine.argtypes = [Grid, i64, C.POINTER(Block)]
        L.ob_mg_run.argtypes = [C.POINTER(MgConfig), C.POINTER(MgResult)]
        L.ob_residual_qcomp_omp.argtypes = [Grid, C.POINTER(Block), C.POINTER(Block), i64, i64, i64,
                                            i64, C.POINTER(Block), C.POINTER(Flags), C.c_int]
        _lib = L
    return _lib


# ---------------------------------------------------------------------------
# numpy-level helpers


class OBlock:
    """An oracle block owning an int64 numpy mantissa array."""

    def __init__(self, m, q: int, e: int):
        self.m = np.ascontiguousarray(np.asarray(m, dtype=np.int64))
        self.q, self.e = int(q), int(e)

    @staticmethod
    def empty(n: int) -> "OBlock":
        return OBlock(np.zeros(max(n, 1), dtype=np.int64)[:n] if n else np.zeros(0, np.int64), 1, 0)

    def c(self) -> Block:
        b = Block(len(self.m), self.q, self.e,
                  self.m.ctypes.data_as(C.POINTER(C.c_int64)) if len(self.m) else
                  C.cast(C.pointer(C.c_int64(0)), C.POINTER(C.c_int64)))
        return b

    def update(self, b: Block):
        self.q, self.e = int(b.q), int(b.e)

    def __repr__(self):
        return f"OBlock(q={self.q}, e={self.e}, m={self.m.tolist()[:8]}...)"


class OracleError(RuntimeError):
    pass


def _chk(rc: int, what: str):
    if rc:
        raise OracleError(f"{what}: oracle status {rc}")


def grid(d: int, l: int) -> Grid:
    return Grid(d, l)


def window(kernel_factory, n_out: int, mode: str, w_out: int, w_tmp: int, gm: int, ge: int,
           force: bool = False) -> Tuple[OBlock, Tuple[int, int, int]]:
    """Run qcomp ("q") or nnqcomp ("nn") over a kernel built by kernel_factory(k_ptr)."""
    L = lib()
    k = Kernel()
    keep = kernel_factory(C.byref(k))
    out = OBlock(np.zeros(n_out, dtype=np.int64), w_out, 0)
    ob = out.c()
    fl = Flags()
    if mode == "q":
        _chk(L.ob_qcomp(C.byref(k), w_out, w_tmp, gm, ge, int(force), C.byref(ob), C.byref(fl)),
             "qcomp")
    else:
        _chk(L.ob_nnqcomp(C.byref(k), w_out, gm, ge, C.byref(ob)), "nnqcomp")
    del keep
    out.update(ob)
    return out, (fl.overflow, fl.underflow, fl.recomputed)


def stencil_gemv(d, l, x: OBlock, y: OBlock, alpha, beta, mode, w_out, w_tmp, gm, ge, force=False):
    L = lib()
    xc, yc = x.c(), y.c()

    def mk(kp):
        _chk(L.ob_make_stencil_gemv(kp, Grid(d, l), C.byref(xc), C.byref(yc), *alpha, *beta),
             "stencil")
        return (xc, yc)
    return window(mk, len(y.m), mode, w_out, w_tmp, gm, ge, force)


def jacobi(d, l, x: OBlock, b: OBlock, c, mode, w_out, w_tmp, gm, ge):
    L = lib()
    xc, bc = x.c(), b.c()

    def mk(kp):
        _chk(L.ob_make_jacobi(kp, Grid(d, l), C.byref(xc), C.byref(bc), *c), "jacobi")
        return (xc, bc)
    return window(mk, len(x.m), mode, w_out, w_tmp, gm, ge)


def scal(r: OBlock, c, mode, w_out, w_tmp, gm, ge):
    L = lib()
    rc = r.c()

    def mk(kp):
        _chk(L.ob_make_scal(kp, C.byref(rc), *c), "scal")
        return rc
    return window(mk, len(r.m), mode, w_out, w_tmp, gm, ge)


def restrict(d, lf, r: OBlock, mode, w_out, w_tmp, gm, ge):
    L = lib()
    rc = r.c()
    nc = ((1 << (lf - 1)) - 1) ** d

    def mk(kp):
        _chk(L.ob_make_restrict(kp, Grid(d, lf), C.byref(rc)), "restrict")
        return rc
    return window(mk, nc, mode, w_out, w_tmp, gm, ge)


def prolong(d, lf, xc: OBlock, mode, w_out, w_tmp, gm, ge):
    L = lib()
    cc = xc.c()
    nf = ((1 << lf) - 1) ** d

    def mk(kp):
        _chk(L.ob_make_prolong(kp, Grid(d, lf), C.byref(cc)), "prolong")
        return cc
    return window(mk, nf, mode, w_out, w_tmp, gm, ge)


def prolong_correct(d, lf, ec: OBlock, y: OBlock, mode, w_out, w_tmp, gm, ge):
    L = lib()
    cc, yc = ec.c(), y.c()

    def mk(kp):
        _chk(L.ob_make_prolong_correct(kp, Grid(d, lf), C.byref(cc), C.byref(yc)), "pc")
        return (cc, yc)
    return window(mk, len(y.m), mode, w_out, w_tmp, gm, ge)


def axpby(x: OBlock, y: OBlock, alpha, beta, mode, w_out, w_tmp, gm, ge, force=False):
    L = lib()
    xc, yc = x.c(), y.c()

    def mk(kp):
        _chk(L.ob_make_axpby(kp, C.byref(xc), C.byref(yc), *alpha, *beta), "axpby")
        return (xc, yc)
    return window(mk, len(x.m), mode, w_out, w_tmp, gm, ge, force)


def rows(vals: Sequence[int], q: int, e: int, mode, w_out, w_tmp, gm, ge, force=False):
    L = lib()
    hi = np.array([(v >> 64) for v in vals], dtype=np.int64)
    lo = np.array([(v & ((1 << 64) - 1)) for v in vals], dtype=np.uint64)

    def mk(kp):
        _chk(L.ob_make_rows(kp, len(vals), hi.ctypes.data_as(C.POINTER(C.c_int64)),
                            lo.ctypes.data_as(C.POINTER(C.c_uint64)), q, e), "rows")
        return (hi, lo)
    return window(mk, len(vals), mode, w_out, w_tmp, gm, ge, force)


class OCsr:
    def __init__(self, rows, cols, rowptr, col, m, q, e):
        self.rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int64)
        self.m = np.ascontiguousarray(m, dtype=np.int64)
        self.rows, self.cols, self.q, self.e = rows, cols, q, e
        self.max_row_nnz = int(max((self.rowptr[i + 1] - self.rowptr[i] for i in range(rows)),
                                   default=0))

    def c(self) -> Csr:
        P = C.POINTER(C.c_int64)
        dummy = np.zeros(1, np.int64)
        self._dummy = dummy
        col = self.col if len(self.col) else dummy
        m = self.m if len(self.m) else dummy
        return Csr(self.rows, self.cols, self.q, self.e, self.max_row_nnz,
                   self.rowptr.ctypes.data_as(P), col.ctypes.data_as(P), m.ctypes.data_as(P))


def spmv(a: OCsr, x: OBlock, mode, w_out, w_tmp, gm, ge, m_a=0):
    L = lib()
    ac, xc = a.c(), x.c()

    def mk(kp):
        _chk(L.ob_make_spmv(kp, C.byref(ac), C.byref(xc), m_a), "spmv")
        return (ac, xc)
    return window(mk, a.rows, mode, w_out, w_tmp, gm, ge)


def gemv(a: OCsr, x: OBlock, y: OBlock, alpha, beta, mode, w_out, w_tmp, gm, ge, m_a=0,
         force=False):
    L = lib()
    ac, xc, yc = a.c(), x.c(), y.c()

    def mk(kp):
        _chk(L.ob_make_gemv(kp, C.byref(ac), C.byref(xc), C.byref(yc), *alpha, *beta, m_a), "gemv")
        return (ac, xc, yc)
    return window(mk, a.rows, mode, w_out, w_tmp, gm, ge, force)


def kernel_template(make, *args) -> Tuple[int, int]:
    k = Kernel()
    _chk(make(C.byref(k), *args), "make")
    return int(k.q), int(k.e)


def gen_uniform(d, l, p, seed, stream) -> OBlock:
    n = ((1 << l) - 1) ** d
    b = OBlock(np.zeros(n, np.int64), p, 0)
    bc = b.c()
    _chk(lib().ob_gen_uniform(Grid(d, l), p, seed, stream, C.byref(bc)), "gen_uniform")
    b.update(bc)
    return b


def gen_sine(d, l, p) -> OBlock:
    n = ((1 << l) - 1) ** d
    b = OBlock(np.zeros(n, np.int64), p, 0)
    bc = b.c()
    _chk(lib().ob_gen_sine(Grid(d, l), p, C.byref(bc)), "gen_sine")
    b.update(bc)
    return b


def jacobi_coeff(d, l, qc=16):
    cm, ce = C.c_int64(), C.c_int64()
    lib().ob_jacobi_coeff(Grid(d, l), qc, C.byref(cm), C.byref(ce))
    return cm.value, qc, ce.value


def _lv(v):
    if v is None:
        return [0] * 32
    if isinstance(v, int):
        return [v] * 32
    return list(v) + [0] * (32 - len(v))


def mg_config(d, l_fine, l_coarse=2, nu1=2, nu2=2, n_coarse=16, cycles=1, fmg=False,
              nonnormalized=False, x0_random=False, rhs_kind=1, qc=16, seed=1, p=None, pd=None,
              pc=None, w_add_cap=-1) -> MgConfig:
    cfg = MgConfig()
    cfg.d, cfg.l_fine, cfg.l_coarse, cfg.nu1, cfg.nu2 = d, l_fine, l_coarse, nu1, nu2
    cfg.n_coarse, cfg.cycles, cfg.fmg = n_coarse, cycles, int(fmg)
    cfg.nonnormalized = 2 if nonnormalized == "hybrid" else int(nonnormalized)  # NormMode
    cfg.x0_random, cfg.rhs_kind, cfg.qc, cfg.seed = int(x0_random), rhs_kind, qc, seed
    p, pd, pc = _lv(p), _lv(pd), _lv(pc)
    for i in range(32):
        cfg.p[i], cfg.pd[i], cfg.pc[i] = p[i], pd[i], pc[i]
    cfg.w_add_cap = w_add_cap
    return cfg


def mg_run(cfg: MgConfig, trace_cap: int = 200000):
    L = lib()
    n = ((1 << cfg.l_fine) - 1) ** cfg.d
    x = OBlock(np.zeros(n, np.int64), 1, 0)
    hist = np.zeros(4096, dtype=np.float64)
    trace = (TraceRec * trace_cap)()
    res = MgResult()
    res.x = x.c()
    res.res_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    res.trace = trace
    res.trace_cap = trace_cap
    _chk(L.ob_mg_run(C.byref(cfg), C.byref(res)), "mg_run")
    x.update(res.x)
    tr = [(t.step, t.level, t.w_out, t.w_tmp, t.gm, t.ge, t.overflow, t.underflow, t.recomputed,
           t.normalized) for t in trace[: min(res.n_trace, trace_cap)]]
    return x, hist[: res.n_history].tolist(), tr
