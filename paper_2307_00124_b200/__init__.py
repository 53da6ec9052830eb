"""B200-native BFP multigrid hot path (arXiv 2307.00124) -- Python host mirror.

A thin ctypes layer over the C-ABI of ``_lib/libbfpmg_b200.so``
(``include/bfpmg_b200.h``).  Names, argument meaning and error behaviour
mirror the reference C++ API (paths relative to /root/reference/proj):

  BfpBlock, zero_vec, normalize, quantize     include/bfpmg/bfp.hpp:18-56, src/bfp.cpp:26-122
  inf_norm_upper, dump_block/parse_block      src/bfp.cpp:124-148, 230-272
  qaxpby/qsub/qspmv/qgemv (+ nnq*)            src/blas.cpp:214-258
  qcomp/nnqcomp over fixed rows               src/blas.cpp:144-212
  bfp_one / bfp_minus_one                     src/blas.cpp:257-258

Every compute call runs on the GPU; there is no CPU fallback.  If the shared
library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BFPMG_LIB") or os.path.join(HERE, "_lib", "libbfpmg_b200.so")  # A/B builds
REPO = os.path.dirname(HERE)

# status codes (include/bfpmg_b200.h)
OK, ERR_ARG, ERR_WIDTH, ERR_DOMAIN, ERR_CUDA, ERR_ALIAS, ERR_NOMEM, ERR_STORAGE = range(8)
FLAG_OVERFLOW, FLAG_UNDERFLOW, FLAG_RECOMPUTED, FLAG_NORMALIZED = 1, 2, 4, 8
STEP_NAMES = ["ir-residual", "ir-correction", "v-relax0", "v-relax", "v-residual", "v-restrict",
              "v-correct", "fmg-prolong", "final-residual"]


class BfpError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} ({status})")


class InvalidArgument(BfpError, ValueError):  # std::invalid_argument
    pass


class DomainError(BfpError, ValueError):  # std::domain_error
    pass


class WidthError(BfpError, OverflowError):  # exact row beyond 127 bits
    pass


def _raise(status: int, what: str):
    if status == OK:
        return
    cls = {ERR_ARG: InvalidArgument, ERR_ALIAS: InvalidArgument, ERR_DOMAIN: DomainError,
           ERR_STORAGE: DomainError, ERR_WIDTH: WidthError}.get(status, BfpError)
    raise cls(status, what)


class _Header(C.Structure):
    _fields_ = [("q", C.c_int64), ("e", C.c_int64), ("n", C.c_int64), ("max_abs", C.c_int64),
                ("flags", C.c_int32), ("err", C.c_int32)]


class _Scalar(C.Structure):
    _fields_ = [("m", C.c_int64), ("q", C.c_int64), ("e", C.c_int64)]


class XfC(C.Structure):  # bfp_xf_t
    _fields_ = [("hi", C.c_uint64), ("lo", C.c_uint64), ("e", C.c_int64), ("sticky", C.c_int32),
                ("pad", C.c_int32)]


class MgConfig(C.Structure):
    _fields_ = [("d", C.c_int), ("l_fine", C.c_int), ("l_coarse", C.c_int), ("nu1", C.c_int),
                ("nu2", C.c_int), ("n_coarse", C.c_int), ("cycles", C.c_int), ("fmg", C.c_int),
                ("nonnormalized", C.c_int), ("x0_random", C.c_int), ("rhs_kind", C.c_int),
                ("qc", C.c_int), ("seed", C.c_uint64), ("p", C.c_int * 32), ("pd", C.c_int * 32),
                ("pc", C.c_int * 32), ("w_add_cap", C.c_int), ("fuse_points", C.c_int),
                ("ref_mode", C.c_int), ("ref_c1", XfC), ("ref_kres", XfC),
                ("ref_c1d", _Scalar * 32), ("ref_c2d", _Scalar * 32)]


class TraceRec(C.Structure):
    _fields_ = [("step", C.c_int32), ("level", C.c_int32), ("w_out", C.c_int32),
                ("w_tmp", C.c_int32), ("gm", C.c_int64), ("ge", C.c_int64),
                ("overflow", C.c_int32), ("underflow", C.c_int32), ("recomputed", C.c_int32),
                ("normalized", C.c_int32)]


EXPORTS = [
    "bfp_vec_create", "bfp_vec_create_grid", "bfp_vec_destroy", "bfp_vec_size", "bfp_vec_upload",
    "bfp_vec_upload_i32", "bfp_vec_download", "bfp_vec_download_i32", "bfp_vec_header",
    "bfp_vec_zero", "bfp_vec_dump", "bfp_vec_parse", "bfp_normalize", "bfp_quantize",
    "bfp_inf_norm_upper", "bfp_dot_exact", "bfp_axpby", "bfp_csr_create", "bfp_csr_destroy",
    "bfp_spmv_csr", "bfp_gemv_csr", "bfp_qcomp_rows", "bfp_stencil_gemv", "bfp_stencil_jacobi",
    "bfp_scal", "bfp_restrict_fw", "bfp_prolong", "bfp_prolong_correct", "bfp_jacobi_coeff",
    "bfp_gen_uniform", "bfp_gen_sine", "bfp_mg_create", "bfp_mg_destroy", "bfp_mg_solve",
    "bfp_mg_result", "bfp_mg_vectors", "bfp_mg_level_rhs", "bfp_mg_kernel_launches", "bfp_status_string",
    "bfp_device_sync", "bfp_launch_count", "bfp_profile_enable", "bfp_profile_read",
    "bfp_set_kernel_path", "bfp_vec_download_async_i32", "bfp_vec_create_slab", "bfp_vec_planes",
    "bfp_stencil_gemv_part", "bfp_stencil_jacobi_part", "bfp_window_finalize",
    "bfp_nccl_unique_id", "bfp_mg_create_sharded", "bfp_mg_rank_result", "bfp_dist_create",
    "bfp_set_transport", "bfp_mg_transport",
    "bfp_dist_destroy", "bfp_dist_stencil_gemv", "bfp_dist_stencil_jacobi",
    "bfp_quantize_exact", "bfp_from_doubles", "bfp_kernel_family_counts",
    "bfp_dot_exact_async", "bfp_dot_value", "bfp_dot_exact192", "bfp_dist_dot_exact",
]

_lib: Optional[C.CDLL] = None


def build(verbose: bool = False) -> str:
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
    return LIB_PATH


def lib() -> C.CDLL:
    """Load the sm_100a library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"bfpmg_b200: CUDA library {LIB_PATH} not built (run build())")
    L = C.CDLL(LIB_PATH)
    i64, i32, vp, pi64 = C.c_int64, C.c_int, C.c_void_p, C.POINTER(C.c_int64)
    S = _Scalar
    sig = {
        "bfp_vec_create": (i32, [i64, i32, C.POINTER(vp)]),
        "bfp_vec_create_grid": (i32, [i32, i32, i32, C.POINTER(vp)]),
        "bfp_vec_destroy": (i32, [vp]),
        "bfp_vec_size": (i64, [vp]),
        "bfp_vec_upload": (i32, [vp, vp, i64, i64, vp]),
        "bfp_vec_upload_i32": (i32, [vp, vp, i64, i64, vp]),
        "bfp_vec_download": (i32, [vp, vp, C.POINTER(_Header), vp]),
        "bfp_vec_download_i32": (i32, [vp, vp, C.POINTER(_Header), vp]),
        "bfp_vec_header": (i32, [vp, C.POINTER(_Header), vp]),
        "bfp_vec_zero": (i32, [vp, i64, vp]),
        "bfp_vec_dump": (i64, [vp, C.c_char_p, i64, vp]),
        "bfp_vec_parse": (i32, [C.c_char_p, C.POINTER(vp), vp]),
        "bfp_normalize": (i32, [vp, vp, vp]),
        "bfp_quantize": (i32, [vp, i64, vp, vp]),
        "bfp_inf_norm_upper": (i32, [vp, i64, pi64, pi64, pi64, vp]),
        "bfp_dot_exact": (i32, [vp, vp, pi64, C.POINTER(C.c_uint64), pi64, vp]),
        "bfp_dot_exact_async": (i32, [vp, vp, vp, vp]),
        "bfp_dot_value": (i32, [vp, vp, pi64, C.POINTER(C.c_uint64)]),
        "bfp_dot_exact192": (i32, [vp, vp, vp, pi64, vp]),
        "bfp_dist_dot_exact": (i32, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), vp]),
        "bfp_axpby": (i32, [vp, vp, S, S, i32, i64, i64, S, i32, vp, vp]),
        "bfp_csr_create": (i32, [i64, i64, vp, vp, vp, i64, i64, C.POINTER(vp)]),
        "bfp_csr_destroy": (i32, [vp]),
        "bfp_spmv_csr": (i32, [vp, vp, i64, i32, i64, i64, S, i32, vp, vp]),
        "bfp_gemv_csr": (i32, [vp, vp, vp, S, S, i64, i32, i64, i64, S, i32, vp, vp]),
        "bfp_qcomp_rows": (i32, [i64, vp, vp, i64, i64, i32, i64, i64, S, i32, vp, vp]),
        "bfp_stencil_gemv": (i32, [vp, vp, S, S, i32, i64, i64, S, i32, vp, vp]),
        "bfp_stencil_jacobi": (i32, [vp, vp, S, i32, i64, i64, S, vp, vp]),
        "bfp_scal": (i32, [vp, S, i32, i64, i64, S, vp, vp]),
        "bfp_restrict_fw": (i32, [vp, i32, i64, i64, S, vp, vp]),
        "bfp_prolong": (i32, [vp, i32, i64, i64, S, vp, vp]),
        "bfp_prolong_correct": (i32, [vp, vp, i32, i64, i64, S, vp, vp]),
        "bfp_jacobi_coeff": (i32, [i32, i32, i64, C.POINTER(S)]),
        "bfp_gen_uniform": (i32, [vp, i64, C.c_uint64, C.c_uint64, vp]),
        "bfp_gen_sine": (i32, [vp, i64, vp]),
        "bfp_mg_create": (i32, [C.POINTER(MgConfig), C.POINTER(vp)]),
        "bfp_mg_destroy": (i32, [vp]),
        "bfp_mg_solve": (i32, [vp, i32, vp]),
        "bfp_mg_result": (i32, [vp, vp, C.POINTER(_Header), vp, i32, C.POINTER(i32), vp, i64,
                                pi64, vp]),
        "bfp_mg_vectors": (i32, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
        "bfp_mg_level_rhs": (i32, [vp, i32, C.POINTER(vp), C.POINTER(i32)]),
        "bfp_nccl_unique_id": (i32, [vp, i32]),
        "bfp_quantize_exact": (i32, [vp, vp, i64, i64, vp, vp]),
        "bfp_from_doubles": (i32, [vp, i64, i64, vp, vp]),
        "bfp_dist_create": (i32, [i32, i32, vp, C.POINTER(vp)]),
        "bfp_dist_destroy": (i32, [vp]),
        "bfp_dist_stencil_gemv": (i32, [vp, C.POINTER(vp), C.POINTER(vp), S, S, i32, i64, i64, S,
                                        C.POINTER(vp), vp]),
        "bfp_dist_stencil_jacobi": (i32, [vp, C.POINTER(vp), C.POINTER(vp), S, i32, i64, i64, S,
                                          C.POINTER(vp), vp]),
        "bfp_mg_create_sharded": (i32, [C.POINTER(MgConfig), i32, i32, vp, i32, C.POINTER(vp)]),
        "bfp_set_transport": (i32, [i32]),
        "bfp_mg_transport": (i32, [vp]),
        "bfp_mg_rank_result": (i32, [vp, i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(i32),
                                     C.POINTER(i32)]),
        "bfp_mg_kernel_launches": (i64, [vp]),
        "bfp_status_string": (C.c_char_p, [i32]),
        "bfp_device_sync": (i32, [vp]),
        "bfp_launch_count": (i64, []),
        "bfp_kernel_family_counts": (i32, [pi64, i32]),
        "bfp_profile_enable": (i32, [i32]),
        "bfp_profile_read": (i32, [C.POINTER(C.c_double), pi64, i32]),
        "bfp_set_kernel_path": (i32, [i32]),
        "bfp_vec_download_async_i32": (i32, [vp, vp, vp]),
        "bfp_vec_create_slab": (i32, [i32, i32, i32, i32, i32, C.POINTER(vp)]),
        "bfp_vec_planes": (i32, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                 pi64]),
        "bfp_stencil_gemv_part": (i32, [vp, vp, S, S, i32, i32, i64, i64, S, vp, vp, vp]),
        "bfp_stencil_jacobi_part": (i32, [vp, vp, S, i32, i32, i64, i64, S, vp, vp, vp]),
        "bfp_window_finalize": (i32, [vp, i32, i32, i64, i64, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def status_string(st: int) -> str:
    try:
        return lib().bfp_status_string(st).decode()
    except Exception:  # library not loadable
        return str(st)


_stream: Optional[int] = None


def set_stream(handle: Optional[int]):
    """Use a caller stream (e.g. torch.cuda.current_stream().cuda_stream) for every call."""
    global _stream
    _stream = handle


def _s():
    return C.c_void_p(_stream) if _stream else None


# ---------------------------------------------------------------------------
# BFP scalars


@dataclass(frozen=True)
class Scalar:
    """BfpScalar (m, q, e): value m * 2^e, m in T_q."""
    m: int
    q: int
    e: int

    def c(self) -> _Scalar:
        return _Scalar(self.m, self.q, self.e)


def bfp_one() -> Scalar:
    return Scalar(1, 2, 0)


def bfp_minus_one() -> Scalar:
    return Scalar(-1, 1, 0)


# ---------------------------------------------------------------------------
# device blocks


class BfpVec:
    """A device BFP block: int32/int64 mantissas + one shared exponent.

    ``BfpVec.grid(d, l)`` creates a grid vector with (2^l - 1)^d interior points
    (x fastest); ``BfpVec.flat(n)`` a plain vector.  Mantissas live in HBM, the
    header (q, e, max|m|, flags) on the device too.
    """

    def __init__(self, handle: int, dim: int, level: int, mant_bytes: int):
        self.h = C.c_void_p(handle)
        self.dim, self.level, self.mant_bytes = dim, level, mant_bytes

    @staticmethod
    def flat(n: int, mant_bytes: int = 8) -> "BfpVec":
        h = C.c_void_p()
        _raise(lib().bfp_vec_create(n, mant_bytes, C.byref(h)), "bfp_vec_create")
        return BfpVec(h.value, 0, 0, mant_bytes)

    @staticmethod
    def grid(dim: int, level: int, mant_bytes: int = 4) -> "BfpVec":
        h = C.c_void_p()
        _raise(lib().bfp_vec_create_grid(dim, level, mant_bytes, C.byref(h)), "bfp_vec_create_grid")
        return BfpVec(h.value, dim, level, mant_bytes)

    @staticmethod
    def slab(dim: int, level: int, z_lo: int, z_hi: int, mant_bytes: int = 4) -> "BfpVec":
        """Planes [z_lo, z_hi) of the padded global grid (slowest axis) plus halo planes."""
        h = C.c_void_p()
        _raise(lib().bfp_vec_create_slab(dim, level, z_lo, z_hi, mant_bytes, C.byref(h)),
               "bfp_vec_create_slab")
        v = BfpVec(h.value, dim, level, mant_bytes)
        v.z_lo, v.z_hi = z_lo, z_hi
        return v

    def planes(self):
        """(first, last, halo_lo, halo_hi) device pointers and bytes per plane."""
        f, l, hl, hh, nb = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_int64()
        _raise(lib().bfp_vec_planes(self.h, C.byref(f), C.byref(l), C.byref(hl), C.byref(hh),
                                    C.byref(nb)), "bfp_vec_planes")
        return f.value, l.value, hl.value, hh.value, nb.value

    @staticmethod
    def from_mantissas(m: Sequence[int], q: int, e: int, dim: int = 0, level: int = 0,
                       mant_bytes: int = 8) -> "BfpVec":
        v = BfpVec.grid(dim, level, mant_bytes) if dim else BfpVec.flat(len(m), mant_bytes)
        v.upload(m, q, e)
        return v

    @staticmethod
    def _view(handle: int, dim: int, level: int, mant_bytes: int, owner=None) -> "BfpVec":
        """Non-owning view of a vector owned by the library (e.g. a solver's)."""
        v = BfpVec(handle, dim, level, mant_bytes)
        v._owned, v._owner = False, owner
        return v

    def __del__(self):
        try:
            if getattr(self, "_owned", True) and self.h and self.h.value:
                lib().bfp_vec_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def __len__(self) -> int:
        return int(lib().bfp_vec_size(self.h))

    def upload(self, m, q: int, e: int):
        a = np.ascontiguousarray(np.asarray(m, dtype=np.int64))
        if a.size != len(self):
            raise InvalidArgument(ERR_ARG, "upload: size mismatch")
        _raise(lib().bfp_vec_upload(self.h, a.ctypes.data_as(C.c_void_p), q, e, _s()), "upload")
        hh = _Header()
        _raise(lib().bfp_vec_header(self.h, C.byref(hh), _s()), "upload")  # check_fits

    def header(self) -> _Header:
        hh = _Header()
        _raise(lib().bfp_vec_header(self.h, C.byref(hh), _s()), "header")
        return hh

    def download(self) -> Tuple[np.ndarray, int, int]:
        """(mantissas int64, q, e) with pending shifts applied."""
        n = len(self)
        out = np.zeros(max(n, 1), dtype=np.int64)
        hh = _Header()
        _raise(lib().bfp_vec_download(self.h, out.ctypes.data_as(C.c_void_p), C.byref(hh), _s()),
               "download")
        return out[:n], int(hh.q), int(hh.e)

    @property
    def q(self) -> int:
        return int(self.header().q)

    @property
    def e(self) -> int:
        return int(self.header().e)

    @property
    def flags(self) -> int:
        return int(self.header().flags)

    def mantissas(self) -> np.ndarray:
        return self.download()[0]

    def is_zero(self) -> bool:
        return self.header().max_abs == 0

    def zero(self, q: int):
        _raise(lib().bfp_vec_zero(self.h, q, _s()), "zero")
        return self


def zero_vec(n: int, q: int, mant_bytes: int = 8) -> BfpVec:
    """BfpBlock::zero_vec (src/bfp.cpp:53-55): all zero, e = 0."""
    return BfpVec.flat(n, mant_bytes).zero(q)


def _like(x: BfpVec) -> BfpVec:
    return BfpVec.grid(x.dim, x.level, x.mant_bytes) if x.dim else BfpVec.flat(len(x), x.mant_bytes)


def normalize(x: BfpVec) -> BfpVec:
    out = _like(x)
    _raise(lib().bfp_normalize(x.h, out.h, _s()), "normalize")
    return out


def quantize(x: BfpVec, w: int) -> BfpVec:
    out = _like(x)
    _raise(lib().bfp_quantize(x.h, w, out.h, _s()), "quantize")
    return out


def inf_norm_upper(x: BfpVec, q_gamma: int = 16) -> Scalar:
    m, q, e = C.c_int64(), C.c_int64(), C.c_int64()
    _raise(lib().bfp_inf_norm_upper(x.h, q_gamma, C.byref(m), C.byref(q), C.byref(e), _s()),
           "inf_norm_upper")
    return Scalar(m.value, q.value, e.value)


def _i192(w) -> int:
    v = int(w[0]) | (int(w[1]) << 64) | (int(w[2]) << 128)
    return v - (1 << 192) if v >> 191 else v


def dot_exact(x: BfpVec, y: BfpVec) -> Tuple[int, int]:
    """Exact sum_i m_x m_y as a Python int (192-bit device accumulation), and its exponent
    e_x + e_y."""
    w, e = (C.c_uint64 * 3)(), C.c_int64()
    _raise(lib().bfp_dot_exact192(x.h, y.h, w, C.byref(e), _s()), "dot_exact")
    return _i192(w), e.value


def dot_exact128(x: BfpVec, y: BfpVec) -> Tuple[int, int]:
    """The 128-bit entry point (bfp_dot_exact): raises WidthError when the exact value does
    not fit 128 bits."""
    hi, lo, e = C.c_int64(), C.c_uint64(), C.c_int64()
    _raise(lib().bfp_dot_exact(x.h, y.h, C.byref(hi), C.byref(lo), C.byref(e), _s()),
           "dot_exact128")
    return (hi.value << 64) | lo.value, e.value


def dot_value(acc: Sequence[int]) -> int:
    """Exact value of a device limb accumulator {L0, L1, L2, L3, e} (bfp_dot_value)."""
    a = (C.c_int64 * 5)(*[int(v) for v in acc[:5]])
    w = (C.c_uint64 * 3)()
    lib().bfp_dot_value(a, w, None, None)
    return _i192(w)


def dot_exact_async(x: BfpVec, y: BfpVec, d_acc: int):
    """Stream-ordered exact dot into a device int64[5] accumulator (no synchronisation)."""
    _raise(lib().bfp_dot_exact_async(x.h, y.h, C.c_void_p(d_acc), _s()), "dot_exact_async")


def dump_block(x: BfpVec) -> str:
    n = lib().bfp_vec_dump(x.h, None, 0, _s())
    if n < 0:
        _raise(int(-n), "dump_block")
    buf = C.create_string_buffer(int(n))
    lib().bfp_vec_dump(x.h, buf, n, _s())
    return buf.value.decode()


def parse_block(text: str) -> BfpVec:
    h = C.c_void_p()
    _raise(lib().bfp_vec_parse(text.encode(), C.byref(h), _s()), "parse_block")
    return BfpVec(h.value, 0, 0, 8)


# ---------------------------------------------------------------------------
# windowed BLAS


@dataclass
class QcompResult:
    z: BfpVec
    overflow: bool
    underflow: bool
    recomputed: bool


def _result(out: BfpVec) -> QcompResult:
    f = out.header().flags
    return QcompResult(out, bool(f & FLAG_OVERFLOW), bool(f & FLAG_UNDERFLOW),
                       bool(f & FLAG_RECOMPUTED))


def _chk_window(w_out, w_tmp, gamma: Scalar, qc: bool):
    if w_out < 1 or (qc and w_out > w_tmp):
        raise InvalidArgument(ERR_ARG, "qcomp: need 0 < w_out <= w_tmp")
    if gamma.m <= 0:
        raise InvalidArgument(ERR_ARG, "gamma must be > 0")


def _out_for(x: BfpVec, n: Optional[int] = None, w: int = 0) -> BfpVec:
    mb = 8 if (w > 32 or x.mant_bytes == 8) else x.mant_bytes
    if x.dim:
        return BfpVec.grid(x.dim, x.level, x.mant_bytes)
    return BfpVec.flat(len(x) if n is None else n, mb)


def qaxpby(x, y, alpha: Scalar, beta: Scalar, w_out, w_tmp, gamma: Scalar, force=False,
           nn=False) -> QcompResult:
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = _out_for(x)
    _raise(lib().bfp_axpby(x.h, y.h, alpha.c(), beta.c(), int(nn), w_out, w_tmp, gamma.c(),
                           int(force), out.h, _s()), "qaxpby")
    return _result(out)


def qsub(x, y, w_out, w_tmp, gamma) -> QcompResult:
    return qaxpby(x, y, bfp_one(), bfp_minus_one(), w_out, w_tmp, gamma)


def nnqaxpby(x, y, alpha, beta, w_out, gamma) -> QcompResult:
    return qaxpby(x, y, alpha, beta, w_out, w_out, gamma, nn=True)


def nnqsub(x, y, w_out, gamma) -> QcompResult:
    return nnqaxpby(x, y, bfp_one(), bfp_minus_one(), w_out, gamma)


class BfpCsr:
    """BfpCsr (include/bfpmg/bfp.hpp:62-84) on the device."""

    def __init__(self, rows, cols, rowptr, col, m, q, e):
        self.rows, self.cols, self.q, self.e = rows, cols, q, e
        rp = np.ascontiguousarray(rowptr, dtype=np.int64)
        cl = np.ascontiguousarray(col if len(col) else [0], dtype=np.int64)
        mm = np.ascontiguousarray(m if len(m) else [0], dtype=np.int64)
        h = C.c_void_p()
        _raise(lib().bfp_csr_create(rows, cols, rp.ctypes.data_as(C.c_void_p),
                                    cl.ctypes.data_as(C.c_void_p), mm.ctypes.data_as(C.c_void_p),
                                    q, e, C.byref(h)), "BfpCsr")
        self.h = h
        self.max_row_nnz = int(max((rp[i + 1] - rp[i] for i in range(rows)), default=0))

    def __del__(self):
        try:
            lib().bfp_csr_destroy(self.h)
        except Exception:
            pass


def qspmv(a: BfpCsr, x: BfpVec, w_out, w_tmp, gamma, m_a=0, force=False, nn=False):
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = BfpVec.flat(a.rows, x.mant_bytes)
    _raise(lib().bfp_spmv_csr(a.h, x.h, m_a, int(nn), w_out, w_tmp, gamma.c(), int(force), out.h,
                              _s()), "qspmv")
    return _result(out)


def nnqspmv(a, x, w_out, gamma, m_a=0):
    return qspmv(a, x, w_out, w_out, gamma, m_a, nn=True)


def qgemv(a: BfpCsr, x: BfpVec, y: BfpVec, alpha, beta, w_out, w_tmp, gamma, m_a=0, force=False,
          nn=False):
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = BfpVec.flat(a.rows, x.mant_bytes)
    _raise(lib().bfp_gemv_csr(a.h, x.h, y.h, alpha.c(), beta.c(), m_a, int(nn), w_out, w_tmp,
                              gamma.c(), int(force), out.h, _s()), "qgemv")
    return _result(out)


def nnqgemv(a, x, y, alpha, beta, w_out, gamma, m_a=0):
    return qgemv(a, x, y, alpha, beta, w_out, w_out, gamma, m_a, nn=True)


def qcomp_rows(rows: Sequence[int], q: int, e: int, w_out, w_tmp, gamma: Scalar, force=False,
               nn=False, mant_bytes=8) -> QcompResult:
    """qcomp / nnqcomp over a FixedKernel of exact rows (tests/test_blas.cpp:14-26)."""
    _chk_window(w_out, w_tmp, gamma, not nn)
    n = len(rows)
    hi = np.array([(int(v) >> 64) for v in rows] or [0], dtype=np.int64)
    lo = np.array([(int(v) & ((1 << 64) - 1)) for v in rows] or [0], dtype=np.uint64)
    out = BfpVec.flat(n, mant_bytes)
    _raise(lib().bfp_qcomp_rows(n, hi.ctypes.data_as(C.c_void_p), lo.ctypes.data_as(C.c_void_p),
                                q, e, int(nn), w_out, w_tmp, gamma.c(), int(force), out.h, _s()),
           "qcomp_rows")
    return _result(out)


# ---------------------------------------------------------------------------
# stencil family


def stencil_gemv(x, y, alpha, beta, w_out, w_tmp, gamma, force=False, nn=False, out=None):
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = out or _like(x)
    _raise(lib().bfp_stencil_gemv(x.h, y.h, alpha.c(), beta.c(), int(nn), w_out, w_tmp,
                                  gamma.c(), int(force), out.h, _s()), "stencil_gemv")
    return _result(out)


def residual(x, b, w_out, w_tmp, gamma, nn=False, out=None):
    """r = b - A x (the fine-level residual; alpha = -1, beta = +1)."""
    return stencil_gemv(x, b, bfp_minus_one(), bfp_one(), w_out, w_tmp, gamma, nn=nn, out=out)


def jacobi(x, b, c: Scalar, w_out, w_tmp, gamma, nn=False, out=None):
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = out or _like(x)
    _raise(lib().bfp_stencil_jacobi(x.h, b.h, c.c(), int(nn), w_out, w_tmp, gamma.c(), out.h,
                                    _s()), "jacobi")
    return _result(out)


def scal(r, c: Scalar, w_out, w_tmp, gamma, nn=False):
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = _like(r)
    _raise(lib().bfp_scal(r.h, c.c(), int(nn), w_out, w_tmp, gamma.c(), out.h, _s()), "scal")
    return _result(out)


def restrict_fw(r, w_out, w_tmp, gamma, nn=False):
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = BfpVec.grid(r.dim, r.level - 1, r.mant_bytes)
    _raise(lib().bfp_restrict_fw(r.h, int(nn), w_out, w_tmp, gamma.c(), out.h, _s()), "restrict")
    return _result(out)


def prolong(xc, w_out, w_tmp, gamma, nn=False):
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = BfpVec.grid(xc.dim, xc.level + 1, xc.mant_bytes)
    _raise(lib().bfp_prolong(xc.h, int(nn), w_out, w_tmp, gamma.c(), out.h, _s()), "prolong")
    return _result(out)


def prolong_correct(ec, y, w_out, w_tmp, gamma, nn=False):
    _chk_window(w_out, w_tmp, gamma, not nn)
    out = _like(y)
    _raise(lib().bfp_prolong_correct(ec.h, y.h, int(nn), w_out, w_tmp, gamma.c(), out.h, _s()),
           "prolong_correct")
    return _result(out)


def quantize_exact(z: Sequence[int], k: Sequence[int], w: int, mant_bytes: int = 8,
                   dim: int = 0, level: int = 0, out: Optional[BfpVec] = None) -> BfpVec:
    """quantize_exact (src/bfp.cpp:163-187) of entries z_i 2^k_i on the device (int64 z),
    into a new vector or into `out`."""
    za = np.ascontiguousarray(np.asarray(z, dtype=np.int64))
    ka = np.ascontiguousarray(np.asarray(k, dtype=np.int64))
    if za.shape != ka.shape:
        raise InvalidArgument(ERR_ARG, "quantize_exact: size mismatch")
    if out is None:
        out = BfpVec.grid(dim, level, mant_bytes) if dim else BfpVec.flat(len(za), mant_bytes)
    _raise(lib().bfp_quantize_exact(za.ctypes.data_as(C.c_void_p), ka.ctypes.data_as(C.c_void_p),
                                    len(za), w, out.h, _s()), "quantize_exact")
    return out


def from_doubles(v: Sequence[float], w: int, mant_bytes: int = 8, dim: int = 0,
                 level: int = 0) -> BfpVec:
    """from_extfloat (src/bfp.cpp:189-194) for IEEE doubles (exact z 2^k split)."""
    a = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    out = BfpVec.grid(dim, level, mant_bytes) if dim else BfpVec.flat(len(a), mant_bytes)
    _raise(lib().bfp_from_doubles(a.ctypes.data_as(C.c_void_p), len(a), w, out.h, _s()),
           "from_doubles")
    return out


def jacobi_coeff(dim: int, level: int, qc: int = 16) -> Scalar:
    s = _Scalar()
    _raise(lib().bfp_jacobi_coeff(dim, level, qc, C.byref(s)), "jacobi_coeff")
    return Scalar(s.m, s.q, s.e)


def gen_uniform(v: BfpVec, p: int, seed: int, stream_id: int) -> BfpVec:
    _raise(lib().bfp_gen_uniform(v.h, p, seed, stream_id, _s()), "gen_uniform")
    return v


def gen_sine(v: BfpVec, p: int) -> BfpVec:
    _raise(lib().bfp_gen_sine(v.h, p, _s()), "gen_sine")
    return v


# ---------------------------------------------------------------------------
# multigrid solver


class PrecisionSchedule:
    """Per-level mantissa widths, 1-based (index 0 unused): wcheck (inputs / matrices), w
    (working) and wdot (inner), with wcheck >= w >= wdot >= 1 -- the reference's
    PrecisionSchedule (P/include/bfpmg/multigrid.hpp:16-27, P/src/multigrid.cpp:13-44)."""

    def __init__(self, wcheck: Sequence[int], w: Sequence[int], wdot: Sequence[int]):
        self.wcheck, self.w, self.wdot = list(wcheck), list(w), list(wdot)

    @classmethod
    def flat(cls, levels: int, wc: int, ww: int, wd: int) -> "PrecisionSchedule":
        return cls([0] + [wc] * levels, [0] + [ww] * levels, [0] + [wd] * levels)

    @classmethod
    def affine(cls, levels: int, m: int, k: int, q_check: int, q_w: int,
               q_dot: int) -> "PrecisionSchedule":
        """wcheck_j = (m + k) j + q_check, w_j = k j + q_w, wdot_j = m j + q_dot, clamped so
        that the ordering invariant holds on every level (:22-35)."""
        wc, w, wd = [0], [0], [0]
        for j in range(1, levels + 1):
            wj = k * j + q_w
            w.append(wj)
            wc.append(max((m + k) * j + q_check, wj))
            wd.append(min(m * j + q_dot, wj))
        return cls(wc, w, wd)

    def levels(self) -> int:
        return len(self.w) - 1

    def validate(self) -> None:
        """Raises ValueError (the reference's std::invalid_argument, :37-44)."""
        for j in range(1, self.levels() + 1):
            if not (self.wcheck[j] >= self.w[j] >= self.wdot[j] >= 1):
                raise ValueError(f"PrecisionSchedule: width ordering violated at level {j}")


# step names of the reference (P/src/multigrid.cpp:49-60); the config-mode driver adds the
# first sweep from zero and the diagnostic final residual
REF_STEP_NAMES = {"ir-residual", "ir-correction", "v-relax", "v-residual", "v-restrict",
                  "v-correct", "fmg-prolong"}


def gamma_str(gm: int, ge: int, digits: int = 6) -> str:
    """gamma = gm 2^ge printed like the reference's ExtFloat::str(6) (mpfr "%.6Rg",
    P/src/extfloat.cpp:65-73): the exact value rounded to `digits` significant digits."""
    from fractions import Fraction
    v = Fraction(gm) * (Fraction(2) ** ge)
    try:
        f = float(v)
        if f != 0.0 and Fraction(f) == v:
            return "%.*g" % (digits, f)
    except OverflowError:
        pass
    if v == 0:
        return "0"
    # beyond double range: scientific notation from the exact rational
    import math
    neg, a = v < 0, abs(v)
    e10 = int(math.floor((a.numerator.bit_length() - a.denominator.bit_length()) * 0.30103))
    while a >= Fraction(10) ** (e10 + 1):
        e10 += 1
    while a < Fraction(10) ** e10:
        e10 -= 1
    scaled = a / Fraction(10) ** (e10 - digits + 1)
    n = int(scaled)
    rem = scaled - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2):
        n += 1
    if n == 10 ** digits:
        n //= 10
        e10 += 1
    mant = str(n).rstrip("0") or "0"
    mant = mant[0] + ("." + mant[1:] if len(mant) > 1 else "")
    return ("-" if neg else "") + f"{mant}e{'+' if e10 >= 0 else '-'}{abs(e10):02d}"


@dataclass
class TraceRecord:
    """One run_step record (P/include/bfpmg/multigrid.hpp:74-87)."""
    step: int
    level: int
    w_out: int
    w_tmp: int
    gm: int
    ge: int
    overflow: int
    underflow: int
    recomputed: int
    normalized: int

    def step_name(self) -> str:
        return STEP_NAMES[self.step]

    def to_line(self) -> str:
        """TraceRecord::to_line (P/src/multigrid.cpp:157-163), byte for byte."""
        return (f"{self.step_name()} level={self.level} w_out={self.w_out} w_tmp={self.w_tmp} "
                f"gamma={gamma_str(self.gm, self.ge)} overflow={int(bool(self.overflow))} "
                f"underflow={int(bool(self.underflow))} recompute={int(bool(self.recomputed))} "
                f"normalized={int(bool(self.normalized))}")


class SolverTrace:
    """SolverTrace (P/include/bfpmg/multigrid.hpp:89-94) over a solve's trace records."""

    def __init__(self, records):
        self.records = [r if isinstance(r, TraceRecord) else TraceRecord(*r) for r in records]

    def recomputes_at_level(self, level: int) -> int:  # P/src/multigrid.cpp:165-170
        return sum(1 for r in self.records if r.level == level and (r.overflow or r.underflow))

    def calls_at_level(self, level: int) -> int:       # :172-177
        return sum(1 for r in self.records if r.level == level)

    def lines(self) -> List[str]:
        return [r.to_line() for r in self.records]


def _lv(v):
    if v is None:
        return [0] * 32
    if isinstance(v, int):
        return [v] * 32
    return list(v) + [0] * (32 - len(v))


def mg_config(d, l_fine, l_coarse=2, nu1=2, nu2=2, n_coarse=16, cycles=1, fmg=False,
              nonnormalized=False, x0_random=False, rhs_kind=1, qc=16, seed=1, p=None, pd=None,
              pc=None, w_add_cap=-1, fuse_points=-1) -> MgConfig:
    """Solver config; p / pd / pc are the PrecisionSchedule w / wdot / wcheck per level."""
    cfg = MgConfig()
    cfg.d, cfg.l_fine, cfg.l_coarse, cfg.nu1, cfg.nu2 = d, l_fine, l_coarse, nu1, nu2
    cfg.n_coarse, cfg.cycles, cfg.fmg = n_coarse, cycles, int(fmg)
    cfg.nonnormalized = 2 if nonnormalized == "hybrid" else int(nonnormalized)  # NormMode
    cfg.x0_random, cfg.rhs_kind, cfg.qc, cfg.seed = int(x0_random), rhs_kind, qc, seed
    p, pd, pc = _lv(p), _lv(pd), _lv(pc)
    for i in range(32):
        cfg.p[i], cfg.pd[i], cfg.pc[i] = p[i], pd[i], pc[i]
    cfg.w_add_cap = w_add_cap
    cfg.fuse_points = fuse_points
    return cfg


def mg_config_ref(l_fine, rho, eta, w, wdot=None, wcheck=None, cycles=1, fmg=False,
                  x0_random=False, rhs_kind=1, seed=1, ext_prec=400, w_add_cap=-1,
                  d=1) -> MgConfig:
    """Reference-algorithm mode (d = 1 or 2): the reference solver P/src/multigrid.cpp:430-518
    on its own p = 1 operators (2-D: the bilinear-FEM 9-point operator, P = P1 (x) P1,
    R = P^T), see include/bfpmg_b200.h.  rho / eta: the Chebyshev parameters
    (Hierarchy::set_eta); w / wdot / wcheck: PrecisionSchedule widths (int or per-level
    list, index = level, levels 1..l_fine; >= 3 in 1-D, >= 5 in 2-D)."""
    from . import refmode
    if isinstance(w, PrecisionSchedule):  # the reference's schedule object
        w.validate()
        w, wdot, wcheck = w.w, w.wdot, w.wcheck
    cfg = mg_config(d, l_fine, l_coarse=1, cycles=cycles, fmg=fmg, x0_random=x0_random,
                    rhs_kind=rhs_kind, seed=seed, p=w, pd=wdot, pc=wcheck, w_add_cap=w_add_cap,
                    fuse_points=0)
    cfg.ref_mode = 1
    c1, kres, c1d, c2d = refmode.chebyshev_scalars(rho, eta, ext_prec,
                                                   [cfg.pd[l] or cfg.p[l] for l in range(32)])
    for dst, src in ((cfg.ref_c1, c1), (cfg.ref_kres, kres)):
        dst.hi, dst.lo, dst.e, dst.sticky = src
    for l in range(1, l_fine + 1):
        cfg.ref_c1d[l].m, cfg.ref_c1d[l].q, cfg.ref_c1d[l].e = c1d[l]
        cfg.ref_c2d[l].m, cfg.ref_c2d[l].q, cfg.ref_c2d[l].e = c2d[l]
    return cfg


NCCL_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    """An NCCL unique id (make it on one rank, broadcast it to the others)."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _raise(lib().bfp_nccl_unique_id(buf, NCCL_ID_BYTES), "bfp_nccl_unique_id")
    return buf.raw


class DistOps:
    """Sharded stencil ops over z-slabs (native: halo exchange, partial windows, MAX
    all-reduce and finalize enqueued on the stream, no host synchronisation).

    ``nccl_id`` (from :func:`nccl_unique_id`) makes this process ``rank`` of an NCCL
    group of ``world``; without it the ``world`` ranks run in this process (every call
    then takes one slab per rank)."""

    def __init__(self, world: int, rank: int = 0, nccl_id: Optional[bytes] = None):
        h = C.c_void_p()
        idb = C.create_string_buffer(nccl_id, NCCL_ID_BYTES) if nccl_id is not None else None
        _raise(lib().bfp_dist_create(world, rank, idb, C.byref(h)), "bfp_dist_create")
        self.h, self.world = h, world
        self.local = world if nccl_id is None else 1

    def __del__(self):
        try:
            lib().bfp_dist_destroy(self.h)
        except Exception:
            pass

    def _arr(self, vs):
        if len(vs) != self.local:
            raise InvalidArgument(ERR_ARG, f"expected {self.local} slabs")
        return (C.c_void_p * len(vs))(*[v.h.value for v in vs])

    def gemv(self, xs, ys, alpha: Scalar, beta: Scalar, w_out: int, w_tmp: int, gamma: Scalar,
             outs, nn: bool = False):
        _raise(lib().bfp_dist_stencil_gemv(self.h, self._arr(xs), self._arr(ys), alpha.c(),
                                           beta.c(), int(nn), w_out, w_tmp, gamma.c(),
                                           self._arr(outs), _s()), "bfp_dist_stencil_gemv")

    def dot(self, xs, ys, accs):
        """Sharded exact dot: per-rank limb accumulators (device int64[5] pointers, one per
        local rank) all-reduced with an int64 SUM; returns nothing (stream-ordered)."""
        arr = (C.c_void_p * len(accs))(*[int(a) for a in accs])
        _raise(lib().bfp_dist_dot_exact(self.h, self._arr(xs), self._arr(ys), arr, _s()),
               "bfp_dist_dot_exact")

    def jacobi(self, xs, bs, c: Scalar, w_out: int, w_tmp: int, gamma: Scalar, outs,
               nn: bool = False):
        _raise(lib().bfp_dist_stencil_jacobi(self.h, self._arr(xs), self._arr(bs), c.c(), int(nn),
                                             w_out, w_tmp, gamma.c(), self._arr(outs), _s()),
               "bfp_dist_stencil_jacobi")


class Multigrid:
    """Device multigrid solver: IR with Jacobi V(nu1,nu2) cycles, or FMG.

    ``world > 1`` shards the levels with >= ``min_planes`` planes per rank into slabs
    (d >= 2) and replicates the coarser ones; ``nccl_id`` (bytes from
    :func:`nccl_unique_id`) makes this process ``rank`` of an NCCL group, without it
    all ``world`` ranks run in this process on the current device."""

    def __init__(self, cfg: MgConfig, world: int = 1, rank: int = 0,
                 nccl_id: Optional[bytes] = None, min_planes: int = 16):
        h = C.c_void_p()
        if world == 1 and nccl_id is None:
            _raise(lib().bfp_mg_create(C.byref(cfg), C.byref(h)), "bfp_mg_create")
        else:
            idb = C.create_string_buffer(nccl_id, NCCL_ID_BYTES) if nccl_id is not None else None
            _raise(lib().bfp_mg_create_sharded(C.byref(cfg), world, rank, idb, min_planes,
                                               C.byref(h)), "bfp_mg_create_sharded")
        self.h, self.cfg, self.world = h, cfg, world
        self.local = world if nccl_id is None else 1

    def rank_result(self, local_rank: int = 0):
        """(x_final, r_final, rank, lowest sharded level) of a local rank; x/r are
        non-owning BfpVec views (slabs on sharded levels)."""
        x, r, rk, ls = C.c_void_p(), C.c_void_p(), C.c_int(), C.c_int()
        _raise(lib().bfp_mg_rank_result(self.h, local_rank, C.byref(x), C.byref(r), C.byref(rk),
                                        C.byref(ls)), "bfp_mg_rank_result")
        mb = 4
        xv = BfpVec._view(x.value, self.cfg.d, self.cfg.l_fine, mb, self)
        rv = BfpVec._view(r.value, self.cfg.d, self.cfg.l_fine, mb, self)
        return xv, rv, rk.value, ls.value

    def __del__(self):
        try:
            lib().bfp_mg_destroy(self.h)
        except Exception:
            pass

    def solve(self, use_graph: bool = False):
        _raise(lib().bfp_mg_solve(self.h, int(use_graph), _s()), "bfp_mg_solve")

    def launches(self) -> int:
        return int(lib().bfp_mg_kernel_launches(self.h))

    def transport(self) -> str:
        """Transport of the per-op exponent all-reduce ("local-kernel", "peer-mailbox",
        "nccl-allreduce")."""
        return TRANSPORTS[int(lib().bfp_mg_transport(self.h))]

    def result(self, trace_cap: int = 1 << 20):
        n = ((1 << self.cfg.l_fine) - 1) ** self.cfg.d
        x = np.zeros(n, dtype=np.int64)
        hh = _Header()
        hist = np.zeros(4096, dtype=np.float64)
        tr = (TraceRec * trace_cap)()
        nh, nt = C.c_int(), C.c_int64()
        _raise(lib().bfp_mg_result(self.h, x.ctypes.data_as(C.c_void_p), C.byref(hh),
                                   hist.ctypes.data_as(C.c_void_p), 4096, C.byref(nh), tr,
                                   trace_cap, C.byref(nt), _s()), "bfp_mg_result")
        trace = [(t.step, t.level, t.w_out, t.w_tmp, t.gm, t.ge, t.overflow, t.underflow,
                  t.recomputed, t.normalized) for t in tr[: min(nt.value, trace_cap)]]
        return x, int(hh.q), int(hh.e), hist[: nh.value].tolist(), trace

    def trace(self, trace_cap: int = 1 << 20) -> SolverTrace:
        """The solve's records as the reference's SolverTrace."""
        return SolverTrace(self.result(trace_cap)[4])

    def level_rhs(self, level: int) -> BfpVec:
        """The solver's right-hand side of `level` (rhs_kind 3: written by the caller before a
        solve; include/bfpmg_b200.h: bfp_mg_level_rhs).  The solver owns the vector."""
        b, mb = C.c_void_p(), C.c_int()
        _raise(lib().bfp_mg_level_rhs(self.h, level, C.byref(b), C.byref(mb)), "bfp_mg_level_rhs")
        v = BfpVec(b.value, self.cfg.d, level, mb.value)
        v._owned = False
        v._keep = self  # the handle lives as long as the solver
        return v

    def vectors(self):
        x, b, r = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _raise(lib().bfp_mg_vectors(self.h, C.byref(x), C.byref(b), C.byref(r)), "bfp_mg_vectors")
        return x, b, r


TRANSPORTS = {0: "local-kernel", 1: "peer-mailbox", 2: "nccl-allreduce"}


def set_transport(t: int):
    """Exponent all-reduce transport of sharded solvers created afterwards
    (include/bfpmg_b200.h: bfp_set_transport)."""
    _raise(lib().bfp_set_transport(int(t)), "bfp_set_transport")


def launch_count() -> int:
    return int(lib().bfp_launch_count())


KERNEL_FAMILIES = ["grid", "bulk2", "bulk3", "march", "pro3", "rst3", "pro2", "rst2", "flat",
                   "fused", "coarse"]


def kernel_family_counts() -> dict:
    """Windowed-kernel launches since load per kernel family (include/bfpmg_b200.h)."""
    a = (C.c_int64 * 16)()
    _raise(lib().bfp_kernel_family_counts(a, 16), "bfp_kernel_family_counts")
    return {n: int(a[i]) for i, n in enumerate(KERNEL_FAMILIES)}


def device_sync():
    _raise(lib().bfp_device_sync(_s()), "sync")


def profile_enable(on: bool = True):
    _raise(lib().bfp_profile_enable(int(on)), "profile_enable")


def profile_read(reset: bool = True) -> Tuple[float, int]:
    """(summed device ms, launches) of pass-1 / nnqcomp kernels since the last reset."""
    t, n = C.c_double(), C.c_int64()
    _raise(lib().bfp_profile_read(C.byref(t), C.byref(n), int(reset)), "profile_read")
    return t.value, n.value


def set_kernel_path(bulk: bool = True, pdl: bool = True, skip_recompute: bool = False):
    """Kernel-path switches (see include/bfpmg_b200.h); results are bit-identical."""
    flags = int(bulk) | (0 if pdl else 2) | (4 if skip_recompute else 0)
    _raise(lib().bfp_set_kernel_path(flags), "set_kernel_path")
