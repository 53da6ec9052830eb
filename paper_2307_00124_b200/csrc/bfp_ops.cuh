// bfp_ops.cuh -- exact-row "ExactKernel" functors for sm_100a.
//
// Each op mirrors one reference ExactKernel (include/bfpmg/blas.hpp:25-31):
// setup() computes the reference template exponent e* from the DEVICE headers
// of its operands (src/blas.cpp:41-58, 74-82, 96-120) plus a tight bound on the
// accumulator width from the operands' ACTUAL max/min mantissas, so the
// kernel picks int64 or __int128 accumulation uniformly per launch; eval4()
// produces 4 consecutive exact rows at an output storage offset.
//
// Grid vectors use a padded layout: pitch N = 2^l on
// every axis, index N-1 of each axis is a zero pad, plus a zero halo in front
// and behind.  Every Dirichlet neighbour is therefore a plain load of a zero,
// and every 4-group of outputs is one aligned 128-bit (int32) store.
#pragma once
#include "bfp_dev.cuh"

namespace bfpdev {

__host__ __device__ __forceinline__ int64_t ceil_log2_h(int64_t m) {
  int64_t r = 0, v = 1;
  while (v < m) {
    v <<= 1;
    ++r;
  }
  return r;
}
__host__ __device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

struct Scal {
  int64_t m, q, e;
};

// eaxpby setup (src/blas.cpp:46-58): d = ea - eb, e* = min(ea, eb)
__device__ __forceinline__ void axpby_setup(int64_t ea, int64_t eb, int64_t& d, int64_t& es) {
  d = ea - eb;
  es = imin(ea, eb);
}
// eaxpby setup with all-zero terms dropped: when exactly one term is zero (za / zb), its
// alignment shift is dropped too (d = 0, e* = the other term's exponent) and zd grows by
// e* - min(ea, eb).  Every row then equals the reference row / 2^zd exactly (the dropped
// term contributes nothing), so qcomp/nnqcomp give identical windows in these shifted
// coordinates (only an all-zero qcomp result needs zd: win_finalize).  Without it a zero
// block at e = 0 next to a far-away operand (b = 0 with a diverging iterate, C5 p = 4)
// would push the rows past 127 bits where the reference's mpz rows are just long.
__device__ __forceinline__ void axpby_setup_z(int64_t ea, int64_t eb, bool za, bool zb,
                                              int64_t& d, int64_t& es, int64_t& zd) {
  axpby_setup(ea, eb, d, es);
#ifndef BFP_AB_NO_ELIDE
  if (za != zb) {
    const int64_t ee = za ? eb : ea;
    zd += ee - es;
    es = ee;
    d = 0;
  }
#endif
}
__device__ __forceinline__ bool hdr_zero(const Hdr* h) { return max_abs(h) == 0; }
// One read of a block's published state for the one-thread op setups: every derived
// quantity below comes from these four words (no re-reads between the setup's stores).
struct HSnap {
  int64_t e, shift, bits;  // bits = zbits (0: the block is all zero)
};
__device__ __forceinline__ HSnap hsnap(const Hdr* h) {
  const int64_t e = h->e, s = h->shift, mx = h->max_m, mn = h->min_m;
  const int64_t a = mx >> s, b = mn >> s;
  const int ma = msb(a), mb = msb(b);
  return HSnap{e, s, (a | b) ? (ma > mb ? ma : mb) : 0};
}
// alpha*a*2^max(d,0) + beta*b*2^max(-d,0)  (src/blas.cpp:60-72, 133-141)
template <typename A>
__device__ __forceinline__ A combine(int64_t am, A a, int64_t bm, A b, int64_t d) {
  // shift counts beyond the accumulator only occur on provably-zero operands
  // (the width bound of setup() excludes them), so clamping is exact.
  constexpr int64_t B = AccBits<A>::value - 1;
  A ta = (A)am * a, tb = (A)bm * b;
  if (d < 0)
    tb = tb << (int)imin(-d, B);
  else
    ta = ta << (int)imin(d, B);
  return ta + tb;
}
// combine with 64-bit operand products (exact when msb(am) + bits(a) <= 63 and
// msb(bm) + bits(b) <= 63), widened to A only for the power-of-two shift
template <typename A>
__device__ __forceinline__ A combine_w(int64_t am, int64_t a, int64_t bm, int64_t b, int64_t d) {
  constexpr int64_t B = AccBits<A>::value - 1;
  A ta = (A)(am * a), tb = (A)(bm * b);
  if (d < 0)
    tb = tb << (int)imin(-d, B);
  else
    ta = ta << (int)imin(d, B);
  return ta + tb;
}
#ifndef BFP_W128_PTX
#define BFP_W128_PTX 1
#endif
// Two-word rows for the int64-storage fast window (all shift counts < 64, uniform per
// launch): value = hi * 2^64 + lo, two's complement over 128 bits.
struct W128 {
  uint64_t lo;
  int64_t hi;
};
__device__ __forceinline__ W128 w_shl(int64_t a, int s) {  // a * 2^s, 0 <= s < 64
  return W128{(uint64_t)a << s, s ? (a >> (64 - s)) : (a >> 63)};
}
// two-word adds through the carry chain (add.cc / addc: four IADD3s, no compare/select)
__device__ __forceinline__ W128 w_add(W128 x, W128 y) {
#if BFP_W128_PTX
  W128 r;
  asm("add.cc.u64 %0, %2, %4;\n\taddc.u64 %1, %3, %5;"
      : "=l"(r.lo), "=l"(r.hi)
      : "l"(x.lo), "l"(x.hi), "l"(y.lo), "l"(y.hi));
  return r;
#else
  const uint64_t lo = x.lo + y.lo;
  return W128{lo, x.hi + y.hi + (int64_t)(lo < x.lo)};
#endif
}
__device__ __forceinline__ W128 w_add(W128 x, int64_t b) {
  return w_add(x, W128{(uint64_t)b, b >> 63});
}
__device__ __forceinline__ W128 w_mul_u32(W128 x, uint32_t c) {  // x * c mod 2^128
  // 32-bit limbs: four IMAD.WIDE.U32 / IMAD, each limb product absorbing the carry word
  const uint64_t p0 = (uint64_t)(uint32_t)x.lo * c;
  const uint64_t p1 = (uint64_t)(uint32_t)(x.lo >> 32) * c + (p0 >> 32);
  const uint64_t p2 = (uint64_t)(uint32_t)x.hi * c + (p1 >> 32);
  const uint32_t p3 = (uint32_t)((uint64_t)x.hi >> 32) * c + (uint32_t)(p2 >> 32);
  return W128{(p1 << 32) | (uint32_t)p0, (int64_t)(((uint64_t)p3 << 32) | (uint32_t)p2)};
}
__device__ __forceinline__ int64_t w_shr_lo(W128 z, int rs) {  // low word of floor(z/2^rs)
  return (int64_t)(rs ? (z.lo >> rs) | ((uint64_t)z.hi << (64 - rs)) : z.lo);
}
__device__ __forceinline__ void w_or_mag(W128 z, uint64_t& olo, uint64_t& ohi) {
  const uint64_t s = (uint64_t)(z.hi >> 63);
  olo |= z.lo ^ s;
  ohi |= (uint64_t)z.hi ^ s;
}

// width bound of alpha*a*2^max(d,0) + beta*b*2^max(-d,0) given operand widths
// (a width of 0 marks an all-zero operand, whose term is excluded)
__device__ __forceinline__ int64_t combine_bits(int64_t am, int64_t ba, int64_t bm, int64_t bb,
                                                int64_t d) {
  int64_t x = (ba && am) ? msb((int64_t)am) + ba + (d > 0 ? d : 0) : 0;
  int64_t y = (bb && bm) ? msb((int64_t)bm) + bb + (d < 0 ? -d : 0) : 0;
  return imax(imax(x, y), 1) + 1;
}
// width of a block's values, 0 if the block is all zero
__device__ __forceinline__ int64_t zbits(const Hdr* h) { return max_abs(h) ? eff_bits(h) : 0; }
__device__ __forceinline__ int64_t grow(int64_t b, int64_t extra) { return b ? b + extra : 0; }

// ---- vector loads (pending shift applied) ---------------------------------
// NC = true: read-only (non-coherent) path, valid when the data was produced by
// an earlier kernel; NC = false: coherent loads for the fused single-CTA kernel,
// which reads data it wrote itself earlier in the same launch.
template <bool NC, typename T> __device__ __forceinline__ T ldx(const T* p) {
  if constexpr (NC) return __ldg(p);
  else return *p;
}

template <typename M, bool NC = true> struct V4;
template <bool NC> struct V4<int32_t, NC> {
  __device__ static __forceinline__ void load(const Vec& v, int64_t o, int64_t sh, int64_t r[4]) {
    int4 t = ldx<NC>(reinterpret_cast<const int4*>((const int32_t*)v.data + o));
    r[0] = ((int64_t)t.x) >> sh;
    r[1] = ((int64_t)t.y) >> sh;
    r[2] = ((int64_t)t.z) >> sh;
    r[3] = ((int64_t)t.w) >> sh;
  }
  __device__ static __forceinline__ void load32(const Vec& v, int64_t o, int sh, int r[4]) {
    int4 t = ldx<NC>(reinterpret_cast<const int4*>((const int32_t*)v.data + o));
    r[0] = t.x >> sh;
    r[1] = t.y >> sh;
    r[2] = t.z >> sh;
    r[3] = t.w >> sh;
  }
  __device__ static __forceinline__ void store(const Vec& v, int64_t o, const int32_t r[4]) {
    int4 t = make_int4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<int4*>((int32_t*)v.data + o) = t;
  }
};
template <bool NC> struct V4<int64_t, NC> {
  __device__ static __forceinline__ void load(const Vec& v, int64_t o, int64_t sh, int64_t r[4]) {
    const longlong2* p = reinterpret_cast<const longlong2*>((const int64_t*)v.data + o);
    longlong2 a = ldx<NC>(p), b = ldx<NC>(p + 1);
    r[0] = a.x >> sh;
    r[1] = a.y >> sh;
    r[2] = b.x >> sh;
    r[3] = b.y >> sh;
  }
  __device__ static __forceinline__ void store(const Vec& v, int64_t o, const int64_t r[4]) {
    longlong2* p = reinterpret_cast<longlong2*>((int64_t*)v.data + o);
    p[0] = make_longlong2(r[0], r[1]);
    p[1] = make_longlong2(r[2], r[3]);
  }
};
template <typename M, bool NC = true>
__device__ __forceinline__ int64_t ld1(const Vec& v, int64_t o, int64_t sh) {
  return ((int64_t)ldx<NC>((const M*)v.data + o)) >> sh;
}

// pad mask of 4 consecutive grid storage offsets starting at o (o % 4 == 0); z0 is the
// global index of local plane 0 along the slowest axis (slabs), 0 for full grids
__device__ __forceinline__ bool plane_pad(int dim, int l, int z0, int64_t o) {
  const int64_t mask = ((int64_t)1 << l) - 1;
  if (dim == 2) return (o >> l) + z0 == mask;
  if (dim == 3) return ((o >> l) & mask) == mask || (o >> (2 * l)) + z0 == mask;
  return false;
}
__device__ __forceinline__ void pad4(int dim, int l, int64_t o, bool pad[4], int z0 = 0) {
  const int64_t N = (int64_t)1 << l, mask = N - 1;
  const bool rowpad = plane_pad(dim, l, z0, o);
  const int64_t ix = o & mask;
#pragma unroll
  // (ix + j > mask only for the 1-D level 1, N = 2, whose storage is padded to 4)
  for (int j = 0; j < 4; ++j) pad[j] = rowpad || (ix + j >= mask);
}

// 32-bit stencil (used when the width bound proves |S x| < 2^31)
template <bool NC>
__device__ __forceinline__ void stencil4_32(const Vec& x, int sx, int dim, int l, int64_t o,
                                            int g[4], int c[4]) {
  V4<int32_t, NC>::load32(x, o, sx, c);
  const int32_t* p = (const int32_t*)x.data;
  const int lf = ldx<NC>(p + o - 1) >> sx, rt = ldx<NC>(p + o + 4) >> sx;
  int nb[4] = {lf + c[1], c[0] + c[2], c[1] + c[3], c[2] + rt};
  if (dim >= 2) {
    const int64_t N = (int64_t)1 << l;
    int u[4], d[4];
    V4<int32_t, NC>::load32(x, o - N, sx, u);
    V4<int32_t, NC>::load32(x, o + N, sx, d);
#pragma unroll
    for (int j = 0; j < 4; ++j) nb[j] += u[j] + d[j];
    if (dim >= 3) {
      const int64_t N2 = N * N;
      V4<int32_t, NC>::load32(x, o - N2, sx, u);
      V4<int32_t, NC>::load32(x, o + N2, sx, d);
#pragma unroll
      for (int j = 0; j < 4; ++j) nb[j] += u[j] + d[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) g[j] = 2 * dim * c[j] - nb[j];
}
// alpha*g*2^max(d,0) + beta*y*2^max(-d,0) with 32-bit operands, 64-bit result
__device__ __forceinline__ int64_t combine32(int am, int g, int bm, int y, int64_t d) {
  int64_t ta = (int64_t)am * (int64_t)g, tb = (int64_t)bm * (int64_t)y;
  if (d < 0)
    tb <<= (int)imin(-d, 63);
  else
    ta <<= (int)imin(d, 63);
  return ta + tb;
}
__device__ __forceinline__ bool fits32(int64_t v) { return v >= INT32_MIN && v <= INT32_MAX; }
// a * 2^s + add for a 32-bit a and a uniform s in [0, 62] (exact by the width bound):
// s <= 30 is one signed IMAD.WIDE, s >= 32 only touches the high word.
__device__ __forceinline__ int64_t mad_pow2(int a, int s, int64_t add) {
  if (s <= 30) return (int64_t)a * (int64_t)(1 << s) + add;
  if (s >= 32) return (int64_t)((uint64_t)(uint32_t)(a << (s - 32)) << 32) + add;
  return (int64_t)((uint64_t)(int64_t)a << 31) + add;
}

// stencil S_d applied to 4 consecutive points at storage offset o (mantissa units)
template <typename M, typename A, bool NC>
__device__ __forceinline__ void stencil4(const Vec& x, int64_t sx, int dim, int l, int64_t o,
                                         A g[4], int64_t c[4]) {
  V4<M, NC>::load(x, o, sx, c);
  int64_t lf = ld1<M, NC>(x, o - 1, sx), rt = ld1<M, NC>(x, o + 4, sx);
  A nb[4];
  nb[0] = (A)lf + (A)c[1];
  nb[1] = (A)c[0] + (A)c[2];
  nb[2] = (A)c[1] + (A)c[3];
  nb[3] = (A)c[2] + (A)rt;
  if (dim >= 2) {
    const int64_t N = (int64_t)1 << l;
    int64_t u[4], d[4];
    V4<M, NC>::load(x, o - N, sx, u);
    V4<M, NC>::load(x, o + N, sx, d);
#pragma unroll
    for (int j = 0; j < 4; ++j) nb[j] += (A)u[j] + (A)d[j];
    if (dim >= 3) {
      const int64_t N2 = N * N;
      V4<M, NC>::load(x, o - N2, sx, u);
      V4<M, NC>::load(x, o + N2, sx, d);
#pragma unroll
      for (int j = 0; j < 4; ++j) nb[j] += (A)u[j] + (A)d[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) g[j] = (A)(2 * dim) * (A)c[j] - nb[j];
}

// 2-D 9-point stencil (8, -1 x 8) on 4 consecutive points at storage offset o: the
// reference's bilinear-FEM operator A1(x)M1 + M1(x)A1 after the D = I scaling
// (centre 1, eight neighbours -1/8; P/src/fem.cpp:426-457, P/src/multigrid.cpp:277-306)
template <typename M, typename A, bool NC>
__device__ __forceinline__ void stencil9_4(const Vec& x, int64_t sx, int l, int64_t o, A g[4],
                                           int64_t c[4]) {
  const int64_t N = (int64_t)1 << l;
  V4<M, NC>::load(x, o, sx, c);
  A nb[4];
  const int64_t lf = ld1<M, NC>(x, o - 1, sx), rt = ld1<M, NC>(x, o + 4, sx);
  nb[0] = (A)lf + (A)c[1];
  nb[1] = (A)c[0] + (A)c[2];
  nb[2] = (A)c[1] + (A)c[3];
  nb[3] = (A)c[2] + (A)rt;
#pragma unroll
  for (int r = -1; r <= 1; r += 2) {  // the rows above and below: 3 taps each
    const int64_t ro = o + r * N;
    int64_t v[4];
    if (l >= 2) {
      V4<M, NC>::load(x, ro, sx, v);
    } else {  // level 1 (N = 2): the neighbouring rows are not 16-B aligned
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = ld1<M, NC>(x, ro + j, sx);
    }
    const int64_t vl = ld1<M, NC>(x, ro - 1, sx), vr = ld1<M, NC>(x, ro + 4, sx);
    nb[0] += (A)vl + (A)v[0] + (A)v[1];
    nb[1] += (A)v[0] + (A)v[1] + (A)v[2];
    nb[2] += (A)v[1] + (A)v[2] + (A)v[3];
    nb[3] += (A)v[2] + (A)v[3] + (A)vr;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) g[j] = (A)8 * (A)c[j] - nb[j];
}

// split-window parameters (see bulk3_loop / grid_loop in bfp_kernels.cuh)
struct SplitWin {
  uint64_t m0, m1;  // 2^ad, and 2^(ad-rs) or 1
  int s1, s2;       // rs, 0  or  ad, rs - ad
  int a0, a1;       // the multipliers' exponents: ad, and ad - rs or 0
};
template <typename T, typename = void> struct HasSplit {
  static constexpr bool value = false;
};
template <typename T> struct HasSplit<T, decltype((void)T::split_tag)> {
  static constexpr bool value = true;
};


// ops with a split window in the 3-D pipeline (bulk3_loop SP): b3_split_ok / b3_split_setup /
// point_sp
template <typename T, typename = void> struct HasB3Split {
  static constexpr bool value = false;
};
template <typename T> struct HasB3Split<T, decltype((void)T::b3split_tag)> {
  static constexpr bool value = true;
};

__device__ __forceinline__ SplitWin split_win(int64_t d, int rs) {
  const int ad = (int)(d < 0 ? -d : d);
  SplitWin sw;
  sw.m0 = 1ull << ad;
  sw.a0 = ad;
  if (ad >= rs)
    sw.a1 = ad - rs, sw.s1 = rs, sw.s2 = 0;
  else
    sw.a1 = 0, sw.s1 = ad, sw.s2 = rs - ad;
  sw.m1 = 1ull << sw.a1;
  return sw;
}

// ---------------------------------------------------------------------------
// z = alpha*(A_l x) + beta*y  (EgemvKernel with A = 2^{2l} S_d)

struct GemvOp {
  Vec x, y;
  Scal al, be;
  int dim, l, z0;  // z0: slab offset along the slowest axis (0 for full grids)
  // operator representation: e_A (2l for the config stencil) and a mantissa scale 2^gs
  // (reference-algorithm mode: a quantize_csr'd operator has mantissas 2^gs (2d, -1),
  // e_A = its quantized exponent -- values equal, templates as in the reference)
  int ea, gs;
  int st9;  // 2-D 9-point operator (reference mode, d = 2) instead of the 5-point S_2
  // derived (uniform per launch)
  int64_t sx, sy, d, zd;
  bool narrow;  // 32-bit stencil and products, 64-bit combine: exact by the width bound
  bool w64;     // 64-bit stencil and products, A-wide shift / sum (int64 storage)
  bool fwi;     // ... and the alignment shift < 64: two-word rows (W128)
  bool swap;
  bool sp32;  // 32-bit operand products, alignment < 64: split window (eval4_sp)
  int P, Q, PX, QY;
  static constexpr int zd_tag = 0;
  __device__ void setup(int64_t& e_star, int64_t& need) {
    const HSnap hx = hsnap(x.hdr), hy = hsnap(y.hdr);
    const int64_t ge = ea + hx.e;  // e_A + e_x
    int64_t dd, es, z = 0;
    axpby_setup_z(al.e + ge, be.e + hy.e, al.m == 0 || hx.bits == 0, be.m == 0 || hy.bits == 0,
                  dd, es, z);
    e_star = es;
    const int64_t ssx = hx.shift, ssy = hy.shift;
    const int64_t bg = grow(hx.bits, ceil_log2_h(st9 ? 16 : 4 * dim) + 1 + gs), by = hy.bits;
    const int64_t nd = combine_bits(al.m, bg, be.m, by, dd);
    need = nd;
    // z = X * P + Q * Y with (X, Y) = (g, y), P = alpha 2^d, Q = beta   when d >= 0
    //                         (X, Y) = (y, g), P = beta 2^-d, Q = alpha  when d < 0
    const int64_t ad = dd >= 0 ? dd : -dd;
    const int64_t pm = dd >= 0 ? al.m : be.m, qm = dd >= 0 ? be.m : al.m;
    const int64_t bx_ = dd >= 0 ? bg : by, by_ = dd >= 0 ? by : bg;
    const int mp = msb(pm), mq = msb(qm);
    // 32-bit operands: stencil, y and the Q product in 32 bits
    const bool ops32 = !gs && !st9 && ssx < 32 && ssy < 32 && bg <= 31 && by <= 31 &&
                       fits32(pm) && fits32(qm) && (by_ == 0 || mq + by_ <= 32);
    const bool nar = ops32 && l >= 2 && nd <= 63 && ad <= 30 && mp + ad <= 32 &&
                     (bx_ == 0 || mp + ad + bx_ <= 63);
    const bool x32 = ops32 && (bx_ == 0 || mp + bx_ <= 32);  // ... and the P product
    // beyond the narrow path (1-D: h^-2 = 2^{2l} puts A x ~40 bits above b at config 1):
    // the split window of the grid kernel
    const bool sp = x32 && ad <= 63;
    const bool w6 = !gs && !st9 && bg <= 62 && ssx < 64 && ssy < 64 && msb(al.m) + bg <= 63 &&
                    msb(be.m) + by <= 63;
    d = dd;
    zd = z;
    sx = ssx;
    sy = ssy;
    narrow = nar;
    sp32 = sp;
    w64 = w6;
    fwi = w6 && nd <= 127 && ad < 64;
    swap = dd < 0;
    P = nar ? (int)(pm << ad) : 0;
    Q = (int)qm;
    PX = sp ? (int)pm : 0;
    QY = sp ? (int)qm : 0;
  }
  // march-kernel interface (narrow, int32 storage)
  __host__ __device__ __forceinline__ const Vec& sv() const { return x; }
  __host__ __device__ __forceinline__ const Vec& yv2() const { return y; }
  __device__ __forceinline__ int shs() const { return (int)sx; }
  __device__ __forceinline__ int shy() const { return (int)sy; }
  __device__ __forceinline__ int64_t point(int g, int c, int yv) const {
    (void)c;
    const int X = swap ? yv : g, Y = swap ? g : yv;
    return (int64_t)X * (int64_t)P + (int64_t)(Q * Y);
  }
  __device__ __forceinline__ bool swapped() const { return swap; }
  template <bool SW> __device__ __forceinline__ int64_t point_t(int g, int c, int yv) const {
    (void)c;
    return SW ? (int64_t)yv * (int64_t)P + (int64_t)(Q * g)
              : (int64_t)g * (int64_t)P + (int64_t)(Q * yv);
  }
  // generic exact point (int64 storage): alpha g 2^max(d,0) + beta y 2^max(-d,0)
  template <typename A> __device__ __forceinline__ A point_w(int64_t g, int64_t c, int64_t yv) const {
    (void)c;
    return combine_w<A>(al.m, g, be.m, yv, d);
  }
  // two-word rows; SW = (d < 0) is uniform per launch (fw_swap) and templated
  __device__ __forceinline__ bool fw_swap() const { return d < 0; }
  template <bool SW>
  __device__ __forceinline__ W128 point_fw(int64_t g, int64_t c, int64_t yv) const {
    (void)c;
    const int64_t a = al.m * g, b = be.m * yv;
    return SW ? w_add(w_shl(b, (int)-d), a) : w_add(w_shl(a, (int)d), b);
  }
  // split window (int64 storage, qcomp pass 1 / recompute): the stored value
  // t = floor(z / 2^rs) and the low word zl = z mod 2^64 in 64-bit arithmetic only
  // (SplitWin, bfp_kernels.cuh); z = X 2^|d| + Y with (X, Y) = (alpha g, beta y) or,
  // SW (d < 0), (beta y, alpha g)
  static constexpr int split_tag = 0;
  static constexpr int b3split_tag = 0;
  __device__ __forceinline__ bool b3_split_ok(int64_t need, int rs) const { return need - rs <= 63; }
  __device__ __forceinline__ SplitWin b3_split_setup(int rs) const { return split_win(d, rs); }
  template <bool SW>
  __device__ __forceinline__ void point_sp(int64_t g, int64_t cx, int64_t yv, const SplitWin& w,
                                           int64_t& t, int64_t& zl) const {
    (void)cx;
    const int64_t a = al.m * g, b = be.m * yv;  // exact: w64 bounds |a|, |b| < 2^62
    const int64_t X = SW ? b : a, Y = SW ? a : b;
    zl = (int64_t)((uint64_t)X * w.m0 + (uint64_t)Y);
    t = (int64_t)((uint64_t)X * w.m1 + (uint64_t)(Y >> w.s1)) >> w.s2;
  }
  // split window over int32 storage (grid_loop SP): t = floor(z / 2^rs) and zl = z mod 2^64
  // from 32-bit operand products X = PX * (g | y), Y = QY * (y | g), z = X 2^ad + Y
  template <bool NC>
  __device__ __forceinline__ void eval4_sp(int64_t o, const SplitWin& w, int64_t t[4],
                                           int64_t zl[4]) const {
    int g[4], c[4], yv[4];
    stencil4_32<NC>(x, (int)sx, dim, l, o, g, c);
    V4<int32_t, NC>::load32(y, o, (int)sy, yv);
    const uint32_t mN = (1u << l) - 1;
    const bool xpad = ((uint32_t)o & mN) == mN - 3;
    const bool rowpad = plane_pad(dim, l, z0, o);
    const int s1 = w.s1 > 31 ? 31 : w.s1;  // floor(Y / 2^s1) of a 32-bit Y
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int X = (swap ? yv[j] : g[j]) * PX, Y = (swap ? g[j] : yv[j]) * QY;
      const int64_t xs = (int64_t)X;
      zl[j] = (int64_t)(((uint64_t)xs << w.a0) + (uint64_t)(int64_t)Y);
      t[j] = (int64_t)(((uint64_t)xs << w.a1) + (uint64_t)(int64_t)(Y >> s1)) >> w.s2;
    }
    if (xpad) t[3] = zl[3] = 0;
    if (rowpad) t[0] = t[1] = t[2] = t[3] = zl[0] = zl[1] = zl[2] = zl[3] = 0;
  }
  template <typename M, typename A, bool NC = true>
  __device__ __forceinline__ void eval4(int64_t o, A z[4]) {
    if constexpr (sizeof(M) == 4 && sizeof(A) == 8) {
      if (narrow) {
        int g[4], c[4], yv[4];
        stencil4_32<NC>(x, (int)sx, dim, l, o, g, c);
        V4<int32_t, NC>::load32(y, o, (int)sy, yv);
        const uint32_t mN = (1u << l) - 1;
        const uint32_t ix = (uint32_t)o & mN;
        const bool rowpad = plane_pad(dim, l, z0, o);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int X = swap ? yv[j] : g[j], Y = swap ? g[j] : yv[j];
          z[j] = (int64_t)X * (int64_t)P + (int64_t)(Q * Y);
        }
        if (ix == mN - 3) z[3] = 0;  // x pad (only the last lane of a 4-group)
        if (rowpad) z[0] = z[1] = z[2] = z[3] = 0;
        return;
      }
    }
    A g[4];
    int64_t c[4], yv[4];
    if (st9)
      stencil9_4<M, A, NC>(x, sx, l, o, g, c);
    else
      stencil4<M, A, NC>(x, sx, dim, l, o, g, c);
    V4<M, NC>::load(y, o, sy, yv);
    bool pad[4];
    pad4(dim, l, o, pad, z0);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      z[j] = pad[j] ? A(0) : combine<A>(al.m, g[j] << gs, be.m, (A)yv[j], d);
  }
};

// z = x + c*(b - A_l x): egemv(A,x,b,-1,+1) composed with eaxpby(x,r,+1,c)
struct JacobiOp {
  Vec x, b;
  Scal c;
  int dim, l, z0;
  int64_t sx, sb, d1, d2;
  bool narrow;
  bool w64;   // 64-bit stencil and r-term products (int64 storage)
  bool fwi;   // ... and every alignment shift < 64: two-word rows (W128)
  bool neg1;  // d1 < 0: the b term carries the power of two
  int Pg, Pb, s2;
  int64_t zd;
  static constexpr int zd_tag = 0;
#ifndef BFP_B3_DJ
#define BFP_B3_DJ 3
#endif
#ifndef BFP_B3_MINBJ
#define BFP_B3_MINBJ 4
#endif
#ifndef BFP_B3_D64J
#define BFP_B3_D64J 3
#endif
  static constexpr int b3_depth = BFP_B3_DJ, b3_minb = BFP_B3_MINBJ;  // bulk3 tuning (int32; B3Tune)
  static constexpr int b3_depth64 = BFP_B3_D64J;                       // (int64 storage)
  __device__ void setup(int64_t& e_star, int64_t& need) {
    const HSnap hx = hsnap(x.hdr), hb = hsnap(b.hdr);
    const int64_t ge = 2 * l + hx.e;
    const bool zx = hx.bits == 0, zb = hb.bits == 0;
    // reference template chain (e* only; the rows are those of the chain below * 2^zd)
    const int64_t es_ref = imin(hx.e, c.e + imin(ge, hb.e));
    int64_t er, zr = 0, dd1, dd2, es;  // zr: unused (zd is taken against the reference chain)
    axpby_setup_z(ge, hb.e, zx, zb, dd1, er, zr);  // r template (alpha q=1 e=0, beta q=2 e=0)
    axpby_setup_z(hx.e, c.e + er, zx, c.m == 0 || (zx && zb), dd2, es, zr);
    e_star = es;
    const int64_t ssx = hx.shift, ssb = hb.shift;
    const int64_t bx = hx.bits, bbb = hb.bits;
    const int64_t bg = grow(bx, ceil_log2_h(4 * dim) + 1);
    const int64_t br = combine_bits(-1, bg, 1, bbb, dd1);
    const int64_t nd = combine_bits(1, bx, c.m, br, dd2);
    need = nd;
    // r = -g 2^d1 + b (d1 >= 0) or b 2^-d1 - g (d1 < 0): one IMAD.WIDE either way;
    // z = x 2^d2 + c r (d2 >= 0)
    const bool nar = l >= 2 && bg <= 31 && bbb <= 31 && c.m >= 0 && c.m <= 0x7fffffff &&
                     nd <= 63 && ssx < 32 && ssb < 32 && dd1 >= -30 && dd1 <= 30 && dd2 >= 0 &&
                     dd2 <= 62 && dd2 != 31 && bx <= 31 && (bx == 0 || bx + dd2 <= 63);
    const bool w6 = bg <= 62 && bbb <= 62 && ssx < 64 && ssb < 64;
    d1 = dd1;
    d2 = dd2;
    zd = es - es_ref;
    sx = ssx;
    sb = ssb;
    narrow = nar;
    w64 = w6;
    fwi = w6 && nd <= 127 && dd1 > -64 && dd1 < 64 && dd2 >= 0 && dd2 < 64 && c.m >= 0 &&
          c.m <= 0xffffffffll && bx <= 62;
    // split window (point_sp): three 32-bit limbs
    sp96 = fwi && c.m <= 0x7fffffffll && dd1 >= -31 && dd1 <= 31 && nd <= 96;
    a1 = (int)(dd1 < 0 ? -dd1 : dd1);
    neg1 = dd1 < 0;
    Pg = nar ? (neg1 ? -1 : -(1 << (int)dd1)) : 0;
    Pb = nar ? (neg1 ? (1 << (int)(-dd1)) : 1) : 0;
    s2 = nar ? (int)dd2 : 0;
  }
  __host__ __device__ __forceinline__ const Vec& sv() const { return x; }
  __host__ __device__ __forceinline__ const Vec& yv2() const { return b; }
  __device__ __forceinline__ int shs() const { return (int)sx; }
  __device__ __forceinline__ int shy() const { return (int)sb; }
  // r = b 2^max(-d1,0) - g 2^max(d1,0) as two IMAD.WIDEs (no per-point selects on the sign
  // of d1): (Pg, Pb) = (-2^d1, 1) or (-1, 2^-d1)
  __device__ __forceinline__ int64_t rterm(int g, int bv) const {
    return mad_wide(g, Pg, mul_wide(bv, Pb));
  }
  __device__ __forceinline__ int64_t point(int g, int cx, int bv) const {
    const int64_t r = rterm(g, bv);
    const int64_t cr = (int64_t)((uint64_t)r * (uint64_t)c.m);
    return mad_pow2(cx, s2, cr);
  }
  // the "swap" template slot selects the shift class of x 2^d2: d2 <= 30 (one IMAD.WIDE)
  // or d2 >= 32 (high word only); d2 == 31 is not narrow
  __device__ __forceinline__ bool swapped() const { return s2 >= 32; }
  template <bool HI> __device__ __forceinline__ int64_t point_t(int g, int cx, int bv) const {
    const int64_t r = rterm(g, bv);
    const int64_t cr = (int64_t)((uint64_t)r * (uint64_t)(uint32_t)c.m);  // exact by the bound
    if (HI) return (int64_t)((uint64_t)(uint32_t)(cx << (s2 - 32)) << 32) + cr;
    return (int64_t)cx * (int64_t)(1 << s2) + cr;
  }
  template <typename A> __device__ __forceinline__ A point_w(int64_t g, int64_t cx, int64_t bv) const {
    return combine<A>(1, (A)cx, c.m, combine_w<A>(-1, g, 1, bv, d1), d2);
  }
  __device__ __forceinline__ bool fw_swap() const { return d1 < 0; }
  template <bool SW>
  __device__ __forceinline__ W128 point_fw(int64_t g, int64_t cx, int64_t bv) const {
    const W128 r = SW ? w_add(w_shl(bv, (int)-d1), -g) : w_add(w_shl(-g, (int)d1), bv);
    return w_add(w_shl(cx, (int)d2), w_mul_u32(r, (uint32_t)c.m));
  }
  // Split window of the int64 Jacobi row (3-D pipeline): z = x 2^d2 + c b 2^a - c g 2^a'
  // (one of a, a' is |d1| <= 31, the other 0) in three 32-bit limbs.  c v for a 64-bit v is
  // two IMAD.WIDEs (c v_lo, then c v_hi plus the carry word), the |d1| alignment three funnel
  // shifts, the sums two carry chains; the stored value is the 64-bit field of z at the
  // window shift rs < 64 and the low word z mod 2^64 serves mu* exactly as in the
  // residual's split window (bulk3_loop).  Exact when z fits 96 bits (need <= 96 bounds
  // every partial sum: the r term's bound is part of need) and 0 <= c < 2^31.
  bool sp96;
  int a1;
  static constexpr int b3split_tag = 0;
  __device__ __forceinline__ bool b3_split_ok(int64_t need, int rs) const {
    return sp96 && need - rs <= 63;
  }
  __device__ __forceinline__ SplitWin b3_split_setup(int rs) const {
    SplitWin w{};
    w.a0 = d2 >= 32;                               // x 2^d2 starts at limb 1
    w.s1 = (int)(d2 >= 32 ? d2 - 32 : 32 - d2);
    w.a1 = rs >= 32;                               // the stored field starts at limb 1
    w.s2 = rs & 31;
    w.m0 = (uint64_t)c.m;
    return w;
  }
  static __device__ __forceinline__ void mul96(uint32_t cm, int64_t v, uint32_t& p0, uint32_t& p1,
                                               uint32_t& p2) {
    uint64_t lo;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(lo) : "r"(cm), "r"((uint32_t)v));
    const int64_t hi = mad_wide((int)cm, (int)(v >> 32), (int64_t)(lo >> 32));
    p0 = (uint32_t)lo, p1 = (uint32_t)hi, p2 = (uint32_t)((uint64_t)hi >> 32);
  }
  template <bool SW>
  __device__ __forceinline__ void point_sp(int64_t g, int64_t cx, int64_t bv, const SplitWin& w,
                                           int64_t& t, int64_t& zl) const {
    const uint32_t cm = (uint32_t)w.m0;
    uint32_t q0, q1, q2, b0, b1, b2;
    mul96(cm, g, q0, q1, q2);
    mul96(cm, bv, b0, b1, b2);
    if (SW) {  // d1 < 0: the b term carries 2^|d1|
      b2 = __funnelshift_l(b1, b2, a1), b1 = __funnelshift_l(b0, b1, a1), b0 <<= a1;
    } else {
      q2 = __funnelshift_l(q1, q2, a1), q1 = __funnelshift_l(q0, q1, a1), q0 <<= a1;
    }
    uint32_t x0, x1, x2;
    if (w.a0) {
      const uint64_t xs = (uint64_t)cx << w.s1;
      x0 = 0, x1 = (uint32_t)xs, x2 = (uint32_t)(xs >> 32);
    } else {
      const int64_t xs = cx >> w.s1;  // s1 = 32 - d2 in [1, 32]
      x0 = (uint32_t)cx << ((32 - w.s1) & 31), x1 = (uint32_t)xs, x2 = (uint32_t)((uint64_t)xs >> 32);
    }
    uint32_t z0, z1, z2;
    asm("sub.cc.u32 %0, %3, %6;\n\tsubc.cc.u32 %1, %4, %7;\n\tsubc.u32 %2, %5, %8;"
        : "=r"(z0), "=r"(z1), "=r"(z2)
        : "r"(b0), "r"(b1), "r"(b2), "r"(q0), "r"(q1), "r"(q2));
    asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
        : "+r"(z0), "+r"(z1), "+r"(z2)
        : "r"(x0), "r"(x1), "r"(x2));
    zl = (int64_t)(((uint64_t)z1 << 32) | z0);
    uint32_t tl, th;
    if (w.a1) {
      tl = __funnelshift_r(z1, z2, w.s2), th = (uint32_t)((int)z2 >> w.s2);
    } else {
      tl = __funnelshift_r(z0, z1, w.s2), th = __funnelshift_r(z1, z2, w.s2);
    }
    t = (int64_t)(((uint64_t)th << 32) | tl);
  }
  template <typename M, typename A, bool NC = true>
  __device__ __forceinline__ void eval4(int64_t o, A z[4]) {
    if constexpr (sizeof(M) == 4 && sizeof(A) == 8) {
      if (narrow) {
        int g[4], cx[4], bv[4];
        stencil4_32<NC>(x, (int)sx, dim, l, o, g, cx);
        V4<int32_t, NC>::load32(b, o, (int)sb, bv);
        const uint32_t mN = (1u << l) - 1;
        const uint32_t ix = (uint32_t)o & mN;
        const bool rowpad = plane_pad(dim, l, z0, o);
        const uint64_t cm = (uint64_t)c.m;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t r = rterm(g[j], bv[j]);
          const int64_t cr = (int64_t)((uint64_t)r * cm);  // exact: |c r| < 2^63 by the bound
          z[j] = mad_pow2(cx[j], s2, cr);
        }
        if (ix == mN - 3) z[3] = 0;
        if (rowpad) z[0] = z[1] = z[2] = z[3] = 0;
        return;
      }
    }
    A g[4];
    int64_t cx[4], bv[4];
    stencil4<M, A, NC>(x, sx, dim, l, o, g, cx);
    V4<M, NC>::load(b, o, sb, bv);
    bool pad[4];
    pad4(dim, l, o, pad, z0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      A r = combine<A>(-1, g[j], 1, (A)bv[j], d1);
      z[j] = pad[j] ? A(0) : combine<A>(1, (A)cx[j], c.m, r, d2);
    }
  }
};

// z = c*r (pointwise over the storage span; pads stay zero)
// Pointwise ops with a 32-bit fast loop (grid_loop_pt, bfp_kernels.cuh): int32 storage,
// coefficients in int32, rows in 64 bits -- point4() gives 4 exact rows from narrow loads.
template <typename T, typename = void> struct HasPoint {
  static constexpr bool value = false;
};
template <typename T> struct HasPoint<T, decltype((void)T::point_tag)> {
  static constexpr bool value = true;
};

struct ScalOp {
  Vec r;
  Scal c;
  int64_t sr;
  bool p32;  // c.m in int32, pending shift < 32: the 32-bit pointwise loop applies
  static constexpr int point_tag = 0;
  __device__ void setup(int64_t& e_star, int64_t& need) {
    e_star = c.e + r.hdr->e;
    sr = r.hdr->shift;
    need = msb((int64_t)c.m) + eff_bits(r.hdr) + 1;
    p32 = fits32(c.m) && sr < 32;
  }
  static constexpr int kPointUnroll = 4;
  struct Raw {
    int4 v;
  };
  __device__ __forceinline__ Raw point_load(int64_t o) const {
    return Raw{__ldg(reinterpret_cast<const int4*>((const int32_t*)r.data + o))};
  }
  __device__ __forceinline__ void point4(const Raw& w, int64_t z[4]) const {
    const int s = (int)sr, m = (int)c.m;
    z[0] = mul_wide(m, w.v.x >> s);
    z[1] = mul_wide(m, w.v.y >> s);
    z[2] = mul_wide(m, w.v.z >> s);
    z[3] = mul_wide(m, w.v.w >> s);
  }
  template <typename M, typename A, bool NC = true>
  __device__ __forceinline__ void eval4(int64_t o, A z[4]) {
    int64_t v[4];
    V4<M, NC>::load(r, o, sr, v);
#pragma unroll
    for (int j = 0; j < 4; ++j) z[j] = (A)c.m * (A)v[j];
  }
};

// z = alpha*x*2^max(d,0) + beta*y*2^max(-d,0)  (EaxpbyKernel, pointwise)
struct AxpbyOp {
  Vec x, y;
  Scal al, be;
  int64_t sx, sy, d, zd;
  bool p32;    // the 32-bit pointwise loop applies: z = x Pa + y Pb with int32 Pa = alpha 2^d+,
  int da, db;  // Pb = beta 2^d- (here named da, db)
  static constexpr int zd_tag = 0;
  static constexpr int point_tag = 0;
  __device__ void setup(int64_t& e_star, int64_t& need) {
    const HSnap hx = hsnap(x.hdr), hy = hsnap(y.hdr);
    int64_t dd, es, z = 0;
    axpby_setup_z(al.e + hx.e, be.e + hy.e, al.m == 0 || hx.bits == 0, be.m == 0 || hy.bits == 0,
                  dd, es, z);
    e_star = es;
    need = combine_bits(al.m, hx.bits, be.m, hy.bits, dd);
    d = dd;
    zd = z;
    sx = hx.shift;
    sy = hy.shift;
    // the alignment folded into the coefficients: z = x Pa + y Pb, two IMAD.WIDE
    const int64_t sa = dd > 0 ? dd : 0, sb = dd < 0 ? -dd : 0;
    p32 = sx < 32 && sy < 32 && sa <= 30 && sb <= 30 && fits32(al.m) && fits32(be.m) &&
          fits32(al.m << sa) && fits32(be.m << sb);
    da = p32 ? (int)(al.m << sa) : 0;  // Pa
    db = p32 ? (int)(be.m << sb) : 0;  // Pb
  }
  static constexpr int kPointUnroll = 2;
  struct Raw {
    int4 a, b;
  };
  __device__ __forceinline__ Raw point_load(int64_t o) const {
    return Raw{__ldg(reinterpret_cast<const int4*>((const int32_t*)x.data + o)),
               __ldg(reinterpret_cast<const int4*>((const int32_t*)y.data + o))};
  }
  __device__ __forceinline__ void point4(const Raw& w, int64_t z[4]) const {
    const int s0 = (int)sx, s1 = (int)sy;
    const int xa[4] = {w.a.x >> s0, w.a.y >> s0, w.a.z >> s0, w.a.w >> s0};
    const int yb[4] = {w.b.x >> s1, w.b.y >> s1, w.b.z >> s1, w.b.w >> s1};
#pragma unroll
    for (int j = 0; j < 4; ++j) z[j] = mad_wide(xa[j], da, mul_wide(yb[j], db));
  }
  template <typename M, typename A, bool NC = true>
  __device__ __forceinline__ void eval4(int64_t o, A z[4]) {
    int64_t xv[4], yv[4];
    V4<M, NC>::load(x, o, sx, xv);
    V4<M, NC>::load(y, o, sy, yv);
#pragma unroll
    for (int j = 0; j < 4; ++j) z[j] = combine<A>(al.m, (A)xv[j], be.m, (A)yv[j], d);
  }
};

// coarse z = R r, full weighting R = (1,2,1)^{(x)d} 2^{-2d}  (EspmvKernel)

struct RestrictOp {
  Vec r;       // fine, level l
  int dim, l;  // fine level
  int zc;      // slab: global index of the output's local plane 0 (coarse)
  int er, gs;  // e_R (-2 dim: full weighting) and mantissa scale 2^gs (reference mode)
  int64_t sr;
  bool narrow;  // int32 storage, |R r| < 2^31: vectorised 32-bit path
  __device__ void setup(int64_t& e_star, int64_t& need) {
    e_star = er + r.hdr->e;
    sr = r.hdr->shift;
    need = eff_bits(r.hdr) + 2 * dim + 2 + gs;
    narrow = need <= 31 && sr < 32 && dim >= 2 && gs == 0;
  }
  // fine line weights (1,2,1) for 4 consecutive coarse points from fine row base f
  template <bool NC>
  __device__ __forceinline__ void line4(const int32_t* f, int sh, int w[4]) const {
    const int4 a = ldx<NC>(reinterpret_cast<const int4*>(f));
    const int4 b = ldx<NC>(reinterpret_cast<const int4*>(f + 4));
    const int e = ldx<NC>(f + 8) >> sh;
    const int v0 = a.x >> sh, v1 = a.y >> sh, v2 = a.z >> sh, v3 = a.w >> sh;
    const int v4 = b.x >> sh, v5 = b.y >> sh, v6 = b.z >> sh, v7 = b.w >> sh;
    w[0] = v0 + 2 * v1 + v2;
    w[1] = v2 + 2 * v3 + v4;
    w[2] = v4 + 2 * v5 + v6;
    w[3] = v6 + 2 * v7 + e;
  }
  template <typename M, typename A, bool NC = true>
  __device__ __forceinline__ void eval4(int64_t o, A z[4]) {
    const int lc = l - 1;
    const int64_t Nc = (int64_t)1 << lc, mc = Nc - 1, Nf = (int64_t)1 << l;
    bool pad[4];
    pad4(dim, lc, o, pad, zc);  // slabs: fine z0 = 2 zc, so local fine = 2 local coarse (+1)
    const int64_t J = (o >> lc) & mc, K = (o >> (2 * lc)) & mc;
    if constexpr (sizeof(M) == 4 && sizeof(A) == 8) {
      if (narrow) {
        // fine columns 2I0 .. 2I0+8 of fine rows 2J..2J+2 (and planes 2K..2K+2 in 3-D)
        const int64_t I0 = o & mc;
        int64_t base = 2 * I0 + 2 * J * Nf;
        if (dim >= 3) base += 2 * K * Nf * Nf;
        const int32_t* f = (const int32_t*)r.data + base;
        const int sh = (int)sr;
        int acc[4] = {0, 0, 0, 0}, w[4];
        const int planes = dim >= 3 ? 3 : 1;
        for (int pz = 0; pz < planes; ++pz) {
          const int wz = dim >= 3 ? (pz == 1 ? 2 : 1) : 1;
          const int32_t* fp = f + (dim >= 3 ? pz * Nf * Nf : 0);
#pragma unroll
          for (int py = 0; py < 3; ++py) {
            line4<NC>(fp + py * Nf, sh, w);
            const int wy = (py == 1 ? 2 : 1) * wz;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] += wy * w[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) z[j] = pad[j] ? 0 : (int64_t)acc[j];
        return;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t I = (o + j) & mc;
      int64_t fc = 2 * I + 1;
      if (dim >= 2) fc += (2 * J + 1) * Nf;
      if (dim >= 3) fc += (2 * K + 1) * Nf * Nf;
      A acc = 0;
      if (!pad[j]) {
        // x-line weights (1,2,1) on each contributing fine row
        auto line = [&](int64_t base) -> A {
          return (A)ld1<M, NC>(r, base - 1, sr) + 2 * (A)ld1<M, NC>(r, base, sr) +
                 (A)ld1<M, NC>(r, base + 1, sr);
        };
        if (dim == 1) {
          acc = line(fc);
        } else if (dim == 2) {
          acc = line(fc - Nf) + 2 * line(fc) + line(fc + Nf);
        } else {
          const int64_t N2 = Nf * Nf;
          A pm = line(fc - N2 - Nf) + 2 * line(fc - N2) + line(fc - N2 + Nf);
          A p0 = line(fc - Nf) + 2 * line(fc) + line(fc + Nf);
          A pp = line(fc + N2 - Nf) + 2 * line(fc + N2) + line(fc + N2 + Nf);
          acc = pm + 2 * p0 + pp;
        }
      }
      z[j] = acc << gs;
    }
  }
};

// linear interpolation: per axis taps (i-1)>>1 and i>>1 with weight 1 each
// (odd i -> both taps = (i-1)/2, i.e. weight 2).  Coarse pads/halo are zero.
// zp = z0(fine) - 2 z0(coarse) shifts the slowest axis when the fine output is a slab
// (0 for slabs aligned with a coarse slab, z0 of the fine slab for a full coarse grid)
template <typename M, typename A, bool NC = true>
__device__ __forceinline__ A prolong_at(const Vec& xc, int64_t sc, int dim, int l, int64_t o,
                                        int zp = 0) {
  const int64_t Nf = (int64_t)1 << l, mf = Nf - 1;
  const int lc = l - 1;
  const int64_t Nc = (int64_t)1 << lc;
  const int64_t i = o & mf;
  const int64_t a0 = (i - 1) >> 1, a1 = i >> 1;
  if (dim == 1) return (A)ld1<M, NC>(xc, a0, sc) + (A)ld1<M, NC>(xc, a1, sc);
  const int64_t j = dim == 2 ? (o >> l) + zp : (o >> l) & mf;
  const int64_t b0 = ((j - 1) >> 1) * Nc, b1 = (j >> 1) * Nc;
  auto line = [&](int64_t rowoff) -> A {
    return (A)ld1<M, NC>(xc, rowoff + a0, sc) + (A)ld1<M, NC>(xc, rowoff + a1, sc);
  };
  if (dim == 2) return line(b0) + line(b1);
  const int64_t k = (o >> (2 * l)) + zp;
  const int64_t Nc2 = Nc * Nc;
  const int64_t c0 = ((k - 1) >> 1) * Nc2, c1 = (k >> 1) * Nc2;
  return line(c0 + b0) + line(c0 + b1) + line(c1 + b0) + line(c1 + b1);
}

// coarse taps of 4 consecutive fine points along x (i0 even): c[I0-1], c[I0], c[I0+1]
template <bool NC>
__device__ __forceinline__ void prolong_xline(const int32_t* c, int sh, int t[4]) {
  const int a = ldx<NC>(c - 1) >> sh, b = ldx<NC>(c) >> sh, e = ldx<NC>(c + 1) >> sh;
  t[0] = a + b;
  t[1] = 2 * b;
  t[2] = b + e;
  t[3] = 2 * e;
}
// g = P xc at 4 consecutive fine points (int32 storage, |g| < 2^31 by the width bound)
template <bool NC>
__device__ __forceinline__ void prolong4_32(const Vec& xc, int sh, int dim, int l, int zp,
                                            int64_t o, int g[4]) {
  const int64_t Nf = (int64_t)1 << l, mf = Nf - 1, Nc = Nf >> 1;
  const int64_t i0 = o & mf;
  const int32_t* cb = (const int32_t*)xc.data + (i0 >> 1);
  int t[4];
  g[0] = g[1] = g[2] = g[3] = 0;
  if (dim == 1) {
    prolong_xline<NC>(cb, sh, g);
    return;
  }
  const int64_t j = dim == 2 ? (o >> l) + zp : (o >> l) & mf;
  const int64_t r0 = ((j - 1) >> 1) * Nc, r1 = (j >> 1) * Nc;
  int64_t p0 = 0, p1 = 0;
  if (dim >= 3) {
    const int64_t k = (o >> (2 * l)) + zp;
    p0 = ((k - 1) >> 1) * Nc * Nc;
    p1 = (k >> 1) * Nc * Nc;
  }
  const int np = dim >= 3 ? 2 : 1;
  for (int pz = 0; pz < np; ++pz) {
    const int64_t pb = pz ? p1 : p0;
    prolong_xline<NC>(cb + pb + r0, sh, t);
#pragma unroll
    for (int q = 0; q < 4; ++q) g[q] += t[q];
    prolong_xline<NC>(cb + pb + r1, sh, t);
#pragma unroll
    for (int q = 0; q < 4; ++q) g[q] += t[q];
  }
}


// fine z = P xc  (EspmvKernel with P, m_P = 2^d, e_P = -d, q_P = d+2)
struct ProlongOp {
  Vec xc;
  int dim, l;  // fine level
  int zf, zp;  // slab: fine z0 and the slowest-axis shift of prolong_at
  int ep, gs;  // e_P (-dim) and mantissa scale 2^gs (reference mode)
  int64_t sc;
  bool narrow;  // int32 storage and |P xc| < 2^31: vectorised coarse rows
  static constexpr bool kCorr = false;
  __host__ __device__ __forceinline__ const Vec& cv() const { return xc; }
  __host__ __device__ __forceinline__ const Vec& yv() const { return xc; }  // unused
  __device__ __forceinline__ int shc() const { return (int)sc; }
  __device__ __forceinline__ int shy() const { return 0; }
  bool wide;    // int64 storage and |P xc| < 2^63: the 3-D march in 64 bits
  __device__ __forceinline__ int64_t corr(int g, int yv) const { (void)yv; return g; }
  __device__ __forceinline__ int64_t corr_w(int64_t g, int64_t yv) const { (void)yv; return g; }
  __device__ void setup(int64_t& e_star, int64_t& need) {
    e_star = ep + xc.hdr->e;
    sc = xc.hdr->shift;
    need = eff_bits(xc.hdr) + dim + 2 + gs;
    narrow = need <= 31 && sc < 32 && gs == 0;
    wide = need <= 63 && sc < 64 && gs == 0;
  }
  template <typename M, typename A, bool NC = true>
  __device__ __forceinline__ void eval4(int64_t o, A z[4]) {
    bool pad[4];
    pad4(dim, l, o, pad, zf);
    if constexpr (sizeof(M) == 4 && sizeof(A) == 8) {
      if (narrow) {
        int g[4];
        prolong4_32<NC>(xc, (int)sc, dim, l, zp, o, g);
#pragma unroll
        for (int q = 0; q < 4; ++q) z[q] = pad[q] ? 0 : (int64_t)g[q];
        return;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      z[j] = pad[j] ? A(0) : prolong_at<M, A, NC>(xc, sc, dim, l, o + j, zp) << gs;
  }
};

// fine z = P ec + y  (EgemvKernel(P, ec, y, bfp_one, bfp_one))
struct ProlongCorrectOp {
  Vec ec, y;
  int dim, l;
  int zf, zp;  // slab: fine z0 and the slowest-axis shift of prolong_at
  int ep, gs;  // e_P (-dim) and mantissa scale 2^gs (reference mode)
  Scal al, be;  // z = al P ec + be y (config: +1, +1; reference V-correct: -1, +1)
  int64_t sc, sy, d;
  bool narrow, swap;  // int32 storage: g = P ec in 32 bits, z = X 2^|d| + Y (one IMAD.WIDE)
  int P;
  static constexpr bool kCorr = true;
  __host__ __device__ __forceinline__ const Vec& cv() const { return ec; }
  __host__ __device__ __forceinline__ const Vec& yv() const { return y; }
  __device__ __forceinline__ int shc() const { return (int)sc; }
  __device__ __forceinline__ int shy() const { return (int)sy; }
  __device__ __forceinline__ int64_t corr(int g, int yy) const {
    const int X = swap ? yy : g, Y = swap ? g : yy;
    return (int64_t)X * (int64_t)P + (int64_t)Y;
  }
  // int64 storage (wide): z = X 2^|d| + Y in 64 bits, exact by need <= 63
  bool wide;
  int AD;
  __device__ __forceinline__ int64_t corr_w(int64_t g, int64_t yy) const {
    const int64_t X = swap ? yy : g, Y = swap ? g : yy;
    return (int64_t)((uint64_t)X << AD) + Y;
  }
  int64_t zd;
  static constexpr int zd_tag = 0;
  __device__ void setup(int64_t& e_star, int64_t& need) {
    const HSnap hc = hsnap(ec.hdr), hy = hsnap(y.hdr);
    const int64_t ge = ep + hc.e;
    int64_t dd, es, z = 0;
    axpby_setup_z(al.e + ge, be.e + hy.e, al.m == 0 || hc.bits == 0, be.m == 0 || hy.bits == 0,
                  dd, es, z);
    e_star = es;
    const int64_t bg = grow(hc.bits, dim + 2 + gs), by = hy.bits;
    const int64_t nd = combine_bits(al.m, bg, be.m, by, dd);
    need = nd;
    const int64_t ad = dd >= 0 ? dd : -dd;
    const bool nar = nd <= 63 && bg <= 31 && by <= 31 && ad <= 30 && hc.shift < 32 &&
                     hy.shift < 32 && gs == 0 && al.m == 1 && be.m == 1;
    d = dd;
    zd = z;
    sc = hc.shift;
    sy = hy.shift;
    narrow = nar;
    wide = nd <= 63 && ad < 64 && hc.shift < 64 && hy.shift < 64 && gs == 0 && al.m == 1 &&
           be.m == 1;
    AD = wide ? (int)ad : 0;
    swap = dd < 0;
    P = nar ? (1 << (int)ad) : 0;
  }
  template <typename M, typename A, bool NC = true>
  __device__ __forceinline__ void eval4(int64_t o, A z[4]) {
    bool pad[4];
    pad4(dim, l, o, pad, zf);
    if constexpr (sizeof(M) == 4 && sizeof(A) == 8) {
      if (narrow) {
        int g[4];
        prolong4_32<NC>(ec, (int)sc, dim, l, zp, o, g);
        int yv[4];
        V4<int32_t, NC>::load32(y, o, (int)sy, yv);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int X = swap ? yv[q] : g[q], Y = swap ? g[q] : yv[q];
          z[q] = pad[q] ? 0 : (int64_t)X * (int64_t)P + (int64_t)Y;
        }
        return;
      }
    }
    int64_t yv[4];
    V4<M, NC>::load(y, o, sy, yv);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      A g = prolong_at<M, A, NC>(ec, sc, dim, l, o + j, zp) << gs;
      z[j] = pad[j] ? A(0) : combine<A>(al.m, g, be.m, (A)yv[j], d);
    }
  }
};

// ---------------------------------------------------------------------------
// flat (one row per thread, int128 accumulation) ops for the generic CSR path

struct CsrDev {
  int64_t rows, cols, q, e, max_row_nnz;
  const int64_t *rowptr, *col, *m;
};

// z = A x  (EspmvKernel, src/blas.cpp:74-94)
struct CsrSpmvOp {
  CsrDev a;
  Vec x;
  int64_t m_a;
  int64_t sx;
  __device__ void setup(int64_t& e_star, int64_t& need) {
    e_star = a.e + x.hdr->e;
    sx = x.hdr->shift;
    need = a.q + eff_bits(x.hdr) + ceil_log2_h(imax(m_a, 1)) + 1;
  }
  template <typename M> __device__ __forceinline__ i128 eval1(int64_t i) {
    i128 acc = 0;
    for (int64_t k = a.rowptr[i]; k < a.rowptr[i + 1]; ++k)
      acc += (i128)a.m[k] * (i128)ld1<M>(x, a.col[k], sx);
    return acc;
  }
};

// z = alpha A x + beta y  (EgemvKernel, src/blas.cpp:96-142)
struct CsrGemvOp {
  CsrDev a;
  Vec x, y;
  Scal al, be;
  int64_t m_a;
  int64_t sx, sy, d, zd;
  static constexpr int zd_tag = 0;
  __device__ void setup(int64_t& e_star, int64_t& need) {
    const int64_t ge = a.e + x.hdr->e;
    zd = 0;
    axpby_setup_z(al.e + ge, be.e + y.hdr->e, al.m == 0 || hdr_zero(x.hdr),
                  be.m == 0 || hdr_zero(y.hdr), d, e_star, zd);
    sx = x.hdr->shift;
    sy = y.hdr->shift;
    int64_t bg = grow(zbits(x.hdr), a.q + ceil_log2_h(imax(m_a, 1)) + 1);
    need = combine_bits(al.m, bg, be.m, zbits(y.hdr), d);
  }
  template <typename M> __device__ __forceinline__ i128 eval1(int64_t i) {
    i128 g = 0;
    for (int64_t k = a.rowptr[i]; k < a.rowptr[i + 1]; ++k)
      g += (i128)a.m[k] * (i128)ld1<M>(x, a.col[k], sx);
    return combine<i128>(al.m, g, be.m, (i128)ld1<M>(y, i, sy), d);
  }
};

// explicit exact rows (the test FixedKernel, tests/test_blas.cpp:14-26)
struct RowsOp {
  const int64_t* hi;
  const uint64_t* lo;
  int64_t e;
  __device__ void setup(int64_t& e_star, int64_t& need) {
    e_star = e;
    need = 0;
  }
  template <typename M> __device__ __forceinline__ i128 eval1(int64_t i) {
    return (i128)(((u128)(uint64_t)hi[i] << 64) | (u128)lo[i]);
  }
};

}  // namespace bfpdev
