// bfp_dev.cuh -- device-side BFP primitives, block headers and the qcomp /
// nnqcomp window epilogue shared by every sm_100a kernel of the hot path.
//
// Reference semantics restated here (paths relative to /root/reference/proj):
//   msb                    src/wideint.cpp:15-25
//   shift_floor / wrap     src/wideint.cpp:94-107
//   clamp (saturation)     src/blas.cpp:196-209
//   qcomp window           src/blas.cpp:144-187
//   nnqcomp window         src/blas.cpp:189-212
// Every vector carries a DEVICE-resident header (exponent, width, pending
// shift, max/min mantissa) so exponents and norms never force a host round
// trip: a whole V-cycle is stream-ordered and graph-capturable.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bfpdev {

typedef __int128 i128;
typedef unsigned __int128 u128;

// ---------------------------------------------------------------------------
// device header of a BFP block (one per vector, 128-byte aligned)
struct alignas(128) Hdr {
  // published state of the block
  int64_t q;        // declared width w_out
  int64_t e;        // block exponent
  int64_t shift;    // pending arithmetic right shift applied on every load (deferred qcomp)
  int64_t max_m;    // max of STORED mantissas (pads included: >= 0)
  int64_t min_m;    // min of STORED mantissas (<= 0)
  int32_t flags;    // BFP_FLAG_*
  int32_t err;      // sticky BFP_ERR_*
  // qcomp staging, written by pass-1 finalize, read by the recompute pass
  int64_t lam_out;
  int32_t need_recompute;
  int32_t st_zd;  // pass-1 elision shift of the window context (WinCtx::zd), with st_*
  // cross-block accumulators (reset by each finalize)
  unsigned long long acc_or_lo, acc_or_hi;  // OR over rows of z ^ sign(z): bitlen = max msb - 1
  long long acc_max, acc_min;
  unsigned int acc_done;
  int32_t acc_err;
  // partial (multi-rank) windows: the pass-1 window context, for the finalize kernel
  int64_t st_estar, st_mutmp, st_lam, st_gm, st_ge;
};

enum { FLAG_OVERFLOW = 1, FLAG_UNDERFLOW = 2, FLAG_RECOMPUTED = 4, FLAG_NORMALIZED = 8 };
enum { ERR_WIDTH = 2, ERR_STORAGE = 7 };

// device view of a vector passed to kernels by value
struct Vec {
  void* data;      // element 0 (after the front halo for grids)
  Hdr* hdr;
  int32_t ebytes;  // 4 or 8
  int32_t dim;     // 0 = flat, 1..3 = grid
  int32_t l;       // grid level (N = 2^l)
  int32_t z0;      // slab: global index of local plane 0 along the slowest axis
  int64_t n;       // storage span in elements (flat: padded to 4; grid: nz * N^(dim-1))
  int64_t nlog;    // logical entries
  int32_t nz;      // planes along the slowest axis held locally (N for a full grid)
  int32_t pad;
};

// trace record (bfp_trace_rec_t layout)
struct TraceRec {
  int32_t step, level, w_out, w_tmp;
  int64_t gm, ge;
  int32_t overflow, underflow, recomputed, normalized;
};

// ---------------------------------------------------------------------------
// programmatic dependent launch (sm_90+): wait for the previous grid's results /
// let the next grid be scheduled
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// integer primitives

// 32 x 32 -> 64-bit signed multiply(-add): one IMAD.WIDE on the FMA pipe (the compiler
// otherwise widens a product with a launch-uniform factor to a 64 x 64 multiply)
__device__ __forceinline__ int64_t mul_wide(int a, int b) {
  int64_t r;
  asm("mul.wide.s32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ int64_t mad_wide(int a, int b, int64_t c) {
  int64_t r;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}

__device__ __forceinline__ int bitlen64(uint64_t u) { return u ? 64 - __clzll((long long)u) : 0; }
__device__ __forceinline__ int bitlen128(u128 u) {
  uint64_t hi = (uint64_t)(u >> 64);
  return hi ? 128 - __clzll((long long)hi) : bitlen64((uint64_t)u);
}
// msb: minimal two's complement width (msb(0) = msb(-1) = 1)
__device__ __forceinline__ int msb(int64_t v) { return bitlen64((uint64_t)(v ^ (v >> 63))) + 1; }
__device__ __forceinline__ int msb(i128 v) { return bitlen128((u128)(v ^ (v >> 127))) + 1; }
__host__ __device__ __forceinline__ int msb_h(int64_t v) {
  uint64_t u = (uint64_t)(v ^ (v >> 63));
#ifdef __CUDA_ARCH__
  return (u ? 64 - __clzll((long long)u) : 0) + 1;
#else
  return (u ? 64 - __builtin_clzll(u) : 0) + 1;
#endif
}

template <typename A> struct AccBits;
template <> struct AccBits<int64_t> { static constexpr int value = 64; };
template <> struct AccBits<i128> { static constexpr int value = 128; };

// floor(x / 2^s) for s >= 0
template <typename A> __device__ __forceinline__ A sar(A x, int64_t s) {
  constexpr int B = AccBits<A>::value;
  return s >= B - 1 ? (x < 0 ? A(-1) : A(0)) : (x >> s);
}
// wrap_w(floor(x / 2^s)), w <= 64, s of either sign (low bits only, no overflow)
template <typename A> __device__ __forceinline__ int64_t wrap_shift(A x, int64_t s, int64_t w) {
  uint64_t lo;
  if (s >= 0) {
    lo = (uint64_t)sar<A>(x, s);
  } else {
    int64_t k = -s;
    if (k >= w) return 0;
    lo = ((uint64_t)x) << k;
  }
  int sh = 64 - (int)w;
  return (int64_t)(lo << sh) >> sh;
}
// floor(x / 2^s) clamped to T_w (nnqcomp, w <= 64): saturates when a left shift leaves T_w
template <typename A> __device__ __forceinline__ int64_t shift_clamp(A x, int64_t s, int64_t w) {
  // T_w bounds without a 64-bit shift by 64 (w = 1: [-1, 0]; w = 64: the int64 range)
  const int64_t hi = w >= 64 ? INT64_MAX : (int64_t)((1ull << (w - 1)) - 1), lo = -hi - 1;
  A r;
  if (s >= 0) {
    r = sar<A>(x, s);
  } else {
    int64_t k = -s;
    if (x == 0) return 0;
    if (msb(x) + k > w) return x < 0 ? lo : hi;
    r = x << k;
  }
  return r > (A)hi ? hi : (r < (A)lo ? lo : (int64_t)r);
}
// exact floor(x / 2^s) where the result is known to fit 64 bits (recompute pass)
template <typename A> __device__ __forceinline__ int64_t shift_exact(A x, int64_t s) {
  if (s >= 0) return (int64_t)sar<A>(x, s);
  return (int64_t)(x << (-s));
}

// ---------------------------------------------------------------------------
// stored mantissa load/store with pending shift

template <typename M> __device__ __forceinline__ int64_t ldm(const Vec& v, int64_t i, int64_t sh) {
  return ((int64_t)((const M*)v.data)[i]) >> sh;
}

// eff width of a block: smallest w with every (stored >> shift) in T_w
__device__ __forceinline__ int eff_bits(const Hdr* h) {
  int64_t s = h->shift;
  int64_t a = h->max_m >> s, b = h->min_m >> s;
  int ma = msb(a), mb = msb(b);
  return ma > mb ? ma : mb;
}
__device__ __forceinline__ uint64_t max_abs(const Hdr* h) {
  int64_t s = h->shift;
  int64_t a = h->max_m >> s, b = h->min_m >> s;
  uint64_t ua = a < 0 ? (uint64_t)0 - (uint64_t)a : (uint64_t)a;
  uint64_t ub = b < 0 ? (uint64_t)0 - (uint64_t)b : (uint64_t)b;
  return ua > ub ? ua : ub;
}

// ---------------------------------------------------------------------------
// gamma arithmetic: 15-bit round-up values

struct G15 {
  int64_t m, e;
};
__host__ __device__ __forceinline__ int bitlen_h(uint64_t u) {
#ifdef __CUDA_ARCH__
  return u ? 64 - __clzll((long long)u) : 0;
#else
  return u ? 64 - __builtin_clzll(u) : 0;
#endif
}
__host__ __device__ inline G15 g15_from(uint64_t mag, int64_t e) {
  G15 r = {0, 0};
  if (mag == 0) return r;
  int b = bitlen_h(mag);
  if (b <= 15) {
    r.m = (int64_t)(mag << (15 - b));
    r.e = e - (15 - b);
  } else {
    int s = b - 15;
    uint64_t m = (mag >> s) + ((mag & ((1ull << s) - 1)) != 0);
    if (m == (1ull << 15)) {
      m >>= 1;
      ++s;
    }
    r.m = (int64_t)m;
    r.e = e + s;
  }
  return r;
}
__host__ __device__ inline G15 g15_mul(G15 a, G15 b) {
  if (a.m == 0 || b.m == 0) return G15{0, 0};
  return g15_from((uint64_t)a.m * (uint64_t)b.m, a.e + b.e);
}
__host__ __device__ inline G15 g15_add(G15 a, G15 b) {
  if (a.m == 0) return b;
  if (b.m == 0) return a;
  if (a.e < b.e) {
    G15 t = a;
    a = b;
    b = t;
  }
  int64_t gap = a.e - b.e;
  if (gap <= 100) {
    u128 s = ((u128)(uint64_t)a.m << gap) + (u128)(uint64_t)b.m;
    int bl = 0;
    {
      uint64_t hi = (uint64_t)(s >> 64);
      bl = hi ? 64 + bitlen_h(hi) : bitlen_h((uint64_t)s);
    }
    if (bl <= 64) return g15_from((uint64_t)s, b.e);
    int sh = bl - 64;
    uint64_t top = (uint64_t)(s >> sh) | (uint64_t)((s & ((((u128)1) << sh) - 1)) != 0);
    return g15_from(top, b.e + sh);
  }
  G15 r = a;
  r.m += 1;
  if (r.m == (1 << 15)) {
    r.m = 1 << 14;
    r.e += 1;
  }
  return r;
}

// gamma rule: add_up chain over up to 3 terms c_t (x) X_t
struct GTerm {
  const Hdr* v;    // nullptr: X = 1
  int64_t cm, ce;  // cm == 0: no coefficient
  int32_t kind;    // 0 = norm(v), 1 = ulp(v) (zero if v is all zero)
  int32_t sticky;  // exact rules: the coefficient has nonzero bits below cm_hi:cm
  uint64_t cm_hi;  // exact rules: 128-bit coefficient (cm_hi:cm as unsigned)
};
struct GammaRule {
  int32_t literal;  // 1: (lm, le) as given
  int32_t nterms;
  int64_t lm, le;
  GTerm t[3];
  int32_t exact;  // 1: sum_t c_t X_t evaluated exactly, one round-up at the end
  int32_t pad;
};

__device__ inline G15 gterm_eval(const GTerm& t) {
  G15 x;
  if (t.v == nullptr) {
    x = G15{1 << 14, -14};
  } else if (t.kind == 0) {
    x = g15_from(max_abs(t.v), t.v->e);
  } else {
    x = max_abs(t.v) ? g15_from(1, t.v->e) : G15{0, 0};
  }
  if (t.cm != 0) x = g15_mul(g15_from((uint64_t)t.cm, t.ce), x);
  return x;
}
// Exact gamma rules (reference-algorithm mode, gamma_policy_eval P/src/multigrid.cpp:
// 121-155): the reference's ExtFloat chain rounds up at >= 64 / 400 bits and scalar_up
// then ceils to 15 significant bits; nested round-ups to a coarser grid equal one, so
// gamma = ceil_15(sum_t c_t X_t) of the exact value.  Terms are 128-bit coefficients
// (+ a sticky tail) times 64-bit block norms, accumulated in a 256-bit window.
struct X256 {
  uint64_t w[4];  // w[3] most significant; value = w * 2^e (+ tail if sticky)
  int64_t e;
  bool sticky;
};
__device__ inline int x256_bitlen(const X256& a) {
  for (int i = 3; i >= 0; --i)
    if (a.w[i]) return 64 * i + bitlen_h(a.w[i]);
  return 0;
}
// shift left by s (0 <= s < 256), bits never lost (caller guarantees headroom)
__device__ inline void x256_shl(X256& a, int s) {
  while (s >= 64) {
    a.w[3] = a.w[2]; a.w[2] = a.w[1]; a.w[1] = a.w[0]; a.w[0] = 0;
    s -= 64;
    a.e -= 64;
  }
  if (s) {
    for (int i = 3; i > 0; --i) a.w[i] = (a.w[i] << s) | (a.w[i - 1] >> (64 - s));
    a.w[0] <<= s;
    a.e -= s;
  }
}
// shift right by s, dropped bits go to sticky
__device__ inline void x256_shr(X256& a, int64_t s) {
  if (s >= 256) {
    a.sticky = a.sticky || a.w[0] || a.w[1] || a.w[2] || a.w[3];
    a.w[0] = a.w[1] = a.w[2] = a.w[3] = 0;
    a.e += s;
    return;
  }
  while (s >= 64) {
    a.sticky = a.sticky || a.w[0];
    a.w[0] = a.w[1]; a.w[1] = a.w[2]; a.w[2] = a.w[3]; a.w[3] = 0;
    s -= 64;
    a.e += 64;
  }
  if (s) {
    a.sticky = a.sticky || (a.w[0] << (64 - s));
    for (int i = 0; i < 3; ++i) a.w[i] = (a.w[i] >> s) | (a.w[i + 1] << (64 - s));
    a.w[3] >>= s;
    a.e += s;
  }
}
__device__ inline void x256_norm(X256& a) {  // top bit at position 254 (one bit of headroom)
  const int b = x256_bitlen(a);
  if (b == 0) return;
  if (b < 255) x256_shl(a, 255 - b);
  else if (b > 255) x256_shr(a, b - 255);
}
__device__ inline X256 x256_term(const GTerm& t) {
  X256 r = {{0, 0, 0, 0}, 0, false};
  uint64_t X;
  int64_t ex;
  if (t.v == nullptr) {
    X = 1;
    ex = 0;
  } else {
    X = max_abs(t.v);
    ex = t.v->e;
  }
  if (X == 0) return r;
  const uint64_t clo = (uint64_t)t.cm, chi = t.cm_hi;
  // (chi:clo) * X  -> 192 bits
  const u128 p0 = (u128)clo * X, p1 = (u128)chi * X;
  r.w[0] = (uint64_t)p0;
  const u128 mid = (p0 >> 64) + (uint64_t)p1;
  r.w[1] = (uint64_t)mid;
  r.w[2] = (uint64_t)(p1 >> 64) + (uint64_t)(mid >> 64);
  r.e = t.ce + ex;
  r.sticky = t.sticky != 0;
  return r;
}
__device__ inline void exact_gamma(const GammaRule& g, int64_t& gm, int64_t& ge) {
  X256 acc = {{0, 0, 0, 0}, 0, false};
  bool any = false;
  for (int i = 0; i < g.nterms; ++i) {
    X256 t = x256_term(g.t[i]);
    if (!x256_bitlen(t) && !t.sticky) continue;
    x256_norm(t);
    if (!any) {
      acc = t;
      any = true;
      continue;
    }
    // align to the larger exponent (both normalised at bit 254), add, renormalise
    if (acc.e < t.e) {
      X256 s = acc;
      acc = t;
      t = s;
    }
    x256_shr(t, acc.e - t.e);
    uint64_t carry = 0;
    for (int k = 0; k < 4; ++k) {
      const u128 s = (u128)acc.w[k] + t.w[k] + carry;
      acc.w[k] = (uint64_t)s;
      carry = (uint64_t)(s >> 64);
    }
    acc.sticky = acc.sticky || t.sticky;
    x256_norm(acc);
  }
  if (!any) {  // zero: degenerate gamma (scalar_up, :85-89)
    gm = 1 << 14;
    ge = -400 - 14;
    return;
  }
  // ceil to 15 significant bits: the top 15 of the 255-bit window
  const int sh = 255 - 15;
  uint64_t m = acc.w[3] >> (sh - 192);
  bool rest = acc.sticky || (acc.w[3] & ((1ull << (sh - 192)) - 1)) || acc.w[2] || acc.w[1] ||
              acc.w[0];
  int64_t e = acc.e + sh;
  if (rest) ++m;
  if (m == (1ull << 15)) {
    m >>= 1;
    ++e;
  }
  gm = (int64_t)m;
  ge = e;
}

// returns (gm, ge) of the BFP scalar gamma (q = 16); degenerate 2^-400 if zero
__device__ inline void gamma_eval(const GammaRule& r, int64_t& gm, int64_t& ge) {
  if (r.literal) {
    gm = r.lm;
    ge = r.le;
    return;
  }
  if (r.exact) {
    exact_gamma(r, gm, ge);
    return;
  }
  G15 acc{0, 0};
  for (int i = 0; i < r.nterms; ++i) acc = g15_add(acc, gterm_eval(r.t[i]));
  if (acc.m == 0) {
    gm = 1 << 14;
    ge = -400 - 14;
  } else {
    gm = acc.m;
    ge = acc.e;
  }
}

// ---------------------------------------------------------------------------
// window context (one per op launch; computed redundantly by every block)

enum { MODE_QCOMP = 0, MODE_NNQ = 1, MODE_RECOMPUTE = 2 };

struct WinParams {
  int64_t w_out, w_tmp;
  int32_t mode, force;
  int32_t trace_slot, step;
  int32_t level, hist_slot;
  TraceRec* trace;
  double* hist;   // residual-norm history slot (ldexp(max|m|, e)), or nullptr
  int64_t* part;  // multi-rank: write {mu*, max, -min, err} partials here instead of finalizing
  int32_t defer;  // multi-block pass 1: accumulate only, a deferred-finalize kernel follows
  int32_t pad_;
#ifdef BFP_TIMING
  long long* dbg;  // phase stamps of grid_win_kernel launches (measurement builds)
#endif
  GammaRule gamma;
};

struct WinCtx {
  int64_t e_star, mu_tmp, lam;  // lam: lam_tmp (qcomp), lam_out (nnq / recompute)
  int64_t gm, ge;
  int32_t store_tmp;            // qcomp: tmp fits the storage and is stored
  int32_t skip;                 // recompute pass with nothing to do
  int32_t rs, ls;               // stored value = (z >> rs) << ls  (lam >= 0: rs = lam)
  int64_t zd;                   // e* - e*_ref >= 0 when the op's template drops an all-zero
                                // term (op_zd): rows are z_ref / 2^zd, see win_finalize
};

// Ops whose eaxpby template drops an all-zero term carry `zd` (axpby_setup_z); the
// window runs in the shifted coordinates, which changes nothing but the all-zero result.
template <class T, class = void> struct HasZd {
  static constexpr bool value = false;
};
template <class T> struct HasZd<T, decltype((void)T::zd_tag)> {
  static constexpr bool value = true;
};
template <class Op> __device__ __forceinline__ int64_t op_zd(const Op& o) {
  if constexpr (HasZd<Op>::value)
    return o.zd;
  else
    return 0;
}

// per-thread running reductions.  mu* = max_i msb(z_i) is recovered exactly
// from the bitwise OR of z_i ^ sign(z_i): bitlen(a | b) = max(bitlen a, bitlen b).
struct Red {
  uint64_t olo, ohi;
  int64_t mx, mn;
  int err;
  __device__ void init() {
    olo = ohi = 0;
    mx = INT64_MIN;
    mn = INT64_MAX;
    err = 0;
  }
  __device__ void val(int64_t v) {
    mx = v > mx ? v : mx;
    mn = v < mn ? v : mn;
  }
};
template <typename A> __device__ __forceinline__ void or_mag(A z, uint64_t& lo, uint64_t& hi);
template <> __device__ __forceinline__ void or_mag<int64_t>(int64_t z, uint64_t& lo, uint64_t& hi) {
  lo |= (uint64_t)(z ^ (z >> 63));
}
template <> __device__ __forceinline__ void or_mag<i128>(i128 z, uint64_t& lo, uint64_t& hi) {
  u128 u = (u128)(z ^ (z >> 127));
  lo |= (uint64_t)u;
  hi |= (uint64_t)(u >> 64);
}

__device__ __forceinline__ int64_t shfl_max64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t > v ? t : v;
  }
  return v;
}
__device__ __forceinline__ int64_t shfl_min64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t < v ? t : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t shfl_or64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block reduction of the per-thread running values; the result is valid in thread 0.
struct BlockRed {
  uint64_t lo, hi;
  int err;
  int64_t mx, mn;
};
__device__ inline BlockRed block_reduce(const Red& r) {
  __shared__ unsigned long long s_lo[32], s_hi[32];
  __shared__ int s_err[32];
  __shared__ long long s_mx[32], s_mn[32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  BlockRed b;
  b.lo = shfl_or64(r.olo);
  b.hi = shfl_or64(r.ohi);
  b.err = __reduce_or_sync(0xffffffffu, r.err);
  b.mx = shfl_max64(r.mx);
  b.mn = shfl_min64(r.mn);
  if (lane == 0) {
    s_lo[wid] = b.lo;
    s_hi[wid] = b.hi;
    s_err[wid] = b.err;
    s_mx[wid] = b.mx;
    s_mn[wid] = b.mn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) {
      b.lo |= s_lo[w];
      b.hi |= s_hi[w];
      b.err |= s_err[w];
      b.mx = s_mx[w] > b.mx ? s_mx[w] : b.mx;
      b.mn = s_mn[w] < b.mn ? s_mn[w] : b.mn;
    }
  }
  return b;
}
__device__ __forceinline__ int mu_bits(uint64_t lo, uint64_t hi) {
  return (hi ? 64 + bitlen64(hi) : bitlen64(lo)) + 1;  // mu* (init 1, src/blas.cpp:153)
}
// one block's contribution to the header accumulators (fire-and-forget atomics)
__device__ __forceinline__ void accumulate(Hdr* h, const BlockRed& b) {
  if (b.lo) atomicOr(&h->acc_or_lo, (unsigned long long)b.lo);
  if (b.hi) atomicOr(&h->acc_or_hi, (unsigned long long)b.hi);
  atomicMax(&h->acc_max, (long long)b.mx);
  atomicMin(&h->acc_min, (long long)b.mn);
  if (b.err) atomicOr(&h->acc_err, b.err);
}

// Block reduce + cross-block atomics + last-block finalize.  `fin` is called
// by exactly one thread of the last block to finish, after every block's
// contribution is visible: fin(mu_star, max, min, err).
template <typename Fin>
__device__ inline void reduce_and_finalize(Red& r, Hdr* h, Fin fin) {
  __shared__ bool s_last;
  BlockRed b = block_reduce(r);
  if (gridDim.x == 1) {  // single block: finalize directly, no global accumulators
    if (threadIdx.x == 0) fin(mu_bits(b.lo, b.hi), b.mx, b.mn, b.err);
    return;
  }
  if (threadIdx.x == 0) {
    accumulate(h, b);
    __threadfence();
    unsigned int done = atomicAdd(&h->acc_done, 1u);
    s_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    volatile Hdr* vh = h;
    uint64_t flo = vh->acc_or_lo, fhi = vh->acc_or_hi;
    int64_t fmx = vh->acc_max, fmn = vh->acc_min;
    int ferr = vh->acc_err;
    // reset accumulators for the next op writing this block
    h->acc_or_lo = 0;
    h->acc_or_hi = 0;
    h->acc_max = INT64_MIN;
    h->acc_min = INT64_MAX;
    h->acc_err = 0;
    h->acc_done = 0;
    fin(mu_bits(flo, fhi), fmx, fmn, ferr);
  }
}

__device__ inline void write_trace(const WinParams& p, const WinCtx& c, int ovf, int unf, int rc,
                                   int normalized) {
  if (p.trace == nullptr || p.trace_slot < 0) return;
  TraceRec& t = p.trace[p.trace_slot];
  t.step = p.step;
  t.level = p.level;
  t.w_out = (int32_t)p.w_out;
  t.w_tmp = (int32_t)(normalized ? p.w_tmp : p.w_out);
  t.gm = c.gm;
  t.ge = c.ge;
  t.overflow = ovf;
  t.underflow = unf;
  t.recomputed = rc;
  t.normalized = normalized;
}

// window setup common to all ops: e* from the op's template, gamma from the rule
__device__ inline void win_setup(const WinParams& p, const Hdr* out_h, int64_t e_star,
                                 int storage_bits, WinCtx& c) {
  c.e_star = e_star;
  c.skip = 0;
  c.zd = 0;
  if (p.mode == MODE_RECOMPUTE) {
    const volatile Hdr* vh = out_h;  // may have been finalized earlier in this launch
    c.skip = !vh->need_recompute;
    c.lam = vh->lam_out;
    c.store_tmp = 1;
    c.rs = (int32_t)(c.lam >= 0 ? (c.lam > 127 ? 127 : c.lam) : 0);
    c.ls = (int32_t)(c.lam < 0 ? (-c.lam > 64 ? 64 : -c.lam) : 0);
    return;
  }
  gamma_eval(p.gamma, c.gm, c.ge);
  c.mu_tmp = msb(c.gm) + c.ge - e_star;
  if (p.mode == MODE_QCOMP) {
    c.lam = c.mu_tmp - p.w_tmp;          // lam_tmp
    c.store_tmp = p.w_tmp <= storage_bits && !p.force;
  } else {
    c.lam = c.mu_tmp - p.w_out;          // lam_out
    c.store_tmp = 1;
  }
  c.rs = (int32_t)(c.lam >= 0 ? (c.lam > 127 ? 127 : c.lam) : 0);
  c.ls = (int32_t)(c.lam < 0 ? (-c.lam > 64 ? 64 : -c.lam) : 0);
}

// stored value of an exact row: floor(z / 2^lam) truncated to the storage type.
// qcomp fast path: when no flag fires the w_tmp wrap of src/blas.cpp:160 is the
// identity, and when a flag fires the recompute pass overwrites the block, so
// the wrap is never needed; the recompute pass result always fits (T_w_out).
template <typename M, typename A>
__device__ __forceinline__ M store_shift(A z, const WinCtx& c) {
  constexpr int B = AccBits<A>::value;
  A r = c.rs >= B - 1 ? (z < 0 ? A(-1) : A(0)) : (z >> c.rs);
  if (c.ls == 0) return (M)r;
  // ls >= storage bits only happens when qcomp overflows (lam_tmp >= 1 - w_tmp on the
  // fast path), so these values are never the result: keep just their zero-ness, which
  // the all-zero test of win_finalize reads (mx, mn)
  if (c.ls >= 8 * (int)sizeof(M)) return (M)((r > 0) - (r < 0));
  return (M)((uint64_t)r << c.ls);
}

__device__ inline void write_hist(const WinParams& p, const Hdr* h) {
  if (p.hist == nullptr || p.hist_slot < 0) return;
  p.hist[p.hist_slot] = ldexp((double)max_abs(h), (int)h->e);
}

// multi-rank: record the launch's partial reduction and window context (one thread)
__device__ inline void win_partial(const WinParams& p, const WinCtx& c, Hdr* h, int bits,
                                   int64_t mx, int64_t mn, int err) {
  p.part[0] = bits;
  p.part[1] = mx;
  p.part[2] = mn == INT64_MIN ? INT64_MAX : -mn;
  p.part[3] = err;
  if (p.mode != MODE_RECOMPUTE) {
    h->st_estar = c.e_star;
    h->st_mutmp = c.mu_tmp;
    h->st_lam = c.lam;
    h->st_gm = c.gm;
    h->st_ge = c.ge;
    h->st_zd = (int32_t)c.zd;
  }
}

// finalize for one launch (runs on one thread); returns need_recompute
__device__ inline int win_finalize(const WinParams& p, const WinCtx& c, Hdr* h, int bits,
                                   int64_t mx, int64_t mn, int err) {
  if (p.part) {
    win_partial(p, c, h, bits, mx, mn, err);
    return 0;
  }
  int64_t mu_star = bits;                   // src/blas.cpp:153,158
  if (p.mode == MODE_QCOMP && c.zd > 0 && bits <= 1) {
    // mu* starts at 1 in the reference's coordinates, 1 - zd in the op's (an all-zero
    // result); rows in {0, -1} are told apart by their stored values (store_shift keeps
    // -1 nonzero)
    if (!c.store_tmp)
      err |= ERR_WIDTH;  // nothing stored (w_tmp beyond the storage, forced): fail loudly
    else if (mn >= 0 && mx <= 0)
      mu_star = 1 - c.zd;
  }
  if (err) h->err |= err;
  if (p.mode == MODE_QCOMP) {
    int64_t lam_out = mu_star - p.w_out;    // :164
    int ovf = c.mu_tmp < mu_star;           // :167
    int unf = lam_out < c.lam;              // :168
    int rc = ovf || unf || p.force || !c.store_tmp || err;
    h->q = p.w_out;
    h->e = c.e_star + lam_out;
    h->lam_out = lam_out;
    h->need_recompute = rc;
    if (!rc) {
      h->shift = lam_out - c.lam;           // deferred fast-path shift (:178-184)
      h->max_m = mx;
      h->min_m = mn;
      write_hist(p, h);
    }
    h->flags = (ovf ? FLAG_OVERFLOW : 0) | (unf ? FLAG_UNDERFLOW : 0) |
               (rc ? FLAG_RECOMPUTED : 0) | FLAG_NORMALIZED;
    write_trace(p, c, ovf, unf, rc, 1);
    return rc;
  } else if (p.mode == MODE_NNQ) {
    h->q = p.w_out;
    h->e = c.e_star + c.lam;                // src/blas.cpp:211
    h->shift = 0;
    h->max_m = mx;
    h->min_m = mn;
    h->need_recompute = 0;
    h->flags = 0;
    write_trace(p, c, 0, 0, 0, 0);
    write_hist(p, h);
  } else {
    h->shift = 0;
    h->max_m = mx;
    h->min_m = mn;
    h->need_recompute = 0;
    write_hist(p, h);
  }
  return 0;
}

// multi-rank finalize (one thread): apply the all-reduced partials {mu*, max, -min, err} with
// the window context recorded by pass 1 -- exactly the single-rank win_finalize
__device__ inline void finalize_from_partials(const Vec& out, WinParams p, const int64_t* part,
                                              int storage_bits) {
  Hdr* h = out.hdr;
  if (p.mode == MODE_RECOMPUTE && !h->need_recompute) return;  // fast path: nothing ran
  WinCtx c;
  c.e_star = h->st_estar;
  c.mu_tmp = h->st_mutmp;
  c.lam = p.mode == MODE_RECOMPUTE ? h->lam_out : h->st_lam;
  c.gm = h->st_gm;
  c.ge = h->st_ge;
  c.zd = h->st_zd;
  c.rs = 0;
  c.ls = c.lam < 0 ? (int32_t)(-c.lam > 64 ? 64 : -c.lam) : 0;
  c.store_tmp = p.mode == MODE_QCOMP ? (p.w_tmp <= storage_bits && !p.force) : 1;
  c.skip = 0;
  p.part = nullptr;
  win_finalize(p, c, h, (int)part[0], part[1], part[2] == INT64_MAX ? INT64_MIN : -part[2],
               (int)part[3]);
}

// Reduction + finalize of a windowed pass.  A multi-block pass 1 (qcomp or nnqcomp)
// launched with p.defer only accumulates: each block's partial goes to the header with
// fire-and-forget atomics and block 0 records the window context; the stream-ordered
// deferred-finalize kernel (one thread, bfp_lib.cu) then applies win_finalize from the
// accumulators.  The kernel boundary makes every contribution visible, so the
// threadfence / counter / last-block round trips of reduce_and_finalize (~2 us on a
// dependent chain) leave the critical path.
template <typename Fin>
__device__ inline void window_reduce(Red& r, Hdr* h, const WinParams& p, const WinCtx& c,
                                     Fin fin) {
  if (!p.defer || gridDim.x == 1 || p.mode == MODE_RECOMPUTE) {
    reduce_and_finalize(r, h, fin);
    return;
  }
  BlockRed b = block_reduce(r);
  if (threadIdx.x == 0) {
    accumulate(h, b);
    if (blockIdx.x == 0) {
      h->st_estar = c.e_star;
      h->st_mutmp = c.mu_tmp;
      h->st_lam = c.lam;
      h->st_gm = c.gm;
      h->st_ge = c.ge;
      h->st_zd = (int32_t)c.zd;
    }
  }
}

// deferred finalize of a multi-block pass 1 (window_reduce with p.defer; one thread): the
// blocks' accumulated {OR, max, min, err} and block 0's window context -> win_finalize, and
// the accumulators are reset for the next op writing this vector; returns need_recompute
__device__ inline int deferred_finalize(const Vec& out, WinParams p, int storage_bits) {
  Hdr* h = out.hdr;
  const volatile Hdr* vh = h;
  const uint64_t lo = vh->acc_or_lo, hi = vh->acc_or_hi;
  const int64_t mx = vh->acc_max, mn = vh->acc_min;
  const int err = vh->acc_err;
  WinCtx c;
  c.e_star = vh->st_estar;
  c.mu_tmp = vh->st_mutmp;
  c.lam = vh->st_lam;
  c.gm = vh->st_gm;
  c.ge = vh->st_ge;
  c.zd = vh->st_zd;
  c.store_tmp = p.mode == MODE_QCOMP ? (p.w_tmp <= storage_bits && !p.force) : 1;
  c.skip = 0;
  c.rs = 0;
  c.ls = c.lam < 0 ? (int32_t)(-c.lam > 64 ? 64 : -c.lam) : 0;
  h->acc_or_lo = 0;
  h->acc_or_hi = 0;
  h->acc_max = INT64_MIN;
  h->acc_min = INT64_MAX;
  h->acc_err = 0;
  p.defer = 0;
  return win_finalize(p, c, h, mu_bits(lo, hi), mx, mn, err);
}

}  // namespace bfpdev
