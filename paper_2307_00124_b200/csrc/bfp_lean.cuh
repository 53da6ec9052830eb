// bfp_lean.cuh -- the lean coarse engine (int32 storage): the op list of the bottom of a
// V-cycle / FMG (P/src/multigrid.cpp:430-518 on levels of a few thousand points) runs inside
// ONE launch with a per-op critical path of ~1 us, against 5-9 us for a kernel launch per op.
//
// The generic engine of bfp_coarse.cuh measured, per warm op, 4600 clk of one-thread setup,
// 1400 clk of finalize and 1900 clk of body, and three times that on instruction-cache
// misses (its per-op code path is ~1 MB of SASS).  What the lean engine changes:
//   * qcomp is value-determined (P/src/blas.cpp:144-187): the output is floor(z / 2^lam_out)
//     with lam_out = mu* - w_out whatever gamma is; gamma only decides the flags.  The exact
//     rows z wait in a private shared-memory slot per thread while mu* = max msb(z) is
//     reduced, then floor(z / 2^lam_out) is stored directly: no deferred shift, no recompute
//     pass.  A qcomp output is normalised, so its width is w_out unless it is all zero: the
//     next op's setup needs nothing else from it.
//   * everything that is not on the data path -- gamma, the flags, the trace record, the
//     history entry, max / min of the stored mantissas -- goes through a per-op LOG
//     (e_out, lam_out, mu*, max, min, producers of the gamma terms) and is evaluated for all
//     ops in parallel when the list ends (one thread per op), as are the final block headers.
//     nnqcomp (P/src/blas.cpp:189-212) needs gamma before the body: its control lane
//     evaluates the rule from the producers' log entries, and its rows are clamped in the
//     body, with max / min reduced there.
//   * warp 0 is the control warp: lane 0 runs core-finalize(i) -> setup(i + 1) in 32-bit
//     arithmetic from a compact per-vector state (exponent, pending shift, width) kept in
//     shared memory; warps 1..15 are the workers.  Three block barriers per op: (A) context
//     published / data visible, (B) partials, (C) lam_out.
//   * the fast path covers the config-mode ops on int32 storage whose rows fit 64 bits from
//     32-bit operands (the `narrow` conditions of bfp_ops.cuh, restated in 32 bits); anything
//     else -- wide rows, reference-mode operators, exact or literal gamma rules, exponents out
//     of range -- takes the generic path of bfp_coarse.cuh inside the same launch (cold
//     code), with the block headers it reads materialised from the log first.
//   * the host digests every record into a 64-byte LeanRec (static eligibility, vector ids,
//     coefficients, data pointers), so the control lane's setup has no per-kind record
//     parsing; it runs in two halves: PRE (record digest, operand states, gamma producers ->
//     registers) while the workers run the previous op's body, POST (alignment, widths,
//     window) after the previous op's core finalize, with that op's fresh output state
//     forwarded in registers.
//   * op records are prefetched three ops ahead through registers (loads issued during one
//     op, stored to shared memory during the next: no thread waits on the load) and their
//     arena pointers rebased on the way (FusedOp::rb marks the pointer words).
#pragma once
#include "bfp_coarse.cuh"

namespace bfpdev {

constexpr int kLeanWorkers = kFusedThreads - 32;

// dynamic window context of a fast op, published by the control lane (the static part is
// the record's LeanRec)
struct LeanDyn {
  int fast;
  int sx, sy;    // pending shifts of the operands
  int P, Q;      // gemv / pcorr: z = X P + Q Y; jacobi: P1 and s2
  int swap;      // gemv / pcorr: operands swapped (d < 0); jacobi: neg1
  int d;         // axpby: alignment
  int lam;       // nnqcomp window
  int needmm;    // reduce max / min in the body (nnqcomp, or qcomp before an nnqcomp op)
};

// compact state of a vector for the control lane's setups (16 bytes: one shared load)
struct alignas(16) FH {
  int e, s;    // exponent, pending shift
  int bits;    // width, 0: all zero
  int effok;   // eff_bits | ok << 8
};
__device__ __forceinline__ FH make_fh(int e, int s, int bits, int eff, bool ok) {
  return FH{e, s, bits, eff | ((int)ok << 8)};
}
// one record per op of the list (shared memory)
enum { LOG_NONE = 0, LOG_FASTQ, LOG_FASTN, LOG_GENERIC, LOG_ZERO };
struct alignas(16) LogRec {
  int e_out, lam, mu;  // block exponent, lam_out, mu*
  int mx, mn;          // max / min of the stored mantissas (pending shift applied)
  int gm, ge;          // nnqcomp: gamma
  int e_star;
  short prod[3];       // producer op of each gamma term's vector (-1: state at entry)
  short st;
  short q, flags;
  int pad;
};
static_assert(sizeof(LogRec) == 48, "LogRec layout (host sizes the log)");

struct LeanShared {
  LeanDyn dyn;
  int lam_store;  // lam_out of the op being stored
  unsigned long long orv[kCoarseWarps];
  long long mx[kCoarseWarps], mn[kCoarseWarps];
  FH fh[kLeanMaxVec];
  int lastw[kLeanMaxVec];       // last op of the list that wrote the vector (-1: none)
  int init_e[kLeanMaxVec];      // norms at entry
  unsigned init_mag[kLeanMaxVec];
};

// ---- 32-bit header snapshot and helpers --------------------------------------------
__device__ __forceinline__ int bitlen32(unsigned u) { return 32 - __clz((int)u); }
__device__ __forceinline__ int msb32(int v) { return bitlen32((unsigned)(v ^ (v >> 31))) + 1; }
struct LH {
  int e, s, bits, eff;  // bits: 0 for an all-zero block; eff: eff_bits (>= 1)
  unsigned mag;         // max |m| after the pending shift
  bool ok;              // exponent, shift and mantissas in the 32-bit fast range
};
__device__ __forceinline__ LH lean_hdr(const Hdr* h) {
  const int64_t e = h->e, s = h->shift, mx = h->max_m, mn = h->min_m;
  LH r;
  r.ok = e > -(1 << 20) && e < (1 << 20) && (uint64_t)s < 32 && mx == (int64_t)(int)mx &&
         mn == (int64_t)(int)mn;
  r.e = (int)e;
  r.s = (int)s & 31;
  const int a = (int)mx >> r.s, b = (int)mn >> r.s;
  const int ma = msb32(a), mb = msb32(b);
  r.eff = ma > mb ? ma : mb;
  r.bits = (a | b) ? r.eff : 0;
  const unsigned ua = a < 0 ? 0u - (unsigned)a : (unsigned)a;
  const unsigned ub = b < 0 ? 0u - (unsigned)b : (unsigned)b;
  r.mag = ua > ub ? ua : ub;
  return r;
}
__device__ __forceinline__ bool small_e(int64_t e) { return e > -(1 << 20) && e < (1 << 20); }
// axpby_setup_z (bfp_ops.cuh) in 32 bits
__device__ __forceinline__ void lean_align(int ea, int eb, bool za, bool zb, int& d, int& es,
                                           int& zd) {
  d = ea - eb;
  es = ea < eb ? ea : eb;
  zd = 0;
  if (za != zb) {
    const int ee = za ? eb : ea;
    zd = ee - es;
    es = ee;
    d = 0;
  }
}
// combine_bits (bfp_ops.cuh) in 32 bits
__device__ __forceinline__ int lean_cbits(int am, int ba, int bm, int bb, int d) {
  const int x = (ba && am) ? msb32(am) + ba + (d > 0 ? d : 0) : 0;
  const int y = (bb && bm) ? msb32(bm) + bb + (d < 0 ? -d : 0) : 0;
  const int m = x > y ? x : y;
  return (m > 1 ? m : 1) + 1;
}

// ---- 15-bit round-up gamma arithmetic in 32 bits (g15_* of bfp_dev.cuh) -------------
struct G32 {
  int m, e;
};
__device__ __forceinline__ G32 g32_from(unsigned mag, int e) {
  G32 r = {0, 0};
  if (mag == 0) return r;
  const int b = bitlen32(mag);
  if (b <= 15) {
    r.m = (int)(mag << (15 - b));
    r.e = e - (15 - b);
  } else {
    int s = b - 15;
    unsigned m = (mag >> s) + ((mag & ((1u << s) - 1)) != 0);
    if (m == (1u << 15)) {
      m >>= 1;
      ++s;
    }
    r.m = (int)m;
    r.e = e + s;
  }
  return r;
}
__device__ __forceinline__ G32 g32_mul(G32 a, G32 b) {
  if (a.m == 0 || b.m == 0) return G32{0, 0};
  return g32_from((unsigned)a.m * (unsigned)b.m, a.e + b.e);
}
__device__ __forceinline__ G32 g32_add(G32 a, G32 b) {
  if (a.m == 0) return b;
  if (b.m == 0) return a;
  if (a.e < b.e) {
    const G32 t = a;
    a = b;
    b = t;
  }
  const int gap = a.e - b.e;
  // gap >= 16: b < one ulp of a, the exact ceiling is a + 1 ulp (what g15_add computes)
  if (gap <= 15) return g32_from(((unsigned)a.m << gap) + (unsigned)b.m, b.e);
  G32 r = a;
  r.m += 1;
  if (r.m == (1 << 15)) {
    r.m = 1 << 14;
    r.e += 1;
  }
  return r;
}
// norm terms: (max |m|, e) of a vector as of op time, from its producer's log entry
struct NormSrc {
  unsigned mag;
  int e;
};
__device__ __forceinline__ NormSrc lean_norm(const LeanShared& ls, const LogRec* log, int vid,
                                             int prod) {
  if (prod < 0) return NormSrc{ls.init_mag[vid], ls.init_e[vid]};
  const LogRec& r = log[prod];
  const unsigned a = r.mx < 0 ? 0u - (unsigned)r.mx : (unsigned)r.mx;
  const unsigned b = r.mn < 0 ? 0u - (unsigned)r.mn : (unsigned)r.mn;
  return NormSrc{a > b ? a : b, r.e_out};
}
// gamma of a config-mode rule from the norms of its terms; the fast
// path only admits rules with 32-bit coefficients (LeanRec::ok)
__device__ __forceinline__ void lean_gamma(const GammaRule& g, const LeanRec& lr,
                                           const LeanShared& ls, const LogRec* log,
                                           const short* prod, int& gm, int& ge) {
  G32 acc{0, 0};
  for (int i = 0; i < g.nterms; ++i) {
    const GTerm& t = g.t[i];
    G32 x;
    if (lr.gv[i] == 0xff) {
      x = G32{1 << 14, -14};
    } else {
      const NormSrc ns = lean_norm(ls, log, lr.gv[i], prod[i]);
      x = t.kind == 0 ? g32_from(ns.mag, ns.e) : (ns.mag ? g32_from(1u, ns.e) : G32{0, 0});
    }
    if (t.cm != 0) x = g32_mul(g32_from((unsigned)t.cm, (int)t.ce), x);
    acc = g32_add(acc, x);
  }
  if (acc.m == 0) {  // degenerate gamma 2^-400 (P/src/multigrid.cpp:84-89)
    gm = 1 << 14;
    ge = -400 - 14;
  } else {
    gm = acc.m;
    ge = acc.e;
  }
}

__device__ __forceinline__ int clog2_4dim(int dim) { return dim == 1 ? 2 : (dim == 2 ? 3 : 4); }

// ---- the control lane's setup, first half: everything that does not depend on the op in
// flight (registers only; runs while the workers are in the previous op's body) ----------
struct LeanPre {
  int kind, ok, nnq, needmm, w_out;
  int vout, va, vb;
  int dim, l, ea, am, ae, bm, be;
  FH ha, hb;
  int gv[3], gok;
  short prod[3];
};
__device__ __forceinline__ void lean_pre(const FusedOp& f, const FusedOp* next,
                                         const LeanShared& ls, LeanPre& q) {
  const LeanRec lr = f.lr;
  q.kind = f.kind;
  q.ok = lr.ok;
  q.nnq = lr.nnq;
  // a qcomp op followed by an nnqcomp op reduces max / min in its body: the next setup
  // needs them (gamma, width) before this op's store phase has finished
  (void)next;
  q.needmm = lr.nnq || lr.nnq_next;
  q.w_out = lr.w_out;
  q.vout = lr.vout;
  q.va = lr.va;
  q.vb = lr.vb;
  q.dim = lr.dim;
  q.l = lr.l;
  q.ea = lr.ea;
  q.am = lr.am, q.ae = lr.ae, q.bm = lr.bm, q.be = lr.be;
  q.ha = lr.va != 0xff ? ls.fh[lr.va] : FH{0, 0, 0, 0x101};
  q.hb = lr.vb != 0xff ? ls.fh[lr.vb] : FH{0, 0, 0, 0x101};
  q.gok = 1;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    q.gv[i] = lr.gv[i];
    q.prod[i] = -1;
    if (lr.gv[i] != 0xff) {
      q.prod[i] = (short)ls.lastw[lr.gv[i]];
      q.gok &= ls.fh[lr.gv[i]].effok >> 8;
    }
  }
}

// the control lane's per-op state (registers)
struct LeanState {
  int e_star, zd;  // template exponent, zero-term elision shift
  int w_out, nnq;
  int gm, ge;      // nnqcomp: gamma
  int vout;        // vector id of the output
  short prod[3];
};

// ---- second half: alignment, width bounds and the `narrow` conditions of bfp_ops.cuh in
// 32-bit arithmetic, from the pre-loaded state with the previous op's output forwarded
// (fv: its vector id, ff: its fresh state, fi: its op index).  True: the op is fast. ------
__device__ __forceinline__ bool lean_post(const FusedOp& f, const LeanPre& qs, int fv,
                                          const FH& ff, int fi, LeanShared& ls,
                                          const LogRec* log, LeanState& st) {
  LeanPre q = qs;
  LeanDyn o;
  o.sx = o.sy = o.P = o.Q = o.swap = o.d = o.lam = 0;
  o.needmm = q.needmm;
  st.vout = q.vout;
  st.nnq = q.nnq;
  st.w_out = q.w_out;
  st.zd = 0;
  bool fast = q.ok;
  if (q.kind != FK_ZERO) {
    if (q.va == fv) q.ha = ff;
    if (q.vb == fv) q.hb = ff;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      st.prod[i] = q.prod[i];
      if (q.gv[i] == fv) {
        st.prod[i] = (short)fi;
        q.gok &= ff.effok >> 8;
      }
    }
    const FH hx = q.ha, hy = q.hb;
    const int effx = hx.effok & 0xff;
    fast = fast && q.gok && (hx.effok >> 8) && (hy.effok >> 8);
    switch (q.kind) {
      case FK_GEMV: {
        const int am = q.am, bm = q.bm;
        int dd, es, zd;
        lean_align(q.ae + q.ea + hx.e, q.be + hy.e, am == 0 || hx.bits == 0,
                   bm == 0 || hy.bits == 0, dd, es, zd);
        const int bg = hx.bits ? hx.bits + clog2_4dim(q.dim) + 1 : 0, by = hy.bits;
        const int nd = lean_cbits(am, bg, bm, by, dd);
        const int ad = dd >= 0 ? dd : -dd;
        const int pm = dd >= 0 ? am : bm, qm = dd >= 0 ? bm : am;
        const int bx_ = dd >= 0 ? bg : by, by_ = dd >= 0 ? by : bg;
        const int mp = msb32(pm), mq = msb32(qm);
        fast = fast && bg <= 31 && by <= 31 && (by_ == 0 || mq + by_ <= 32) && nd <= 63 &&
               ad <= 30 && mp + ad <= 32 && (bx_ == 0 || mp + ad + bx_ <= 63);
        st.e_star = es;
        st.zd = zd;
        o.P = pm << (ad & 31);
        o.Q = qm;
        o.swap = dd < 0;
        break;
      }
      case FK_JACOBI: {
        const int cm = q.am, ce = q.ae;
        const int ge = q.ea + hx.e;  // 2l + e_x
        const bool zx = hx.bits == 0, zb = hy.bits == 0;
        const int gb = ge < hy.e ? ge : hy.e;
        const int es_ref = hx.e < ce + gb ? hx.e : ce + gb;
        int dd1, er, zr, dd2, es;
        lean_align(ge, hy.e, zx, zb, dd1, er, zr);
        lean_align(hx.e, ce + er, zx, cm == 0 || (zx && zb), dd2, es, zr);
        const int bx = hx.bits, bbb = hy.bits;
        const int bg = bx ? bx + clog2_4dim(q.dim) + 1 : 0;
        const int br = lean_cbits(-1, bg, 1, bbb, dd1);
        const int nd = lean_cbits(1, bx, cm, br, dd2);
        fast = fast && bg <= 31 && bbb <= 31 && nd <= 63 && dd1 >= -30 && dd1 <= 30 && dd2 >= 0 &&
               dd2 <= 62 && dd2 != 31 && bx <= 31 && (bx == 0 || bx + dd2 <= 63);
        st.e_star = es;
        st.zd = es - es_ref;
        const int a1 = (dd1 < 0 ? -dd1 : dd1) & 31;
        o.swap = dd1 < 0;
        o.P = dd1 < 0 ? (1 << a1) : -(1 << a1);
        o.Q = dd2;
        break;
      }
      case FK_SCAL:
        st.e_star = q.ae + hx.e;
        break;
      case FK_AXPBY: {
        int dd, es, zd;
        lean_align(q.ae + hx.e, q.be + hy.e, q.am == 0 || hx.bits == 0,
                   q.bm == 0 || hy.bits == 0, dd, es, zd);
        // (a shift count beyond 62 only meets a zero operand)
        fast = fast && lean_cbits(q.am, hx.bits, q.bm, hy.bits, dd) <= 63;
        st.e_star = es;
        st.zd = zd;
        o.d = dd;
        break;
      }
      case FK_RESTRICT:
        // (1,2,1)^d sums of 32-bit operands: 32-bit when they fit, else 64-bit (config 1 runs
        // its V-cycle at 28 bits: 28 + 4 > 31)
        o.swap = effx + 2 * q.dim + 2 > 31;
        st.e_star = q.ea + hx.e;
        break;
      case FK_PROLONG:
        fast = fast && effx + q.dim + 2 <= 31;
        st.e_star = q.ea + hx.e;
        break;
      case FK_PCORR: {
        int dd, es, zd;
        lean_align(q.ae + q.ea + hx.e, q.be + hy.e, hx.bits == 0, hy.bits == 0, dd, es, zd);
        const int bg = hx.bits ? hx.bits + q.dim + 2 : 0, by = hy.bits;
        const int nd = lean_cbits(1, bg, 1, by, dd);
        const int ad = dd >= 0 ? dd : -dd;
        fast = fast && nd <= 63 && bg <= 31 && by <= 31 && ad <= 30;
        st.e_star = es;
        st.zd = zd;
        o.swap = dd < 0;
        o.P = 1 << (ad & 31);
        break;
      }
      default: fast = false;
    }
    o.sx = hx.s;
    o.sy = hy.s;
    if (fast && st.nnq) {  // nnqcomp: gamma fixes the window before the body (:189-212)
      lean_gamma(f.p.gamma, f.lr, ls, log, st.prod, st.gm, st.ge);
      const int lam = msb32(st.gm) + st.ge - st.e_star - st.w_out;
      fast = lam >= -62 && lam <= 1000;
      o.lam = lam;
    }
  }
  o.fast = fast;
  ls.dyn = o;
  return fast;
}

// data pointers of a record are arena byte offsets (below kArenaMaxBytes) or global
template <typename T> __device__ __forceinline__ T* lean_ptr(T* p, char* arena) {
  return (uintptr_t)p < (uintptr_t)kArenaMaxBytes ? reinterpret_cast<T*>(arena + (uintptr_t)p) : p;
}

// ---- worker bodies: 4 exact rows of one output group --------------------------------
__device__ __forceinline__ void lean_eval4(int kind, const LeanRec& s, const LeanDyn& c, int o,
                                           int64_t z[4]) {
  const int dim = s.dim, l = s.l;
  switch (kind) {
    case FK_GEMV: {
      Vec xv;
      xv.data = (void*)s.x;
      int g[4], cc[4], yv[4];
      stencil4_32<false>(xv, c.sx, dim, l, o, g, cc);
      const int4 t = *reinterpret_cast<const int4*>(s.y + o);
      yv[0] = t.x >> c.sy, yv[1] = t.y >> c.sy, yv[2] = t.z >> c.sy, yv[3] = t.w >> c.sy;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int X = c.swap ? yv[j] : g[j], Y = c.swap ? g[j] : yv[j];
        z[j] = (int64_t)X * (int64_t)c.P + (int64_t)(c.Q * Y);
      }
      const unsigned mN = (1u << l) - 1;
      if (((unsigned)o & mN) == mN - 3) z[3] = 0;
      if (plane_pad(dim, l, 0, o)) z[0] = z[1] = z[2] = z[3] = 0;
      break;
    }
    case FK_JACOBI: {
      Vec xv;
      xv.data = (void*)s.x;
      int g[4], cx[4], bv[4];
      stencil4_32<false>(xv, c.sx, dim, l, o, g, cx);
      const int4 t = *reinterpret_cast<const int4*>(s.y + o);
      bv[0] = t.x >> c.sy, bv[1] = t.y >> c.sy, bv[2] = t.z >> c.sy, bv[3] = t.w >> c.sy;
      const uint64_t cm = (uint64_t)(unsigned)s.am;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int X = c.swap ? bv[j] : g[j], Y = c.swap ? -g[j] : bv[j];
        const int64_t r = (int64_t)X * (int64_t)c.P + (int64_t)Y;
        const int64_t cr = (int64_t)((uint64_t)r * cm);
        z[j] = mad_pow2(cx[j], c.Q, cr);
      }
      const unsigned mN = (1u << l) - 1;
      if (((unsigned)o & mN) == mN - 3) z[3] = 0;
      if (plane_pad(dim, l, 0, o)) z[0] = z[1] = z[2] = z[3] = 0;
      break;
    }
    case FK_SCAL: {
      const int4 t = *reinterpret_cast<const int4*>(s.x + o);
      z[0] = (int64_t)s.am * (int64_t)(t.x >> c.sx);
      z[1] = (int64_t)s.am * (int64_t)(t.y >> c.sx);
      z[2] = (int64_t)s.am * (int64_t)(t.z >> c.sx);
      z[3] = (int64_t)s.am * (int64_t)(t.w >> c.sx);
      break;
    }
    case FK_AXPBY: {
      const int4 a = *reinterpret_cast<const int4*>(s.x + o);
      const int4 b = *reinterpret_cast<const int4*>(s.y + o);
      z[0] = combine32(s.am, a.x >> c.sx, s.bm, b.x >> c.sy, c.d);
      z[1] = combine32(s.am, a.y >> c.sx, s.bm, b.y >> c.sy, c.d);
      z[2] = combine32(s.am, a.z >> c.sx, s.bm, b.z >> c.sy, c.d);
      z[3] = combine32(s.am, a.w >> c.sx, s.bm, b.w >> c.sy, c.d);
      break;
    }
    case FK_RESTRICT: {
      const int lc = l - 1;
      const int Nc = 1 << lc, mc = Nc - 1, Nf = 1 << l;
      bool pad[4];
      pad4(dim, lc, o, pad, 0);
      const int I0 = o & mc, J = (o >> lc) & mc, K = (o >> (2 * lc)) & mc;
      int acc[4] = {0, 0, 0, 0}, w[4];
      RestrictOp ro;
      if (c.swap) {  // wide: the same sums in 64 bits
        int64_t a64[4] = {0, 0, 0, 0};
        const int planes = dim >= 3 ? 3 : 1, rows = dim >= 2 ? 3 : 1;
        for (int pz = 0; pz < planes; ++pz)
          for (int py = 0; py < rows; ++py) {
            const int32_t* f = s.x + 2 * I0 + (dim >= 2 ? (2 * J + py) * Nf : 0) +
                               (dim >= 3 ? (2 * K + pz) * Nf * Nf : 0);
            const int wy = (dim >= 2 && py == 1 ? 2 : 1) * (dim >= 3 && pz == 1 ? 2 : 1);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              a64[j] += (int64_t)wy * ((int64_t)(f[2 * j] >> c.sx) + 2 * (int64_t)(f[2 * j + 1] >> c.sx) +
                                       (int64_t)(f[2 * j + 2] >> c.sx));
          }
#pragma unroll
        for (int j = 0; j < 4; ++j) z[j] = pad[j] ? 0 : a64[j];
        break;
      }
      if (dim == 1) {
        ro.template line4<false>(s.x + 2 * I0, c.sx, acc);
      } else {
        int base = 2 * I0 + 2 * J * Nf;
        if (dim >= 3) base += 2 * K * Nf * Nf;
        const int32_t* fb = s.x + base;
        const int planes = dim >= 3 ? 3 : 1;
        for (int pz = 0; pz < planes; ++pz) {
          const int wz = dim >= 3 ? (pz == 1 ? 2 : 1) : 1;
          const int32_t* fp = fb + (dim >= 3 ? pz * Nf * Nf : 0);
#pragma unroll
          for (int py = 0; py < 3; ++py) {
            ro.template line4<false>(fp + py * Nf, c.sx, w);
            const int wy = (py == 1 ? 2 : 1) * wz;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] += wy * w[j];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) z[j] = pad[j] ? 0 : (int64_t)acc[j];
      break;
    }
    case FK_PROLONG: {
      Vec xv;
      xv.data = (void*)s.x;
      bool pad[4];
      pad4(dim, l, o, pad, 0);
      int g[4];
      prolong4_32<false>(xv, c.sx, dim, l, 0, o, g);
#pragma unroll
      for (int q = 0; q < 4; ++q) z[q] = pad[q] ? 0 : (int64_t)g[q];
      break;
    }
    default: {  // FK_PCORR
      Vec xv;
      xv.data = (void*)s.x;
      bool pad[4];
      pad4(dim, l, o, pad, 0);
      int g[4], yv[4];
      prolong4_32<false>(xv, c.sx, dim, l, 0, o, g);
      const int4 t = *reinterpret_cast<const int4*>(s.y + o);
      yv[0] = t.x >> c.sy, yv[1] = t.y >> c.sy, yv[2] = t.z >> c.sy, yv[3] = t.w >> c.sy;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int X = c.swap ? yv[q] : g[q], Y = c.swap ? g[q] : yv[q];
        z[q] = pad[q] ? 0 : (int64_t)X * (int64_t)c.P + (int64_t)Y;
      }
    }
  }
}

}  // namespace bfpdev

namespace bfpdev {
constexpr int kHdrStride = (int)((sizeof(Hdr) + 127) / 128 * 128);  // arena header pitch
__device__ __forceinline__ Hdr* lean_hdr_at(char* arena, int v) {
  return reinterpret_cast<Hdr*>(arena + 128 + kHdrStride * v);
}
// compact state of vector v from its block header
__device__ __forceinline__ LH lean_refresh(int v, LeanShared& ls, char* arena) {
  const LH h = lean_hdr(lean_hdr_at(arena, v));
  ls.fh[v] = make_fh(h.e, h.s, h.bits, h.eff, h.ok);
  return h;
}
// block header of a vector from the log entry of its last writer (fast ops keep only the
// compact state current; the generic path and the end of the list need the header)
__device__ __forceinline__ void lean_materialize(int v, const LeanShared& ls, const LogRec* log,
                                                 char* arena) {
  const int j = ls.lastw[v];
  if (j < 0) return;
  const LogRec& r = log[j];
  if (r.st == LOG_GENERIC) return;
  Hdr* h = lean_hdr_at(arena, v);
  h->q = r.q;
  h->e = r.e_out;
  h->shift = 0;
  h->max_m = r.mx;
  h->min_m = r.mn;
  h->flags = r.flags;
  h->lam_out = r.lam;
  h->need_recompute = 0;
}
// The generic path for op i of the list (bfp_coarse.cuh: setup + gamma, deferred-shift pass,
// finalize, recompute pass when a flag fires), on the block headers: the operands' headers
// are materialised from the log first, the output's compact state refreshed after.
__device__ __noinline__ void lean_generic(FusedOp& f, int i, int nar, char* arena,
                                          CoarseShared& sh, LeanShared& ls, LogRec* log) {
  const int t = threadIdx.x;
  if (t == 0) {
    for (int v = 0; v < nar; ++v) lean_materialize(v, ls, log, arena);
    coarse_prepare<int32_t>(f, arena, sh);
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    Red r;
    r.init();
    const int mode = pass ? MODE_RECOMPUTE : f.p.mode;
    if (!(pass && sh.c.skip)) coarse_body<int32_t>(f, mode, sh, r);
    coarse_publish(r, sh);
    __syncthreads();
    if (t < 32) {
      int bits = 1, err = 0;
      int64_t mx = 0, mn = 0;
      coarse_totals(sh, bits, mx, mn, err);
      if (t == 0) {
        int rc = 0;
        if (!(pass && sh.c.skip)) rc = win_finalize(f.p, sh.c, f.out.hdr, bits, mx, mn, err);
        if (rc && !pass) {
          f.p.mode = MODE_RECOMPUTE;
          WinCtx c2;
          win_setup(f.p, f.out.hdr, sh.c.e_star, 32, c2);
          sh.c = c2;
        }
        sh.rc = rc && !pass;
      }
    }
    __syncthreads();
    if (!sh.rc) break;
  }
  if (t == 0) {
    const int v = f.lr.vout;
    const LH h = lean_refresh(v, ls, arena);
    LogRec& r = log[i];
    r.st = LOG_GENERIC;
    r.e_out = h.e;
    // effective extremes (pending shift applied); a header beyond 32 bits makes every
    // consumer generic, which reads the header itself
    r.mx = (int)(f.out.hdr->max_m >> h.s);
    r.mn = (int)(f.out.hdr->min_m >> h.s);
    ls.lastw[v] = i;
  }
}
}  // namespace bfpdev

// measurement builds (-DBFP_COARSE_TIMING): the lean engine's per-phase clocks share
// g_coarse_prof (slots: 0 wait, 1 arena, 2 post-setup, 3 barrier A, 4 pre-setup, 5 barrier B,
// 6 totals + core finalize, 7 writeback, 10 barrier C, 11 generic ops, 12 epilogue)
__global__ void __launch_bounds__(kFusedThreads) lean_kernel(const FusedOp* ops, int n,
                                                             const ArenaEntry* ar, int nar,
                                                             int zoff, int64_t* zglobal,
                                                             int loff) {
  extern __shared__ __align__(128) char arena[];
  __shared__ __align__(16) CoarseShared sh;
  __shared__ __align__(16) LeanShared ls;
  constexpr int kChunks = (int)(sizeof(FusedOp) / 16);
  static_assert(kChunks <= kLeanWorkers, "one prefetch chunk per worker thread");
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  int64_t* zbuf = zglobal ? zglobal : reinterpret_cast<int64_t*>(arena + zoff);
  LogRec* log = reinterpret_cast<LogRec*>(arena + loff);
  // Record k -> slot k & 3 with cp.async (one 16-byte chunk per stager thread, no
  // registers): issued during op k - 3, waited for during op k - 2, read from op k - 1 on.
  // Arena offsets in the record stay offsets; their readers rebase (lean_ptr / the generic
  // path's coarse_prepare).
  const int wt = t - 32;  // worker index; workers 0 .. kChunks - 1 stage the records
  const bool stager = wt >= 0 && wt < kChunks;
  auto issue = [&](int k) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(reinterpret_cast<int4*>(&sh.f[k & 3]) + wt);
    const int4* src = reinterpret_cast<const int4*>(&ops[k]) + wt;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  };
  auto landed = [&]() { asm volatile("cp.async.wait_all;" ::: "memory"); };
  // records do not depend on the previous kernel: the first three are fetched before the
  // wait, and the rest of the list is pulled into L2
  if (stager) {
    issue(0);
    if (n > 1) issue(1);
    if (n > 2) issue(2);
    landed();
  }
  for (int64_t b = (int64_t)t * 128 + 3 * (int64_t)sizeof(FusedOp); b < (int64_t)n * (int64_t)sizeof(FusedOp);
       b += (int64_t)kFusedThreads * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(ops) + b));
  if (t == 0) sh.rc = 0;
  // the arena entry table is static: stage it before the wait
  __shared__ __align__(16) ArenaEntry s_ar[kLeanMaxVec];
  static_assert(sizeof(ArenaEntry) % 8 == 0, "entry table copied in 8-byte words");
  for (int w = t; w < nar * (int)(sizeof(ArenaEntry) / 8); w += kFusedThreads)
    reinterpret_cast<int64_t*>(s_ar)[w] = __ldg(reinterpret_cast<const int64_t*>(ar) + w);
  CPROF_T();
  griddep_wait();
  CPROF(0);
  __syncthreads();  // the entry table is in shared memory
  // headers always, data while it fits -> shared memory: every copy is issued as cp.async
  // before anything waits (a loop of synchronous copies cost one memory latency per entry,
  // 45,000 clk per launch with ~45 vectors)
  auto async16 = [](void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
  };
  for (int k = 0; k < nar; ++k) {
    const ArenaEntry& e = s_ar[k];
    const int n16 = (int)(e.bytes >> 4);
    for (int i = t; i < n16; i += kFusedThreads) async16(arena + e.off + 16 * i, e.gbase + 16 * i);
    if (t < (int)(sizeof(Hdr) / 16))
      async16(arena + e.hoff + 16 * t, reinterpret_cast<const char*>(e.ghdr) + 16 * t);
  }
  for (int k = t; k < n; k += kFusedThreads) log[k].st = LOG_NONE;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // compact vector states and the norms at entry, one thread per header
  if (t < nar) {
    const LH h = lean_refresh(t, ls, arena);
    ls.init_e[t] = h.e;
    ls.init_mag[t] = h.mag;  // (only read when ok: a header out of range makes its ops generic)
    ls.lastw[t] = -1;
  }
  __syncthreads();
  CPROF(1);
  LeanState st;
  __shared__ LeanPre pre;  // control lane only: written by the first half, read by the second
  const FH nofh = FH{0, 0, 0, 0};
  if (t == 0) {
    lean_pre(sh.f[0], nullptr, ls, pre);
    lean_post(sh.f[0], pre, -1, nofh, -1, ls, log, st);
  }
  CPROF(2);
  CPROF_CNT(8, 1);
  CPROF_CNT(9, n);
  for (int i = 0; i < n; ++i) {
    __syncthreads();  // (A) context of op i published; the data of op i - 1 is visible
    CPROF(3);
    FusedOp& f = sh.f[i & 3];
#ifdef BFP_COARSE_TIMING
    const long long _w0 = clock64();
#endif
    if (stager) {  // record i + 2 (issued during op i - 1) has landed; fetch record i + 3
      landed();
      if (i + 3 < n) issue(i + 3);
    }
#ifdef BFP_COARSE_TIMING
    if (t == 32 && i < 4096) g_coarse_ops[4 * i] = (int)(clock64() - _w0);
#endif
    if (!ls.dyn.fast) {
      lean_generic(f, i, nar, arena, sh, ls, log);
      if (t == 0 && i + 1 < n) {
        lean_pre(sh.f[(i + 1) & 3], nullptr, ls, pre);
        lean_post(sh.f[(i + 1) & 3], pre, -1, nofh, -1, ls, log, st);
      }
      CPROF(11);
      continue;
    }
    // ---- fast path ----
    const int kind = f.kind;
    int32_t* st_out = nullptr;  // the workers' copies for the store phase
    int st_n4 = 0, st_mm = 0;
    if (warp > 0) {
      LeanRec s = f.lr;
      s.x = lean_ptr(s.x, arena);
      s.y = lean_ptr(s.y, arena);
      s.out = lean_ptr(s.out, arena);
      const LeanDyn c = ls.dyn;
      st_out = s.out;
      st_n4 = s.n4;
      st_mm = c.needmm;
      if (kind == FK_ZERO) {
        for (int g = wt; g < s.n4; g += kLeanWorkers)
          reinterpret_cast<int4*>(s.out)[g] = make_int4(0, 0, 0, 0);
      } else {
        // OR of z ^ sign(z) (mu*), with the sign in bit 63 (all rows in {0, -1}: any -1?)
        uint64_t orv = 0;
        int64_t mx = INT64_MIN, mn = INT64_MAX;
        for (int g = wt; g < s.n4; g += kLeanWorkers) {
          int64_t z[4];
          lean_eval4(kind, s, c, 4 * g, z);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (s.nnq) z[j] = shift_clamp<int64_t>(z[j], c.lam, s.w_out);
            orv |= (uint64_t)(z[j] ^ (z[j] >> 63)) | ((uint64_t)z[j] & 0x8000000000000000ull);
            if (st_mm) {
              mx = z[j] > mx ? z[j] : mx;
              mn = z[j] < mn ? z[j] : mn;
            }
          }
          longlong2* zp = reinterpret_cast<longlong2*>(zbuf + 4 * (size_t)g);
          zp[0] = make_longlong2(z[0], z[1]);
          zp[1] = make_longlong2(z[2], z[3]);
        }
        orv = redux_or64(orv);
        if (st_mm) {
          mx = redux_max64(mx);
          mn = redux_min64(mn);
        }
        if (lane == 0) {
          ls.orv[warp] = orv;
          if (st_mm) {
            ls.mx[warp] = mx;
            ls.mn[warp] = mn;
          }
        }
      }
    } else if (t == 0 && i + 1 < n) {
      lean_pre(sh.f[(i + 1) & 3], nullptr, ls, pre);  // first half of the next op's setup
    }
#ifdef BFP_COARSE_TIMING
    if (t == 32 && i < 4096) g_coarse_ops[4 * i + 2] = (int)(clock64() - _w0);
#endif
    CPROF(4);
    __syncthreads();  // (B) warp partials published
    CPROF(5);
    FH ff = nofh;  // control lane: the fresh state of this op's output
    if (warp == 0) {
      if (kind == FK_ZERO) {
        if (t == 0) {  // zero_vec (P/src/bfp.cpp:53-55)
          LogRec r;
          r.st = LOG_ZERO;
          r.q = (short)f.q;
          r.e_out = r.lam = r.mu = r.mx = r.mn = r.flags = 0;
          log[i] = r;
          ff = make_fh(0, 0, 0, 1, true);
          ls.fh[st.vout] = ff;
          ls.lastw[st.vout] = i;
        }
      } else {
        const bool on = lane >= 1 && lane < kCoarseWarps;
        const uint64_t o2 = redux_or64(on ? ls.orv[lane] : 0ull);
        const int mm = ls.dyn.needmm;
        int64_t tmx = 0, tmn = 0;
        if (mm) {
          tmx = redux_max64(on ? ls.mx[lane] : INT64_MIN);
          tmn = redux_min64(on ? ls.mn[lane] : INT64_MAX);
        }
        if (t == 0) {
          int lam, mu = 0, e_out;
          const bool anyneg = (o2 >> 63) != 0;
          const uint64_t mag = o2 & 0x7fffffffffffffffull;
          const bool allzero = mag == 0 && !anyneg;
          LogRec r;
          r.gm = r.ge = 0;
          if (st.nnq) {
            lam = 0;  // rows were clamped in the body; e_out = e* + lam_out (:211)
            e_out = st.e_star + ls.dyn.lam;
            r.st = LOG_FASTN;
            r.gm = st.gm;
            r.ge = st.ge;
            r.mx = (int)tmx;
            r.mn = (int)tmn;
            const int ma = msb32((int)tmx), mb = msb32((int)tmn);
            const int eff = ma > mb ? ma : mb;
            ff = make_fh(e_out, 0, allzero ? 0 : eff, eff, small_e(e_out));
          } else {
            mu = bitlen64(mag) + 1;                    // mu* (init 1, P/src/blas.cpp:153)
            if (st.zd > 0 && allzero) mu = 1 - st.zd;  // all-zero anchor in the op's coordinates
            lam = mu - st.w_out;                       // :164
            e_out = st.e_star + lam;
            r.st = LOG_FASTQ;
            if (mm) {  // the next op is nnqcomp: extremes of the stored values now
              r.mx = (int)(lam >= 0 ? tmx >> (lam > 63 ? 63 : lam) : tmx << -lam);
              r.mn = (int)(lam >= 0 ? tmn >> (lam > 63 ? 63 : lam) : tmn << -lam);
            } else {   // reduced by the workers in the store phase
              r.mx = INT32_MIN;
              r.mn = INT32_MAX;
            }
            // a normalised block: width w_out unless every row is zero
            ff = make_fh(e_out, 0, allzero ? 0 : st.w_out, allzero ? 1 : st.w_out, small_e(e_out));
          }
          ls.lam_store = lam;
          r.e_out = e_out;
          r.lam = lam;
          r.mu = mu;
          r.e_star = st.e_star;
          r.q = (short)st.w_out;
          r.flags = 0;
          r.prod[0] = st.prod[0];
          r.prod[1] = st.prod[1];
          r.prod[2] = st.prod[2];
          r.pad = 0;
          log[i] = r;
          ls.fh[st.vout] = ff;
          ls.lastw[st.vout] = i;
        }
      }
    }
#ifdef BFP_COARSE_TIMING
    if (t == 0 && i < 4096) g_coarse_ops[4 * i + 3] = (int)(clock64() - _ct);
#endif
    CPROF(6);
    __syncthreads();  // (C) lam_out published
    CPROF(10);
    if (warp > 0) {
      if (kind != FK_ZERO) {
        const int lam = ls.lam_store;
        const int rs = lam >= 0 ? (lam > 63 ? 63 : lam) : 0, lsh = lam < 0 ? -lam : 0;
        int smx = INT32_MIN, smn = INT32_MAX;
        for (int g = wt; g < st_n4; g += kLeanWorkers) {
          const longlong2* zp = reinterpret_cast<const longlong2*>(zbuf + 4 * (size_t)g);
          const longlong2 a = zp[0], b = zp[1];
          int4 v;
          v.x = (int)((a.x >> rs) << lsh);
          v.y = (int)((a.y >> rs) << lsh);
          v.z = (int)((b.x >> rs) << lsh);
          v.w = (int)((b.y >> rs) << lsh);
          reinterpret_cast<int4*>(st_out)[g] = v;
          smx = max(max(max(v.x, v.y), max(v.z, v.w)), smx);
          smn = min(min(min(v.x, v.y), min(v.z, v.w)), smn);
        }
        if (!st_mm) {  // extremes of the stored values -> the op's log entry
          smx = __reduce_max_sync(0xffffffffu, smx);
          smn = __reduce_min_sync(0xffffffffu, smn);
          if (lane == 0) {
            atomicMax(&log[i].mx, smx);
            atomicMin(&log[i].mn, smn);
          }
        }
      }
    } else if (t == 0 && i + 1 < n) {
      // second half of the next op's setup, with this op's output state forwarded
      lean_post(sh.f[(i + 1) & 3], pre, st.vout, ff, i, ls, log, st);
#ifdef BFP_COARSE_TIMING
      if (i + 1 < 4096) g_coarse_ops[4 * (i + 1) + 1] = (int)(clock64() - _ct);
#endif
    }
    CPROF(2);
  }
  __syncthreads();
  griddep_launch_dependents();
  // ---- end of the list: gamma, flags, trace and history of every fast op, one thread per
  // op (records re-read from global memory) ----
  for (int k = t; k < n; k += kFusedThreads) {
    LogRec& r = log[k];
    if (r.st != LOG_FASTQ && r.st != LOG_FASTN) continue;
    const FusedOp& g = ops[k];
    const WinParams& p = g.p;
    WinCtx c;
    if (r.st == LOG_FASTN) {
      c.gm = r.gm;
      c.ge = r.ge;
      write_trace(p, c, 0, 0, 0, 0);
    } else {
      int gm, ge;
      lean_gamma(p.gamma, g.lr, ls, log, r.prod, gm, ge);
      c.gm = gm;
      c.ge = ge;
      const int mu_tmp = msb32(gm) + ge - r.e_star;
      const int ovf = mu_tmp < r.mu, unf = r.lam < mu_tmp - (int)p.w_tmp;  // :167-168
      const int rc = ovf || unf;
      r.flags = (short)((ovf ? FLAG_OVERFLOW : 0) | (unf ? FLAG_UNDERFLOW : 0) |
                        (rc ? FLAG_RECOMPUTED : 0) | FLAG_NORMALIZED);
      write_trace(p, c, ovf, unf, rc, 1);
    }
    if (p.hist != nullptr && p.hist_slot >= 0) {
      const unsigned a = r.mx < 0 ? 0u - (unsigned)r.mx : (unsigned)r.mx;
      const unsigned b = r.mn < 0 ? 0u - (unsigned)r.mn : (unsigned)r.mn;
      p.hist[p.hist_slot] = ldexp((double)(a > b ? a : b), r.e_out);
    }
  }
  __syncthreads();
  if (t < nar) lean_materialize(t, ls, log, arena);
  __syncthreads();
  CPROF(12);
  for (int k = 0; k < nar; ++k) {  // publish the fused part's outputs
    const ArenaEntry& e = s_ar[k];
    if (!e.wb) continue;
    if (e.bytes) arena_copy(e.gbase, arena + e.off, e.bytes);
    if (t < (int)(sizeof(Hdr) / 16))
      reinterpret_cast<int4*>(e.ghdr)[t] = reinterpret_cast<const int4*>(arena + e.hoff)[t];
  }
  CPROF(7);
}
