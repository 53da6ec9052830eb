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
//   * op records are prefetched two ops ahead and their arena pointers rebased by the
//     prefetching threads (FusedOp::rb marks the pointer words).
#pragma once
#include "bfp_coarse.cuh"

namespace bfpdev {

constexpr int kLeanWorkers = kFusedThreads - 32;

struct LeanOp {  // window context of a fast op, published by the control lane
  int fast, kind, nnq;
  int needmm;    // qcomp: reduce max / min of z in the body (the next op is nnqcomp)
  int dim, l;
  int sx, sy;    // pending shifts of the operands
  int P, Q;      // gemv / pcorr: z = X P + Q Y; jacobi: P1 and s2
  int swap;      // gemv / pcorr: operands swapped (d < 0); jacobi: neg1
  unsigned cm;   // jacobi: c.m
  int am, bm, d; // axpby / scal: coefficients and alignment
  int lam, wout; // nnqcomp window
  int n4;        // 4-groups of the output
  const int32_t *x, *y;
  int32_t* out;
};

// compact state of a vector for the control lane's setups
struct FH {
  int e, s, bits, eff;  // exponent, pending shift, width (0: all zero), eff_bits
  int ok;
};
// one record per op of the list (shared memory)
enum { LOG_NONE = 0, LOG_FASTQ, LOG_FASTN, LOG_GENERIC, LOG_ZERO };
struct LogRec {
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
  LeanOp op;
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
// path only admits rules with 32-bit coefficients (lean_rule_ok)
__device__ __forceinline__ bool lean_rule_ok(const GammaRule& g) {
  if (g.literal || g.exact || g.nterms > 3) return false;
  for (int i = 0; i < g.nterms; ++i)
    if (g.t[i].cm < 0 || g.t[i].cm > 0xffffffffll || !small_e(g.t[i].ce)) return false;
  return true;
}
template <typename VidFn>
__device__ __forceinline__ void lean_gamma(const GammaRule& g, const LeanShared& ls,
                                           const LogRec* log, const short* prod, VidFn vid,
                                           int& gm, int& ge) {
  G32 acc{0, 0};
  for (int i = 0; i < g.nterms; ++i) {
    const GTerm& t = g.t[i];
    G32 x;
    if (t.v == nullptr) {
      x = G32{1 << 14, -14};
    } else {
      const NormSrc ns = lean_norm(ls, log, vid(t.v), prod[i]);
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

// ---- the control lane's per-op state (registers) ------------------------------------
struct LeanState {
  int e_star, zd;  // template exponent, zero-term elision shift
  int w_out, nnq;
  int gm, ge;      // nnqcomp: gamma
  int vout;        // vector id of the output
  short prod[3];
};

__device__ __forceinline__ int clog2_4dim(int dim) { return dim == 1 ? 2 : (dim == 2 ? 3 : 4); }

// Lean setup of op record f (control lane): true when the op runs on the fast path.
// Restates the setups of bfp_ops.cuh (template exponent, zero-term elision, width bounds and
// the `narrow` conditions) in 32-bit arithmetic on the compact vector states; every rejected
// case takes the generic path.
template <typename VidFn>
__device__ __forceinline__ bool lean_setup(const FusedOp& f, const FusedOp* next, LeanShared& ls,
                                           const LogRec* log, VidFn vid, LeanState& st) {
  LeanOp& o = ls.op;
  const WinParams& p = f.p;
  o.kind = f.kind;
  o.out = (int32_t*)f.out.data;
  o.n4 = (int)(f.out.n >> 2);
  o.nnq = 0;
  o.needmm = 0;
  st.vout = vid(f.out.hdr);
  st.nnq = 0;
  if (f.kind == FK_ZERO) return true;
  if (p.part || p.force || p.w_tmp > 32 || p.w_out > 32 || p.w_out < 1) return false;
  if (p.mode != MODE_QCOMP && p.mode != MODE_NNQ) return false;
  if (!lean_rule_ok(p.gamma)) return false;
  st.w_out = (int)p.w_out;
  st.nnq = p.mode == MODE_NNQ;
  o.nnq = st.nnq;
  // a qcomp op followed by an nnqcomp op reduces max / min in its body: the next setup
  // needs them (gamma, width) before this op's store phase has finished
  o.needmm = !st.nnq && next != nullptr && next->p.mode == MODE_NNQ;
  o.wout = st.w_out;
  st.zd = 0;
  const FH* fh = ls.fh;
  switch (f.kind) {
    case FK_GEMV: {
      const GemvOp& g = f.u.gemv;
      if (g.st9 || g.gs || g.l < 2 || g.z0 || !small_e(g.al.e) || !small_e(g.be.e)) return false;
      if (g.al.m != (int)g.al.m || g.be.m != (int)g.be.m) return false;
      const FH hx = fh[vid(g.x.hdr)], hy = fh[vid(g.y.hdr)];
      if (!hx.ok || !hy.ok) return false;
      const int am = (int)g.al.m, bm = (int)g.be.m;
      int dd, es, zd;
      lean_align((int)g.al.e + g.ea + hx.e, (int)g.be.e + hy.e, am == 0 || hx.bits == 0,
                 bm == 0 || hy.bits == 0, dd, es, zd);
      const int bg = hx.bits ? hx.bits + clog2_4dim(g.dim) + 1 : 0, by = hy.bits;
      const int nd = lean_cbits(am, bg, bm, by, dd);
      const int ad = dd >= 0 ? dd : -dd;
      const int pm = dd >= 0 ? am : bm, qm = dd >= 0 ? bm : am;
      const int bx_ = dd >= 0 ? bg : by, by_ = dd >= 0 ? by : bg;
      const int mp = msb32(pm), mq = msb32(qm);
      const bool nar = bg <= 31 && by <= 31 && (by_ == 0 || mq + by_ <= 32) && nd <= 63 &&
                       ad <= 30 && mp + ad <= 32 && (bx_ == 0 || mp + ad + bx_ <= 63);
      if (!nar) return false;
      st.e_star = es;
      st.zd = zd;
      o.dim = g.dim;
      o.l = g.l;
      o.sx = hx.s;
      o.sy = hy.s;
      o.P = pm << ad;
      o.Q = qm;
      o.swap = dd < 0;
      o.x = (const int32_t*)g.x.data;
      o.y = (const int32_t*)g.y.data;
      break;
    }
    case FK_JACOBI: {
      const JacobiOp& j = f.u.jac;
      if (j.l < 2 || j.z0 || !small_e(j.c.e) || j.c.m < 0 || j.c.m > 0x7fffffff) return false;
      const FH hx = fh[vid(j.x.hdr)], hb = fh[vid(j.b.hdr)];
      if (!hx.ok || !hb.ok) return false;
      const int cm = (int)j.c.m, ce = (int)j.c.e;
      const int ge = 2 * j.l + hx.e;
      const bool zx = hx.bits == 0, zb = hb.bits == 0;
      const int gb = ge < hb.e ? ge : hb.e;
      const int es_ref = hx.e < ce + gb ? hx.e : ce + gb;
      int dd1, er, zr, dd2, es;
      lean_align(ge, hb.e, zx, zb, dd1, er, zr);
      lean_align(hx.e, ce + er, zx, cm == 0 || (zx && zb), dd2, es, zr);
      const int bx = hx.bits, bbb = hb.bits;
      const int bg = bx ? bx + clog2_4dim(j.dim) + 1 : 0;
      const int br = lean_cbits(-1, bg, 1, bbb, dd1);
      const int nd = lean_cbits(1, bx, cm, br, dd2);
      const bool nar = bg <= 31 && bbb <= 31 && nd <= 63 && dd1 >= -30 && dd1 <= 30 &&
                       dd2 >= 0 && dd2 <= 62 && dd2 != 31 && bx <= 31 &&
                       (bx == 0 || bx + dd2 <= 63);
      if (!nar) return false;
      st.e_star = es;
      st.zd = es - es_ref;
      o.dim = j.dim;
      o.l = j.l;
      o.sx = hx.s;
      o.sy = hb.s;
      o.swap = dd1 < 0;
      o.P = dd1 < 0 ? (1 << -dd1) : -(1 << dd1);
      o.Q = dd2;
      o.cm = (unsigned)cm;
      o.x = (const int32_t*)j.x.data;
      o.y = (const int32_t*)j.b.data;
      break;
    }
    case FK_SCAL: {
      const ScalOp& s = f.u.scal;
      if (!small_e(s.c.e) || s.c.m != (int)s.c.m) return false;
      const FH hr = fh[vid(s.r.hdr)];
      if (!hr.ok) return false;
      st.e_star = (int)s.c.e + hr.e;
      o.sx = hr.s;
      o.am = (int)s.c.m;
      o.x = (const int32_t*)s.r.data;
      break;
    }
    case FK_AXPBY: {
      const AxpbyOp& a = f.u.axpby;
      if (!small_e(a.al.e) || !small_e(a.be.e) || a.al.m != (int)a.al.m || a.be.m != (int)a.be.m)
        return false;
      const FH hx = fh[vid(a.x.hdr)], hy = fh[vid(a.y.hdr)];
      if (!hx.ok || !hy.ok) return false;
      const int am = (int)a.al.m, bm = (int)a.be.m;
      int dd, es, zd;
      lean_align((int)a.al.e + hx.e, (int)a.be.e + hy.e, am == 0 || hx.bits == 0,
                 bm == 0 || hy.bits == 0, dd, es, zd);
      const int nd = lean_cbits(am, hx.bits, bm, hy.bits, dd);
      if (nd > 63) return false;  // (a shift count beyond 62 only meets a zero operand)
      st.e_star = es;
      st.zd = zd;
      o.sx = hx.s;
      o.sy = hy.s;
      o.am = am;
      o.bm = bm;
      o.d = dd;
      o.x = (const int32_t*)a.x.data;
      o.y = (const int32_t*)a.y.data;
      break;
    }
    case FK_RESTRICT: {
      const RestrictOp& r = f.u.rst;
      if (r.gs || r.zc || r.l < 3) return false;
      const FH hr = fh[vid(r.r.hdr)];
      if (!hr.ok || hr.eff + 2 * r.dim + 2 > 31) return false;
      st.e_star = r.er + hr.e;
      o.dim = r.dim;
      o.l = r.l;
      o.sx = hr.s;
      o.x = (const int32_t*)r.r.data;
      break;
    }
    case FK_PROLONG: {
      const ProlongOp& q = f.u.pro;
      if (q.gs || q.zf || q.zp || q.l < 3) return false;
      const FH hc = fh[vid(q.xc.hdr)];
      if (!hc.ok || hc.eff + q.dim + 2 > 31) return false;
      st.e_star = q.ep + hc.e;
      o.dim = q.dim;
      o.l = q.l;
      o.sx = hc.s;
      o.x = (const int32_t*)q.xc.data;
      break;
    }
    case FK_PCORR: {
      const ProlongCorrectOp& q = f.u.pc;
      if (q.gs || q.zf || q.zp || q.l < 3 || q.al.m != 1 || q.be.m != 1 || !small_e(q.al.e) ||
          !small_e(q.be.e))
        return false;
      const FH hc = fh[vid(q.ec.hdr)], hy = fh[vid(q.y.hdr)];
      if (!hc.ok || !hy.ok) return false;
      int dd, es, zd;
      lean_align((int)q.al.e + q.ep + hc.e, (int)q.be.e + hy.e, hc.bits == 0, hy.bits == 0, dd, es,
                 zd);
      const int bg = hc.bits ? hc.bits + q.dim + 2 : 0, by = hy.bits;
      const int nd = lean_cbits(1, bg, 1, by, dd);
      const int ad = dd >= 0 ? dd : -dd;
      if (!(nd <= 63 && bg <= 31 && by <= 31 && ad <= 30)) return false;
      st.e_star = es;
      st.zd = zd;
      o.dim = q.dim;
      o.l = q.l;
      o.sx = hc.s;
      o.sy = hy.s;
      o.swap = dd < 0;
      o.P = 1 << ad;
      o.x = (const int32_t*)q.ec.data;
      o.y = (const int32_t*)q.y.data;
      break;
    }
    default: return false;
  }
  // producers of the gamma terms as of now (the rule is evaluated when the list ends)
  for (int i = 0; i < 3; ++i) {
    st.prod[i] = -1;
    if (i < p.gamma.nterms && p.gamma.t[i].v) {
      const int v = vid(p.gamma.t[i].v);
      if (!fh[v].ok) return false;
      st.prod[i] = (short)ls.lastw[v];
    }
  }
  if (st.nnq) {  // nnqcomp: gamma fixes the window before the body (P/src/blas.cpp:189-212)
    lean_gamma(p.gamma, ls, log, st.prod, vid, st.gm, st.ge);
    const int lam = msb32(st.gm) + st.ge - st.e_star - st.w_out;
    if (lam < -62 || lam > 1000) return false;
    o.lam = lam;
  }
  return true;
}

// ---- worker bodies: 4 exact rows of one output group --------------------------------
__device__ __forceinline__ void lean_eval4(const LeanOp& c, int o, int64_t z[4]) {
  switch (c.kind) {
    case FK_GEMV: {
      Vec xv;
      xv.data = (void*)c.x;
      int g[4], cc[4], yv[4];
      stencil4_32<false>(xv, c.sx, c.dim, c.l, o, g, cc);
      const int4 t = *reinterpret_cast<const int4*>(c.y + o);
      yv[0] = t.x >> c.sy, yv[1] = t.y >> c.sy, yv[2] = t.z >> c.sy, yv[3] = t.w >> c.sy;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int X = c.swap ? yv[j] : g[j], Y = c.swap ? g[j] : yv[j];
        z[j] = (int64_t)X * (int64_t)c.P + (int64_t)(c.Q * Y);
      }
      const unsigned mN = (1u << c.l) - 1;
      if (((unsigned)o & mN) == mN - 3) z[3] = 0;
      if (plane_pad(c.dim, c.l, 0, o)) z[0] = z[1] = z[2] = z[3] = 0;
      break;
    }
    case FK_JACOBI: {
      Vec xv;
      xv.data = (void*)c.x;
      int g[4], cx[4], bv[4];
      stencil4_32<false>(xv, c.sx, c.dim, c.l, o, g, cx);
      const int4 t = *reinterpret_cast<const int4*>(c.y + o);
      bv[0] = t.x >> c.sy, bv[1] = t.y >> c.sy, bv[2] = t.z >> c.sy, bv[3] = t.w >> c.sy;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int X = c.swap ? bv[j] : g[j], Y = c.swap ? -g[j] : bv[j];
        const int64_t r = (int64_t)X * (int64_t)c.P + (int64_t)Y;
        const int64_t cr = (int64_t)((uint64_t)r * (uint64_t)c.cm);
        z[j] = mad_pow2(cx[j], c.Q, cr);
      }
      const unsigned mN = (1u << c.l) - 1;
      if (((unsigned)o & mN) == mN - 3) z[3] = 0;
      if (plane_pad(c.dim, c.l, 0, o)) z[0] = z[1] = z[2] = z[3] = 0;
      break;
    }
    case FK_SCAL: {
      const int4 t = *reinterpret_cast<const int4*>(c.x + o);
      z[0] = (int64_t)c.am * (int64_t)(t.x >> c.sx);
      z[1] = (int64_t)c.am * (int64_t)(t.y >> c.sx);
      z[2] = (int64_t)c.am * (int64_t)(t.z >> c.sx);
      z[3] = (int64_t)c.am * (int64_t)(t.w >> c.sx);
      break;
    }
    case FK_AXPBY: {
      const int4 a = *reinterpret_cast<const int4*>(c.x + o);
      const int4 b = *reinterpret_cast<const int4*>(c.y + o);
      z[0] = combine32(c.am, a.x >> c.sx, c.bm, b.x >> c.sy, c.d);
      z[1] = combine32(c.am, a.y >> c.sx, c.bm, b.y >> c.sy, c.d);
      z[2] = combine32(c.am, a.z >> c.sx, c.bm, b.z >> c.sy, c.d);
      z[3] = combine32(c.am, a.w >> c.sx, c.bm, b.w >> c.sy, c.d);
      break;
    }
    case FK_RESTRICT: {
      const int lc = c.l - 1;
      const int Nc = 1 << lc, mc = Nc - 1, Nf = 1 << c.l;
      bool pad[4];
      pad4(c.dim, lc, o, pad, 0);
      const int I0 = o & mc, J = (o >> lc) & mc, K = (o >> (2 * lc)) & mc;
      int acc[4] = {0, 0, 0, 0}, w[4];
      RestrictOp ro;
      if (c.dim == 1) {
        ro.template line4<false>(c.x + 2 * I0, c.sx, acc);
      } else {
        int base = 2 * I0 + 2 * J * Nf;
        if (c.dim >= 3) base += 2 * K * Nf * Nf;
        const int32_t* fb = c.x + base;
        const int planes = c.dim >= 3 ? 3 : 1;
        for (int pz = 0; pz < planes; ++pz) {
          const int wz = c.dim >= 3 ? (pz == 1 ? 2 : 1) : 1;
          const int32_t* fp = fb + (c.dim >= 3 ? pz * Nf * Nf : 0);
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
      xv.data = (void*)c.x;
      bool pad[4];
      pad4(c.dim, c.l, o, pad, 0);
      int g[4];
      prolong4_32<false>(xv, c.sx, c.dim, c.l, 0, o, g);
#pragma unroll
      for (int q = 0; q < 4; ++q) z[q] = pad[q] ? 0 : (int64_t)g[q];
      break;
    }
    default: {  // FK_PCORR
      Vec xv;
      xv.data = (void*)c.x;
      bool pad[4];
      pad4(c.dim, c.l, o, pad, 0);
      int g[4], yv[4];
      prolong4_32<false>(xv, c.sx, c.dim, c.l, 0, o, g);
      const int4 t = *reinterpret_cast<const int4*>(c.y + o);
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

// measurement builds (-DBFP_COARSE_TIMING): the lean engine's per-phase clocks share
// g_coarse_prof (slots: 0 wait, 1 arena, 2 setup, 3 barrier A, 4 body, 5 barrier B,
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
  // block headers sit at arena offsets 128 + k kHdrStride: header pointer -> vector id k
  constexpr int kHdrStride = (int)((sizeof(Hdr) + 127) / 128 * 128);
  const char* hbase = arena + 128;
  auto vid = [hbase](const Hdr* h) { return (int)(((const char*)h - hbase) / kHdrStride); };
  // record k -> slot k & 3, arena pointers rebased on the way (words marked in rb)
  auto fetch = [&](int k, int c) {
    const int4* src = reinterpret_cast<const int4*>(&ops[k]);
    int4 v = __ldg(src + c);
    const int4 m = __ldg(src + 1);  // chunk 0: {kind, pad, q}; chunk 1: {rb[0], rb[1]}
    const uint64_t rb0 = ((uint64_t)(unsigned)m.y << 32) | (unsigned)m.x;
    const uint64_t rb1 = ((uint64_t)(unsigned)m.w << 32) | (unsigned)m.z;
    const int w0 = 2 * c;
    auto marked = [&](int w) { return (int)(((w < 64 ? rb0 >> w : rb1 >> (w - 64))) & 1); };
    if (marked(w0)) {
      const uint64_t a = (uint64_t)(uintptr_t)arena + (((uint64_t)(unsigned)v.y << 32) | (unsigned)v.x);
      v.x = (int)(unsigned)a;
      v.y = (int)(unsigned)(a >> 32);
    }
    if (marked(w0 + 1)) {
      const uint64_t a = (uint64_t)(uintptr_t)arena + (((uint64_t)(unsigned)v.w << 32) | (unsigned)v.z);
      v.z = (int)(unsigned)a;
      v.w = (int)(unsigned)(a >> 32);
    }
    reinterpret_cast<int4*>(&sh.f[k & 3])[c] = v;
  };
  // records 0 and 1 do not depend on the previous kernel: fetch them before the wait
  if (t < kChunks) fetch(0, t);
  if (n > 1 && t >= 64 && t < 64 + kChunks) fetch(1, t - 64);
  if (t == 0) sh.rc = 0;
  CPROF_T();
  griddep_wait();
  CPROF(0);
  for (int k = 0; k < nar; ++k) {  // headers always, data while it fits -> shared memory
    const ArenaEntry e = ar[k];
    if (e.bytes) arena_copy(arena + e.off, e.gbase, e.bytes);
    if (t < (int)(sizeof(Hdr) / 16))
      reinterpret_cast<int4*>(arena + e.hoff)[t] = reinterpret_cast<const int4*>(e.ghdr)[t];
  }
  for (int k = t; k < n; k += kFusedThreads) log[k].st = LOG_NONE;
  __syncthreads();
  // compact vector states and the norms at entry, one thread per header
  auto refresh = [&](int v) {
    const LH h = lean_hdr(reinterpret_cast<const Hdr*>(hbase + kHdrStride * v));
    ls.fh[v] = FH{h.e, h.s, h.bits, h.eff, (int)h.ok};
    return h;
  };
  if (t < nar) {
    const LH h = refresh(t);
    ls.init_e[t] = h.e;
    ls.init_mag[t] = h.mag;  // (only read when ok: a header out of range makes its ops generic)
    ls.lastw[t] = -1;
  }
  __syncthreads();
  CPROF(1);
  LeanState st;
  if (t == 0) ls.op.fast = lean_setup(sh.f[0], n > 1 ? &sh.f[1] : nullptr, ls, log, vid, st);
  CPROF(2);
  CPROF_CNT(8, 1);
  CPROF_CNT(9, n);
  // block header of a vector from the log entry of its last writer (fast ops keep only the
  // compact state current; the generic path and the end of the list need the header)
  auto materialize = [&](int v) {
    const int j = ls.lastw[v];
    if (j < 0) return;
    const LogRec& r = log[j];
    if (r.st == LOG_GENERIC) return;
    Hdr* h = reinterpret_cast<Hdr*>(arena + 128 + kHdrStride * v);
    h->q = r.q;
    h->e = r.e_out;
    h->shift = 0;
    h->max_m = r.mx;
    h->min_m = r.mn;
    h->flags = r.flags;
    h->lam_out = r.lam;
    h->need_recompute = 0;
  };
  for (int i = 0; i < n; ++i) {
    __syncthreads();  // (A) context of op i published; the data of op i - 1 is visible
    CPROF(3);
    FusedOp& f = sh.f[i & 3];
    if (!ls.op.fast) {
      // ---- generic path (bfp_coarse.cuh): setup + gamma, deferred-shift pass, finalize,
      // recompute pass when a flag fires; reads and writes the block headers ----
      if (i + 2 < n && t >= 32 && t < 32 + kChunks) fetch(i + 2, t - 32);
      if (t == 0) {
        for (int v = 0; v < nar; ++v) materialize(v);
#ifdef BFP_LEAN_DEBUG
        if (f.kind == FK_RESTRICT) {
          const int v = vid(f.u.rst.r.hdr), gv = vid(f.p.gamma.t[0].v);
          const Hdr* h = f.u.rst.r.hdr;
          printf("op %d restrict l=%d: in vid %d gamma vid %d lastw %d hdr e=%lld mx=%lld mn=%lld sh=%lld | log st=%d e=%d mx=%d\n",
                 i, f.u.rst.l, v, gv, ls.lastw[v], (long long)h->e, (long long)h->max_m,
                 (long long)h->min_m, (long long)h->shift, ls.lastw[v] >= 0 ? log[ls.lastw[v]].st : -9,
                 ls.lastw[v] >= 0 ? log[ls.lastw[v]].e_out : 0, ls.lastw[v] >= 0 ? log[ls.lastw[v]].mx : 0);
        }
#endif
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
        const int v = vid(f.out.hdr);
        const LH h = refresh(v);
        LogRec& r = log[i];
        r.st = LOG_GENERIC;
        r.e_out = h.e;
        // effective extremes (pending shift applied); a header beyond 32 bits makes every
        // consumer generic, which reads the header itself
        r.mx = (int)(f.out.hdr->max_m >> h.s);
        r.mn = (int)(f.out.hdr->min_m >> h.s);
        ls.lastw[v] = i;
        if (i + 1 < n)
          ls.op.fast = lean_setup(sh.f[(i + 1) & 3], i + 2 < n ? &sh.f[(i + 2) & 3] : nullptr, ls,
                                  log, vid, st);
      }
      CPROF(11);
      continue;
    }
    // ---- fast path ----
    const int kind = ls.op.kind;
    int32_t* st_out = nullptr;  // the workers' copies for the store phase (the control lane
    int st_n4 = 0, st_mm = 0;   // rewrites ls.op for op i + 1 meanwhile)
#ifdef BFP_COARSE_TIMING
    const long long _b0 = clock64();
#endif
    if (warp > 0) {
      const int wt = t - 32;
      if (i + 2 < n && wt < kChunks) fetch(i + 2, wt);
      const LeanOp c = ls.op;
      st_out = c.out;
      st_n4 = c.n4;
      st_mm = c.needmm || c.nnq;
      if (kind == FK_ZERO) {
        for (int g = wt; g < c.n4; g += kLeanWorkers)
          reinterpret_cast<int4*>(c.out)[g] = make_int4(0, 0, 0, 0);
      } else {
        // OR of z ^ sign(z) (mu*), with the sign in bit 63 (all rows in {0, -1}: any -1?)
        uint64_t orv = 0;
        int64_t mx = INT64_MIN, mn = INT64_MAX;
        for (int g = wt; g < c.n4; g += kLeanWorkers) {
          int64_t z[4];
          lean_eval4(c, 4 * g, z);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (c.nnq) z[j] = shift_clamp<int64_t>(z[j], c.lam, c.wout);
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
    }
#ifdef BFP_COARSE_TIMING
    if (t == 479 && i < 4096) {
      g_coarse_ops[4 * i] = kind;
      g_coarse_ops[4 * i + 2] = (int)(clock64() - _b0);
    }
#endif
    CPROF(4);
    __syncthreads();  // (B) warp partials published
    CPROF(5);
    if (warp == 0) {
      LogRec& r = log[i];
      if (kind == FK_ZERO) {
        if (t == 0) {  // zero_vec (P/src/bfp.cpp:53-55)
          r.st = LOG_ZERO;
          r.q = (short)f.q;
          r.e_out = 0;
          r.lam = 0;
          r.mx = r.mn = 0;
          r.flags = 0;
          ls.fh[st.vout] = FH{0, 0, 0, 1, 1};
          ls.lastw[st.vout] = i;
        }
      } else {
        const bool on = lane >= 1 && lane < kCoarseWarps;
        const uint64_t o2 = redux_or64(on ? ls.orv[lane] : 0ull);
        const int mm = ls.op.needmm || ls.op.nnq;
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
          if (st.nnq) {
            lam = 0;  // rows were clamped in the body; e_out = e* + lam_out (:211)
            e_out = st.e_star + ls.op.lam;
            r.st = LOG_FASTN;
            r.gm = st.gm;
            r.ge = st.ge;
            r.mx = (int)tmx;
            r.mn = (int)tmn;
            const int ma = msb32((int)tmx), mb = msb32((int)tmn);
            const int eff = ma > mb ? ma : mb;
            ls.fh[st.vout] = FH{e_out, 0, allzero ? 0 : eff, eff, (int)small_e(e_out)};
          } else {
            mu = bitlen64(mag) + 1;                      // mu* (init 1, P/src/blas.cpp:153)
            if (st.zd > 0 && allzero) mu = 1 - st.zd;    // all-zero anchor in the op's coordinates
            lam = mu - st.w_out;                         // :164
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
            ls.fh[st.vout] = FH{e_out, 0, allzero ? 0 : st.w_out, allzero ? 1 : st.w_out,
                                (int)small_e(e_out)};
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
        for (int g = t - 32; g < st_n4; g += kLeanWorkers) {
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
      ls.op.fast = lean_setup(sh.f[(i + 1) & 3], i + 2 < n ? &sh.f[(i + 2) & 3] : nullptr, ls, log,
                              vid, st);
#ifdef BFP_COARSE_TIMING
      if (i + 1 < 4096) g_coarse_ops[4 * (i + 1) + 1] = (int)(clock64() - _ct);
#endif
    }
    CPROF(2);
  }
  __syncthreads();
  griddep_launch_dependents();
  // ---- end of the list: gamma, flags, trace and history of every fast op, one thread per
  // op (records re-read from global memory: their gamma terms name vectors by arena offset)
  for (int k = t; k < n; k += kFusedThreads) {
    LogRec& r = log[k];
    if (r.st != LOG_FASTQ && r.st != LOG_FASTN) continue;
    const FusedOp& g = ops[k];
    const WinParams& p = g.p;
    auto gvid = [](const Hdr* h) { return (int)(((uintptr_t)h - 128) / kHdrStride); };
    WinCtx c;
    if (r.st == LOG_FASTN) {
      c.gm = r.gm;
      c.ge = r.ge;
      write_trace(p, c, 0, 0, 0, 0);
    } else {
      int gm, ge;
      lean_gamma(p.gamma, ls, log, r.prod, gvid, gm, ge);
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
#ifdef BFP_LEAN_LOGDUMP
  for (int k = t; k < n && k < 1024; k += kFusedThreads) {  // the log of the last launch
    g_coarse_ops[4 * k] = ops[k].kind * 16 + log[k].st;
    g_coarse_ops[4 * k + 1] = log[k].e_out;
    g_coarse_ops[4 * k + 2] = log[k].mx;
    g_coarse_ops[4 * k + 3] = log[k].mn;
  }
#endif
  if (t < nar) materialize(t);
  __syncthreads();
  CPROF(12);
  for (int k = 0; k < nar; ++k) {  // publish the fused part's outputs
    const ArenaEntry e = ar[k];
    if (!e.wb) continue;
    if (e.bytes) arena_copy(e.gbase, arena + e.off, e.bytes);
    if (t < (int)(sizeof(Hdr) / 16))
      reinterpret_cast<int4*>(e.ghdr)[t] = reinterpret_cast<const int4*>(arena + e.hoff)[t];
  }
  CPROF(7);
}
