// bfp_coarse.cuh -- the coarse-level engine: one CTA interprets the op list of the bottom of
// a V-cycle / FMG (every level below the fusion threshold) inside ONE launch.
//
// The drivers (vcycle / ir / fmg, P/src/multigrid.cpp:430-518) run hundreds of windowed ops
// on grids of a few hundred to a few thousand points, where a kernel launch per op costs
// 5-9 us of launch, one-thread setup and finalize latency against < 0.1 us of work.  Here
// the per-op semantics are the SAME device functions as the multi-block kernels (Op::setup,
// win_setup, eval4, win_finalize), so results are bit-identical; what changes is the
// protocol around them:
//   * every block header of the fused levels lives in shared memory for the whole launch
//     (the dependent chain header -> setup -> window -> finalize -> header never leaves the
//     SM); vector data is staged in shared memory too while it fits, else it stays in
//     global memory (L2) behind generic pointers;
//   * op records are prefetched one op ahead into a double buffer;
//   * per op there are two block barriers: (1) window context published / previous data
//     visible, (2) warp partials published.  Between (2) and (1) lane 0 of warp 0 runs the
//     finalize of op i immediately followed by the setup of op i+1 (one serial section, no
//     broadcast in between); warp and cross-warp reductions use redux.sync;
//   * the qcomp recompute pass (rare) is a uniform slow path at the top of the loop.
#pragma once
#include "bfp_kernels.cuh"

namespace bfpdev {

// ---- redux.sync reductions of 64-bit values ---------------------------------------
__device__ __forceinline__ uint64_t redux_or64(uint64_t v) {
  const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)v);
  const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ int64_t redux_max64(int64_t v) {
  const int hi = (int)(v >> 32);
  const int mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? (unsigned)v : 0u);
  return (int64_t)(((uint64_t)(unsigned)mh << 32) | ml);
}
__device__ __forceinline__ int64_t redux_min64(int64_t v) {
  const int hi = (int)(v >> 32);
  const int mh = __reduce_min_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? (unsigned)v : 0xffffffffu);
  return (int64_t)(((uint64_t)(unsigned)mh << 32) | ml);
}

// arena rebasing: pointers of an op record below kArenaMaxBytes are byte offsets into the
// CTA's dynamic shared memory (offset 0 is never used); anything else is a global pointer
__device__ __forceinline__ bool arena_off(const void* p) {
  return (uintptr_t)p != 0 && (uintptr_t)p < (uintptr_t)kArenaMaxBytes;
}
__device__ __forceinline__ void rebase(Vec& v, char* b) {
  if (arena_off(v.data)) v.data = b + (size_t)v.data;
  if (arena_off(v.hdr)) v.hdr = reinterpret_cast<Hdr*>(b + (size_t)v.hdr);
}
__device__ __forceinline__ void rebase_gamma(GammaRule& g, char* b) {
  if (g.literal) return;
  for (int i = 0; i < g.nterms; ++i)
    if (arena_off(g.t[i].v)) g.t[i].v = reinterpret_cast<const Hdr*>(b + (size_t)g.t[i].v);
}
__device__ __forceinline__ void rebase_op(GemvOp& o, char* b) { rebase(o.x, b); rebase(o.y, b); }
__device__ __forceinline__ void rebase_op(JacobiOp& o, char* b) { rebase(o.x, b); rebase(o.b, b); }
__device__ __forceinline__ void rebase_op(ScalOp& o, char* b) { rebase(o.r, b); }
__device__ __forceinline__ void rebase_op(AxpbyOp& o, char* b) { rebase(o.x, b); rebase(o.y, b); }
__device__ __forceinline__ void rebase_op(RestrictOp& o, char* b) { rebase(o.r, b); }
__device__ __forceinline__ void rebase_op(ProlongOp& o, char* b) { rebase(o.xc, b); }
__device__ __forceinline__ void rebase_op(ProlongCorrectOp& o, char* b) {
  rebase(o.ec, b);
  rebase(o.y, b);
}

constexpr int kCoarseWarps = kFusedThreads / 32;

struct CoarseShared {
  FusedOp f[4];  // record ring (the generic engine uses two slots, the lean engine four)
  WinCtx c;
  int64_t need;
  int rc;  // the op just finalized needs its recompute pass
  unsigned long long lo[kCoarseWarps], hi[kCoarseWarps];
  long long mx[kCoarseWarps], mn[kCoarseWarps];
  int err[kCoarseWarps];
};

// one thread: setup of op record f (template exponent, widths, gamma, window)
template <typename M, typename Op>
__device__ __forceinline__ void coarse_setup(Op& op, FusedOp& f, char* ab, CoarseShared& sh) {
  rebase_op(op, ab);
  rebase(f.out, ab);
  rebase_gamma(f.p.gamma, ab);
  int64_t e_star = 0, nd = 0;
  op.setup(e_star, nd);
  WinCtx cc;
  win_setup(f.p, f.out.hdr, e_star, 8 * (int)sizeof(M), cc);
  cc.zd = op_zd(op);
  sh.c = cc;
  sh.need = nd;
}
template <typename M>
__device__ __noinline__ void coarse_prepare(FusedOp& f, char* ab, CoarseShared& sh) {
  switch (f.kind) {
    case FK_GEMV: coarse_setup<M>(f.u.gemv, f, ab, sh); break;
    case FK_JACOBI: coarse_setup<M>(f.u.jac, f, ab, sh); break;
    case FK_SCAL: coarse_setup<M>(f.u.scal, f, ab, sh); break;
    case FK_AXPBY: coarse_setup<M>(f.u.axpby, f, ab, sh); break;
    case FK_RESTRICT: coarse_setup<M>(f.u.rst, f, ab, sh); break;
    case FK_PROLONG: coarse_setup<M>(f.u.pro, f, ab, sh); break;
    case FK_PCORR: coarse_setup<M>(f.u.pc, f, ab, sh); break;
    default: rebase(f.out, ab); break;  // FK_ZERO
  }
}

// every thread: the windowed pass of one op over the output's 4-groups; returns the
// thread's running reductions.  The op record is copied out of shared memory first so its
// fields stay in registers across the (generic-pointer) stores of the loop.
template <typename M, typename Op>
__device__ __forceinline__ void coarse_pass(const Op& sop, const FusedOp& f, int mode,
                                            const CoarseShared& sh, Red& r) {
  Op op = sop;
  const WinCtx c = sh.c;
  const int64_t need = sh.need;
  if (mode == MODE_NNQ)
    grid_body<MODE_NNQ, M, Op, false>(op, f.out, f.p, c, r, need, threadIdx.x, blockDim.x);
  else if (mode == MODE_QCOMP)
    grid_body<MODE_QCOMP, M, Op, false>(op, f.out, f.p, c, r, need, threadIdx.x, blockDim.x);
  else
    grid_body<MODE_RECOMPUTE, M, Op, false>(op, f.out, f.p, c, r, need, threadIdx.x, blockDim.x);
}
template <typename M>
__device__ __noinline__ void coarse_body(const FusedOp& f, int mode, const CoarseShared& sh,
                                         Red& r) {
  switch (f.kind) {
    case FK_GEMV: coarse_pass<M>(f.u.gemv, f, mode, sh, r); break;
    case FK_JACOBI: coarse_pass<M>(f.u.jac, f, mode, sh, r); break;
    case FK_SCAL: coarse_pass<M>(f.u.scal, f, mode, sh, r); break;
    case FK_AXPBY: coarse_pass<M>(f.u.axpby, f, mode, sh, r); break;
    case FK_RESTRICT: coarse_pass<M>(f.u.rst, f, mode, sh, r); break;
    case FK_PROLONG: coarse_pass<M>(f.u.pro, f, mode, sh, r); break;
    case FK_PCORR: coarse_pass<M>(f.u.pc, f, mode, sh, r); break;
    default: {  // FK_ZERO: zero_vec (P/src/bfp.cpp:53-55)
      M* d = (M*)f.out.data;
      for (int64_t o = threadIdx.x; o < f.out.n; o += blockDim.x) d[o] = 0;
    }
  }
}

// warp partials of the running reductions -> shared memory
__device__ __forceinline__ void coarse_publish(const Red& r, CoarseShared& sh) {
  const uint64_t lo = redux_or64(r.olo), hi = redux_or64(r.ohi);
  const int64_t mx = redux_max64(r.mx), mn = redux_min64(r.mn);
  const int err = __reduce_or_sync(0xffffffffu, r.err);
  if ((threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    sh.lo[w] = lo;
    sh.hi[w] = hi;
    sh.mx[w] = mx;
    sh.mn[w] = mn;
    sh.err[w] = err;
  }
}
// warp 0: the block totals from the warp partials (valid in every lane)
__device__ __forceinline__ void coarse_totals(const CoarseShared& sh, int& bits, int64_t& mx,
                                              int64_t& mn, int& err) {
  const int lane = threadIdx.x & 31;
  const bool on = lane < kCoarseWarps;
  const uint64_t lo = redux_or64(on ? sh.lo[lane] : 0ull), hi = redux_or64(on ? sh.hi[lane] : 0ull);
  mx = redux_max64(on ? sh.mx[lane] : INT64_MIN);
  mn = redux_min64(on ? sh.mn[lane] : INT64_MAX);
  err = __reduce_or_sync(0xffffffffu, on ? sh.err[lane] : 0);
  bits = mu_bits(lo, hi);
}

__device__ __forceinline__ void arena_copy(char* dst, const char* src, int64_t bytes) {
  const int64_t n16 = bytes >> 4;
  for (int64_t i = threadIdx.x; i < n16; i += blockDim.x)
    reinterpret_cast<int4*>(dst)[i] = reinterpret_cast<const int4*>(src)[i];
}

}  // namespace bfpdev

// measurement builds (-DBFP_COARSE_TIMING): thread 0's clock64 per phase, summed over launches
#ifdef BFP_COARSE_TIMING
__device__ long long g_coarse_prof[16];
__device__ int g_coarse_ops[4096 * 4];  // per op of the last launch: kind, prepare, body, finalize clk
#define CPROF_OP(i, j, v) \
  if (threadIdx.x == 0 && (i) < 4096) g_coarse_ops[4 * (i) + (j)] = (int)(v)
#define CPROF_T() long long _ct = clock64()
#define CPROF(k)                                                    \
  if (threadIdx.x == 0) {                                           \
    const long long _n = clock64();                                 \
    atomicAdd((unsigned long long*)&g_coarse_prof[k], (unsigned long long)(_n - _ct)); \
    _ct = _n;                                                       \
  }
#define CPROF_CNT(k, v) \
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)&g_coarse_prof[k], (unsigned long long)(v))
#else
#define CPROF_T()
#define CPROF(k)
#define CPROF_CNT(k, v)
#define CPROF_OP(i, j, v)
#endif

template <typename M>
__global__ void __launch_bounds__(kFusedThreads) coarse_kernel(const FusedOp* ops, int n,
                                                               const ArenaEntry* ar, int nar) {
  extern __shared__ __align__(128) char arena[];
  __shared__ __align__(16) CoarseShared sh;
  constexpr int kChunks = (int)(sizeof(FusedOp) / 16);
  static_assert(sizeof(FusedOp) % 16 == 0, "FusedOp staging copies 16-byte granules");
  static_assert(kChunks <= kFusedThreads, "one prefetch chunk per thread");
  const int t = threadIdx.x;
  // op 0's record does not depend on the previous kernel: fetch it before the wait
  if (t < kChunks)
    reinterpret_cast<int4*>(&sh.f[0])[t] = __ldg(reinterpret_cast<const int4*>(&ops[0]) + t);
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
  __syncthreads();
  CPROF(1);
  if (t == 0) coarse_prepare<M>(sh.f[0], arena, sh);
  CPROF(2);
  CPROF_CNT(8, 1);
  CPROF_CNT(9, n);
  int i = 0;
  while (true) {
    __syncthreads();  // (1) window context of op i published; earlier data visible
    CPROF(3);
    if (sh.rc) {
      // qcomp recompute pass of op i - 1 (a flag fired): floor(z / 2^lam_out) from the
      // still-live inputs (P/src/blas.cpp:170-176)
      FusedOp& f = sh.f[(i - 1) & 1];
      __syncthreads();  // everyone has read rc
      if (t == 0) {
        f.p.mode = MODE_RECOMPUTE;
        WinCtx c2;
        win_setup(f.p, f.out.hdr, sh.c.e_star, 8 * (int)sizeof(M), c2);
        sh.c = c2;
        sh.rc = 0;
      }
      __syncthreads();
      Red r;
      r.init();
      if (!sh.c.skip) coarse_body<M>(f, MODE_RECOMPUTE, sh, r);
      coarse_publish(r, sh);
      __syncthreads();
      if (t < 32) {
        int bits, err;
        int64_t mx, mn;
        coarse_totals(sh, bits, mx, mn, err);
        if (t == 0) {
          if (!sh.c.skip) win_finalize(f.p, sh.c, f.out.hdr, bits, mx, mn, err);
          if (i < n) coarse_prepare<M>(sh.f[i & 1], arena, sh);
        }
      }
      continue;
    }
    if (i >= n) break;
    FusedOp& f = sh.f[i & 1];
    const bool pre = i + 1 < n && t < kChunks;
    int4 nx = make_int4(0, 0, 0, 0);
    if (pre) nx = __ldg(reinterpret_cast<const int4*>(&ops[i + 1]) + t);  // next record
    const int kind = f.kind, mode = f.p.mode;
    Red r;
    r.init();
#ifdef BFP_COARSE_TIMING
    const long long _b0 = clock64();
#endif
    coarse_body<M>(f, mode, sh, r);
#ifdef BFP_COARSE_TIMING
    CPROF_OP(i, 0, kind);
    CPROF_OP(i, 2, clock64() - _b0);
#endif
    CPROF(4);
    if (kind != FK_ZERO) coarse_publish(r, sh);
    if (pre) reinterpret_cast<int4*>(&sh.f[(i + 1) & 1])[t] = nx;
    __syncthreads();  // (2) warp partials and the next record published
    CPROF(5);
    if (t < 32) {
      int bits = 1, err = 0;
      int64_t mx = 0, mn = 0;
      if (kind != FK_ZERO) coarse_totals(sh, bits, mx, mn, err);
      if (t == 0) {
        int rc = 0;
        if (kind == FK_ZERO) {
          Hdr* h = f.out.hdr;
          h->q = f.q;
          h->e = 0;
          h->shift = 0;
          h->max_m = 0;
          h->min_m = 0;
          h->flags = 0;
          h->need_recompute = 0;
        } else {
          rc = win_finalize(f.p, sh.c, f.out.hdr, bits, mx, mn, err);
        }
#ifdef BFP_COARSE_TIMING
        CPROF_OP(i, 3, clock64() - _ct);
#endif
        CPROF(6);
        if (rc)
          sh.rc = 1;
        else if (i + 1 < n)
          coarse_prepare<M>(sh.f[(i + 1) & 1], arena, sh);
#ifdef BFP_COARSE_TIMING
        CPROF_OP(i + 1, 1, clock64() - _ct);
#endif
        CPROF(2);
      }
    }
    ++i;
  }
  griddep_launch_dependents();
  for (int k = 0; k < nar; ++k) {  // publish the fused part's outputs
    const ArenaEntry e = ar[k];
    if (!e.wb) continue;
    if (e.bytes) arena_copy(e.gbase, arena + e.off, e.bytes);
    if (t < (int)(sizeof(Hdr) / 16))
      reinterpret_cast<int4*>(e.ghdr)[t] = reinterpret_cast<const int4*>(arena + e.hoff)[t];
  }
  CPROF(7);
}
