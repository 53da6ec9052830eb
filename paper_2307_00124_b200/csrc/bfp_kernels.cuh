// bfp_kernels.cuh -- kernel templates (windowed passes over grids: generic grid
// kernel, register march, bulk-async smem pipeline, fused CTA, flat rows) and their
// host launchers.  Included by the op translation units (op_*.cu) and bfp_lib.cu so
// the instantiations compile in parallel.
#pragma once
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "bfp_bulk.cuh"
#include "bfp_internal.h"

namespace bfp {
// process-wide switches and measurement hooks (defined in bfp_lib.cu)
extern bool g_pdl;             // programmatic dependent launch for the windowed kernels
extern bool g_skip_recompute;  // measurement only: pass 1 alone (flags must be clear)
extern bool g_prof;            // CUDA-event brackets around pass-1 launches
extern bool g_use_bulk;        // 2-D stencils through the bulk-async pipeline
std::pair<cudaEvent_t, cudaEvent_t> prof_pair();
// the one-thread finalize of a deferred multi-block pass 1 (bfp_lib.cu)
int launch_deferred_finalize(const bfpdev::Vec& out, const bfpdev::WinParams& p, int storage_bits,
                             cudaStream_t s);
// pass 1 on more than one block finalizes through the deferred kernel (not multi-rank
// partials, which have their own finalize)
inline int defer_ok(const bfpdev::WinParams& p, int blocks) {
  return blocks > 1 && p.part == nullptr && p.mode != bfpdev::MODE_RECOMPUTE;
}

constexpr int kThreads = 256;
constexpr int kMaxDev = 64;
// current device (index into the per-device caches below)
inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d >= 0 && d < kMaxDev ? d : 0;
}
// One value per device, computed once (thread-safe): function attributes and occupancy
// are per device, so every launcher caches them through this.
template <typename F> inline int per_device(std::atomic<int>* slots, F make) {
  const int d = cur_device();
  int v = slots[d].load(std::memory_order_acquire);
  if (v) return v;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  v = slots[d].load(std::memory_order_relaxed);
  if (!v) {
    v = make();
    slots[d].store(v, std::memory_order_release);
  }
  return v;
}
// streaming multiprocessors of the current device (148 on B200)
inline int sm_count() {
  static std::atomic<int> c[kMaxDev];
  return per_device(c, [] {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, cur_device());
    return v > 0 ? v : 148;
  });
}
inline int max_blocks() { return sm_count() * 8; }
#ifndef BFP_B2_EARLY  // 2-D bulk pipeline: first item's loads issued before the op setup (A/B)
#define BFP_B2_EARLY 1
#endif
#ifndef BFP_SETUP_PREFETCH  // warp-parallel header prefetch before the one-thread setup (A/B)
#define BFP_SETUP_PREFETCH 1
#endif
#ifndef BFP_GRID_SPLIT  // int32-storage split window in the grid kernel (A/B switch)
#define BFP_GRID_SPLIT 1
#endif
#ifndef BFP_GRID_UNROLL  // groups per grid-loop iteration (A/B switch)
#define BFP_GRID_UNROLL 1
#endif

// Launch with Programmatic Dependent Launch: the grid may be scheduled while the
// previous kernel in the stream drains; the kernel executes griddepcontrol.wait
// before touching any data, so stream semantics are unchanged.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}
// smallest level a pipelined (bulk / TMA) kernel takes over from the generic grid kernel;
// BFP_<NAME> in the environment overrides the default (A/B measurements)
inline int min_level(const char* name, int def) {
#ifdef BFP_AB_ENV  // A/B measurement builds only: product builds ignore the environment
  const char* v = getenv(name);
  return v ? atoi(v) : def;
#else
  (void)name;
  return def;
#endif
}
// March depth R (planes per work item) of a one-wave plane march over `units` tiles x NZ
// planes on `ctas` resident CTAs, items handed out round robin (item = unit + chunk *
// units, CTA b takes b, b + ctas, ...).  R = ceil(units NZ / ctas) minimises the item
// count but can leave a short last chunk on a second round for some CTAs (C4: R = 222
// gives 290 planes on the busiest CTA against 221 on average); this picks, among the
// chunk counts 1..64, the R (a multiple of `step`, >= Rmin) with the smallest busiest-CTA
// load, counting `ovh` planes per item for the march prologue.  BFP_MARCH_BALANCE=0 in
// the environment restores the plain R (A/B).
inline int march_R(int64_t units, int64_t NZ, int64_t ctas, int Rmin, int step, int ovh) {
  auto plain = [&] {
    int64_t R = std::max<int64_t>(Rmin, (units * NZ + ctas - 1) / ctas);
    return (int)((R + step - 1) / step * step);
  };
  static const bool on = [] {
#ifdef BFP_AB_ENV
    const char* v = getenv("BFP_MARCH_BALANCE");
    return !(v && v[0] == '0');
#else
    return true;
#endif
  }();
  if (!on || units <= 0 || NZ <= 0) return plain();
  struct Key {
    int64_t u, nz, c;
    int rm, st, ov, R;
  };
  static Key cache[64];
  static int ncache = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < ncache; ++i)
    if (cache[i].u == units && cache[i].nz == NZ && cache[i].c == ctas && cache[i].rm == Rmin &&
        cache[i].st == step && cache[i].ov == ovh)
      return cache[i].R;
  auto makespan = [&](int64_t R) {
    const int64_t nc = (NZ + R - 1) / R, items = units * nc, last = NZ - (nc - 1) * R;
    const int64_t L0 = (nc - 1) * units;  // first item of the last chunk
    int64_t worst = 0;
    for (int64_t b = 0; b < std::min(items, ctas); ++b) {
      const int64_t cnt = (items - 1 - b) / ctas + 1;
      const int64_t jmin = b >= L0 ? 0 : (L0 - b + ctas - 1) / ctas;
      const int64_t nlast = std::max<int64_t>(0, cnt - jmin);
      worst = std::max(worst, cnt * (R + ovh) - nlast * (R - last));
    }
    return worst;
  };
  int64_t bestR = plain(), best = makespan(bestR);
  for (int64_t nc = 1; nc <= 64; ++nc) {
    int64_t R = std::max<int64_t>(Rmin, (NZ + nc - 1) / nc);
    R = (R + step - 1) / step * step;
    const int64_t m = makespan(R);
    if (m < best) best = m, bestR = R;
  }
  if (ncache < 64) cache[ncache++] = Key{units, NZ, ctas, Rmin, step, ovh, (int)bestR};
  return (int)bestR;
}
inline int blocks_for(int64_t work) {
  int64_t b = (work + kThreads - 1) / kThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, max_blocks()));
}
inline int last_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "bfpmg_b200: launch failed: %s\n", cudaGetErrorString(e));
    return BFP_ERR_CUDA;
  }
  return BFP_OK;
}
}  // namespace bfp

// measurement builds (-DBFP_TIMING): thread 0 of block 0 of each grid_win_kernel launch
// records %globaltimer at its phase boundaries into bfp_dbg_stamps (bfp_lib.cu)
#ifdef BFP_TIMING
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BFP_STAMP(k)                                                         \
  long long _st##k = (threadIdx.x == 0 && blockIdx.x == 0) ? gtimer() : 0;  \
  (void)_st##k
#define BFP_STAMP_END()                                                                \
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.dbg) {                                  \
    unsigned i = atomicAdd(reinterpret_cast<unsigned*>(p.dbg), 1u) % 4095 + 1;          \
    long long* d = p.dbg + 8 * i;                                                      \
    d[0] = _st0; d[1] = _st1; d[2] = _st2; d[3] = _st3; d[4] = _st4; d[6] = gtimer();   \
  }
#else
#define BFP_STAMP(k)
#define BFP_STAMP_END()
#endif

using namespace bfpdev;
using bfp::kThreads;
using bfp::launch_pdl;


template <typename M> struct Lim;
template <> struct Lim<int32_t> {
  static constexpr int32_t lo = INT32_MIN, hi = INT32_MAX;
};
template <> struct Lim<int64_t> {
  static constexpr int64_t lo = INT64_MIN, hi = INT64_MAX;
};

// The window pass over 4-groups of the output storage.  MODE is a template
// parameter so each instantiation carries only its own epilogue:
//   QCOMP      OR-accumulate |z| bits (mu*), store floor(z/2^lam_tmp)
//   RECOMPUTE  store floor(z/2^lam_out)
//   NNQ        store clamp(floor(z/2^lam_out))
// Max/min of the STORED values are tracked in the storage type.
// SP (int32 storage, GemvOp::eval4_sp): the split window of bulk3_loop -- the stored value
// t = floor(z / 2^rs) and the low word zl in 64-bit arithmetic, mu* from t (+ rs) or zl.
template <int MODE, typename M, typename Op>
__device__ __forceinline__ void grid_loop_sp(Op& op, const Vec& out, const WinCtx& c, Red& r,
                                             int64_t g0, int64_t stride) {
  const int64_t ngroups = out.n >> 2;
  const SplitWin sw = split_win(op.d, c.rs);
  M mx = Lim<M>::lo, mn = Lim<M>::hi;
  uint64_t ot = 0, oz = 0;
  auto epi = [&](int64_t g, const int64_t t[4], const int64_t zl[4]) {
    M tt[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (MODE == MODE_QCOMP) {
        const uint64_t sg = (uint64_t)(t[j] >> 63);
        ot |= (uint64_t)t[j] ^ sg;
        oz |= (uint64_t)zl[j] ^ sg;
      }
      tt[j] = (M)t[j];
      mx = tt[j] > mx ? tt[j] : mx;
      mn = tt[j] < mn ? tt[j] : mn;
    }
    V4<M>::store(out, g * 4, tt);
  };
  for (int64_t g = g0; g < ngroups; g += stride) {
    int64_t t[4], zl[4];
    op.template eval4_sp<true>(g * 4, sw, t, zl);
    epi(g, t, zl);
  }
  if (MODE == MODE_QCOMP) {
    const int rs = c.rs;
    if (ot) {
      r.olo |= ot << rs;
      r.ohi |= rs ? ot >> (64 - rs) : 0;
    } else {
      r.olo |= oz;
    }
  }
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

// Pointwise ops on int32 storage, fast window (qcomp pass 1 / recompute with 0 <= rs < 32):
// several groups per thread and iteration with all their loads issued first (64 bytes in
// flight per thread: one group per iteration left the generic loop latency-bound at ~0.75
// of HBM), rows from 32-bit operands (IMAD.WIDE), funnel-shift store, 32-bit OR pair.
template <int MODE, typename Op>
__device__ __forceinline__ void grid_loop_pt(Op& op, const Vec& out, const WinCtx& c, Red& r,
                                             int64_t g0, int64_t stride) {
  const int64_t ngroups = out.n >> 2;
  int32_t* O = (int32_t*)out.data;
  int mx = INT32_MIN, mn = INT32_MAX;
  uint32_t olo = 0, ohi = 0;
  const int rs = c.rs;
  auto epi = [&](int64_t g, const typename Op::Raw& w) {
    int64_t z[4];
    op.point4(w, z);
    int t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t zl = (uint32_t)z[j], zh = (uint32_t)((uint64_t)z[j] >> 32);
      if (MODE == MODE_QCOMP) {
        const uint32_t sg = (uint32_t)((int)zh >> 31);
        olo |= zl ^ sg;
        ohi |= zh ^ sg;
      }
      t[j] = (int)__funnelshift_r(zl, zh, rs);
      mx = t[j] > mx ? t[j] : mx;
      mn = t[j] < mn ? t[j] : mn;
    }
    *reinterpret_cast<int4*>(O + 4 * g) = make_int4(t[0], t[1], t[2], t[3]);
  };
  constexpr int U = Op::kPointUnroll;  // groups in flight per thread (per operand)
  int64_t g = g0;
  for (; g + (U - 1) * stride < ngroups; g += U * stride) {
    typename Op::Raw w[U];
#pragma unroll
    for (int k = 0; k < U; ++k) w[k] = op.point_load(4 * (g + k * stride));
#pragma unroll
    for (int k = 0; k < U; ++k) epi(g + k * stride, w[k]);
  }
  for (; g < ngroups; g += stride) epi(g, op.point_load(4 * g));
  r.olo |= ((uint64_t)ohi << 32) | olo;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

template <int MODE, typename M, typename Op, typename A, bool NC = true>
__device__ __forceinline__ void grid_loop(Op& op, const Vec& out, const WinParams& p,
                                          const WinCtx& c, Red& r, int64_t g0, int64_t stride) {
  const int64_t ngroups = out.n >> 2;
  M mx = Lim<M>::lo, mn = Lim<M>::hi;
  uint64_t olo = 0, ohi = 0;
  const bool store = c.store_tmp;
  auto epi = [&](int64_t g, A z[4]) {
    M t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (MODE == MODE_NNQ) {
        t[j] = (M)shift_clamp<A>(z[j], c.lam, p.w_out);
      } else {
        if (MODE == MODE_QCOMP) or_mag<A>(z[j], olo, ohi);
        t[j] = store ? store_shift<M, A>(z[j], c) : (M)0;
      }
      mx = t[j] > mx ? t[j] : mx;
      mn = t[j] < mn ? t[j] : mn;
    }
    V4<M>::store(out, g * 4, t);
  };
#if BFP_GRID_UNROLL > 1
  // two groups per iteration: the second group's loads are issued before the first
  // group's epilogue (more bytes in flight per thread)
  int64_t g = g0;
  for (; g + stride < ngroups; g += 2 * stride) {
    A z0[4], z1[4];
    op.template eval4<M, A, NC>(g * 4, z0);
    op.template eval4<M, A, NC>((g + stride) * 4, z1);
    epi(g, z0);
    epi(g + stride, z1);
  }
  if (g < ngroups) {
    A z[4];
    op.template eval4<M, A, NC>(g * 4, z);
    epi(g, z);
  }
#else
  for (int64_t g = g0; g < ngroups; g += stride) {
    A z[4];
    op.template eval4<M, A, NC>(g * 4, z);
    epi(g, z);
  }
#endif
  r.olo |= olo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;  // sentinels stay neutral
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

// SPLIT: the grid kernel's own body may take the split window; the pipelines' exact
// fallbacks do not (it would only add registers to their hot loops)
// (g0, stride): the groups this thread owns -- by default the launch grid's; a block that runs
// an op alone passes its own (grid_finish_kernel)
template <int MODE, typename M, typename Op, bool NC = true, bool SPLIT = false>
__device__ __forceinline__ void grid_body(Op& op, const Vec& out, const WinParams& p,
                                          const WinCtx& c, Red& r, int64_t need,
                                          int64_t g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                                          int64_t stride = (int64_t)gridDim.x * blockDim.x) {
  if constexpr (SPLIT && HasSplit<Op>::value && sizeof(M) == 4 && NC && MODE != MODE_NNQ) {
    // int32 storage beyond the narrow path (1-D fine levels: A x sits 2l bits above b)
    if (BFP_GRID_SPLIT && !op.narrow && need <= 127 && op.sp32 && c.store_tmp && c.ls == 0 &&
        c.rs < 64 && need - c.rs <= 63) {
      grid_loop_sp<MODE, M, Op>(op, out, c, r, g0, stride);
      return;
    }
  }
  if constexpr (SPLIT && HasPoint<Op>::value && sizeof(M) == 4 && NC && MODE != MODE_NNQ) {
    if (op.p32 && need <= 63 && c.store_tmp && c.ls == 0 && c.rs < 32) {
      grid_loop_pt<MODE, Op>(op, out, c, r, g0, stride);
      return;
    }
  }
  if (need > 127)
    r.err = ERR_WIDTH;
  else if (need <= 63)
    grid_loop<MODE, M, Op, int64_t, NC>(op, out, p, c, r, g0, stride);
  else
    grid_loop<MODE, M, Op, i128, NC>(op, out, p, c, r, g0, stride);
}

// One windowed pass over a grid (or 4-padded flat) output: qcomp pass 1,
// nnqcomp, or the qcomp recompute pass, selected by p.mode.
// The op setup and the gamma rule are uniform per launch: one thread evaluates
// them from the device headers and broadcasts through shared memory.
// The block headers an op's setup reads (published state: the first 64 bytes of each).
__device__ __forceinline__ int op_hdrs(const GemvOp& o, const Hdr** h) { h[0] = o.x.hdr, h[1] = o.y.hdr; return 2; }
__device__ __forceinline__ int op_hdrs(const JacobiOp& o, const Hdr** h) { h[0] = o.x.hdr, h[1] = o.b.hdr; return 2; }
__device__ __forceinline__ int op_hdrs(const AxpbyOp& o, const Hdr** h) { h[0] = o.x.hdr, h[1] = o.y.hdr; return 2; }
__device__ __forceinline__ int op_hdrs(const ProlongCorrectOp& o, const Hdr** h) { h[0] = o.ec.hdr, h[1] = o.y.hdr; return 2; }
__device__ __forceinline__ int op_hdrs(const CsrGemvOp& o, const Hdr** h) { h[0] = o.x.hdr, h[1] = o.y.hdr; return 2; }
__device__ __forceinline__ int op_hdrs(const ScalOp& o, const Hdr** h) { h[0] = o.r.hdr; return 1; }
__device__ __forceinline__ int op_hdrs(const RestrictOp& o, const Hdr** h) { h[0] = o.r.hdr; return 1; }
__device__ __forceinline__ int op_hdrs(const ProlongOp& o, const Hdr** h) { h[0] = o.xc.hdr; return 1; }
__device__ __forceinline__ int op_hdrs(const CsrSpmvOp& o, const Hdr** h) { h[0] = o.x.hdr; return 1; }
template <typename Op> __device__ __forceinline__ int op_hdrs(const Op&, const Hdr**) { return 0; }

// Warp 0 pulls the headers the one-thread setup will read (the op's operands and the
// gamma rule's norm terms) into L1 with one parallel round trip; thread 0's setup then
// runs on L1 hits instead of a chain of dependent L2 reads.
template <typename Op>
__device__ __forceinline__ void prefetch_setup_hdrs(const Op& op, const WinParams& p) {
  const int lane = threadIdx.x & 31;
  const Hdr* h[8];
  int n = op_hdrs(op, h);
  if (!p.gamma.literal)
    for (int i = 0; i < p.gamma.nterms && i < 3; ++i)
      if (p.gamma.t[i].v) h[n++] = p.gamma.t[i].v;
  if (lane < 2 * n) {  // sectors 0 and 1 (q, e, shift, max_m, min_m, ...) of header lane/2
    const int64_t* a = (const int64_t*)h[lane >> 1] + (lane & 1) * 4;
    int64_t v;
    asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    (void)v;
  }
}

template <typename Op, typename M>
__device__ __forceinline__ void block_setup(Op& op, const Vec& out, const WinParams& p, WinCtx& c,
                                            int64_t& need) {
  __shared__ Op s_op;
  __shared__ WinCtx s_c;
  __shared__ int64_t s_need;
  if (p.mode == MODE_RECOMPUTE) {  // fast path: nothing to do, skip the op setup
    __shared__ int s_rc;
    if (threadIdx.x == 0) s_rc = ((volatile Hdr*)out.hdr)->need_recompute;
    __syncthreads();
    if (!s_rc) {
      c.skip = 1;
      return;
    }
  }
#if BFP_SETUP_PREFETCH
  if (threadIdx.x < 32) prefetch_setup_hdrs(op, p);
#endif
  if (threadIdx.x == 0) {
    int64_t e_star = 0, nd = 0;
    Op o = op;
    o.setup(e_star, nd);
    WinCtx cc;
    win_setup(p, out.hdr, e_star, 8 * (int)sizeof(M), cc);
    cc.zd = op_zd(o);
    s_op = o;
    s_c = cc;
    s_need = nd;
  }
  __syncthreads();
  op = s_op;
  c = s_c;
  need = s_need;
}

template <int MODE, typename M, typename Op>
__global__ void __launch_bounds__(kThreads) grid_win_kernel(Op op, Vec out, WinParams p) {
  BFP_STAMP(0);
  griddep_wait();
  BFP_STAMP(1);
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, M>(op, out, p, c, need);
  BFP_STAMP(2);
  if (c.skip) return;
  Red r;
  r.init();
  grid_body<MODE, M, Op, true, true>(op, out, p, c, r, need);
  BFP_STAMP(3);
  if (MODE != MODE_QCOMP || gridDim.x != 1 || p.part) griddep_launch_dependents();
  __shared__ int s_rc;  // single block: thread 0's finalize verdict (need_recompute)
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    s_rc = win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
  BFP_STAMP(4);
  if constexpr (MODE == MODE_QCOMP) {
    // a single-block qcomp runs its recompute pass in the same launch (no second kernel);
    // the fast path decides from shared memory, without re-reading the header
    if (gridDim.x == 1 && !p.part) {
      __syncthreads();  // header finalized by thread 0
      if (!s_rc) {
        BFP_STAMP(5);
        griddep_launch_dependents();
        BFP_STAMP_END();
        return;
      }
      WinParams p2 = p;
      p2.mode = MODE_RECOMPUTE;
      WinCtx c2;
      win_setup(p2, out.hdr, c.e_star, 8 * (int)sizeof(M), c2);
      if (!c2.skip) {
        Red r2;
        r2.init();
        grid_body<MODE_RECOMPUTE, M>(op, out, p2, c2, r2, need);
        reduce_and_finalize(r2, out.hdr, [&](int bits, int64_t mx, int64_t mn, int err) {
          win_finalize(p2, c2, out.hdr, bits, mx, mn, err);
        });
      }
      BFP_STAMP(5);
      griddep_launch_dependents();
    }
  }
  BFP_STAMP_END();
}


// Finish of a multi-block qcomp pass 1 on a mid-size grid, in ONE small launch: thread 0
// applies the deferred finalize (the blocks' accumulated {OR, max, min, err} and block 0's
// window context -> win_finalize); only when a flag fired does this block run the recompute
// pass over the whole vector itself (rare; a few tens of microseconds on these sizes).  It
// replaces the one-thread finalize kernel plus the full-grid recompute launch that exits
// after one header read: one dependent launch boundary less on every such op.
template <typename M, typename Op>
__global__ void __launch_bounds__(kThreads) grid_finish_kernel(Op op, Vec out, WinParams p) {
  griddep_wait();
  __shared__ int s_rc;
  if (threadIdx.x == 0) s_rc = deferred_finalize(out, p, 8 * (int)sizeof(M));
  __syncthreads();
  if (!s_rc) return;
  WinParams p2 = p;
  p2.mode = MODE_RECOMPUTE;
  p2.defer = 0;
  int64_t need = 0;
  WinCtx c2;
  block_setup<Op, M>(op, out, p2, c2, need);
  if (c2.skip) return;
  Red r2;
  r2.init();
  grid_body<MODE_RECOMPUTE, M, Op>(op, out, p2, c2, r2, need, threadIdx.x, blockDim.x);
  const BlockRed b = block_reduce(r2);
  if (threadIdx.x == 0) win_finalize(p2, c2, out.hdr, mu_bits(b.lo, b.hi), b.mx, b.mn, b.err);
}

// ---------------------------------------------------------------------------
// 2.5-D register march for the 2-D / 3-D stencil ops on int32 storage (the
// hot path).  A work item is a 4-wide x strip marching R steps along the
// slowest axis (y in 2-D, z in 3-D): the x values at the previous / current /
// next step stay in registers, x-neighbours come from warp shuffles, and the
// loads of step s+1 are issued before step s is computed.  Each thread writes
// one aligned int4 per step.
constexpr int kMarchMinN = 128;  // GX = N/4 >= 32: a warp spans one row

__device__ __forceinline__ void ld4s(const int32_t* p, int64_t o, int sh, int v[4]) {
  // 128-bit read-only load of 4 mantissas, pending shift applied
  int4 t = __ldg(reinterpret_cast<const int4*>(p + o));
  v[0] = t.x >> sh;
  v[1] = t.y >> sh;
  v[2] = t.z >> sh;
  v[3] = t.w >> sh;
}

// one march step: output row at wp from (P, C, Nx) along the march axis and the
// x neighbours through the warp; prefetches the next step into (NN, Yn, ...).
template <int MODE, int DIM, bool SW, typename Op>
struct MarchStep {
  const Op& op;
  const WinParams& p;
  const WinCtx& c;
  int64_t S, N;
  int sx, sy, lane;
  bool xpad, store;
  int32_t mx, mn;
  uint64_t olo, ohi;

  __device__ __forceinline__ void prefetch(const int32_t* xp, const int32_t* yp, int NN[4],
                                           int Yn[4], int SUn[4], int SDn[4], int& lfn,
                                           int& rtn) const {
    ld4s(xp, 2 * S, sx, NN);
    ld4s(yp, S, sy, Yn);
    if (DIM == 3) {
      ld4s(xp, S - N, sx, SUn);
      ld4s(xp, S + N, sx, SDn);
    }
    if (lane == 0) lfn = __ldg(xp + S - 1) >> sx;
    if (lane == 31) rtn = __ldg(xp + S + 4) >> sx;
  }

  __device__ __forceinline__ void compute(int32_t* wp, const int P[4], const int C[4],
                                          const int Nx[4], const int Y[4], const int SU[4],
                                          const int SD[4], int lf, int rt) {
    int left = __shfl_up_sync(0xffffffffu, C[3], 1);
    int right = __shfl_down_sync(0xffffffffu, C[0], 1);
    if (lane == 0) left = lf;
    if (lane == 31) right = rt;
    const int nb[4] = {left + C[1], C[0] + C[2], C[1] + C[3], C[2] + right};
    int32_t tt[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int n = nb[k] + P[k] + Nx[k];
      if (DIM == 3) n += SU[k] + SD[k];
      const int g = 2 * DIM * C[k] - n;
      int64_t z = op.template point_t<SW>(g, C[k], Y[k]);
      if (k == 3 && xpad) z = 0;
      if (MODE == MODE_NNQ) {
        tt[k] = (int32_t)shift_clamp<int64_t>(z, c.lam, p.w_out);
      } else {
        if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
        tt[k] = store ? store_shift<int32_t, int64_t>(z, c) : 0;
      }
      mx = tt[k] > mx ? tt[k] : mx;
      mn = tt[k] < mn ? tt[k] : mn;
    }
    *reinterpret_cast<int4*>(wp) = make_int4(tt[0], tt[1], tt[2], tt[3]);
  }
};

template <int MODE, int DIM, bool SW, typename Op>
__device__ __forceinline__ void march_loop(const Op& op, const Vec& out, const WinParams& p,
                                           const WinCtx& c, Red& r, int R) {
  const int l = out.l;
  const int64_t N = (int64_t)1 << l, GX = N >> 2;
  const int64_t S = DIM == 2 ? N : N * N;  // march stride
  const int64_t rows = DIM == 3 ? N : 1;
  const int64_t NZ = out.nz, Z0 = out.z0;  // local planes along the march axis, slab offset
  const int64_t chunks = (NZ + R - 1) / R;
  const int64_t items = GX * rows * chunks;
  MarchStep<MODE, DIM, SW, Op> st{op, p, c, S, N, op.shs(), op.shy(), (int)(threadIdx.x & 31),
                              false, (bool)c.store_tmp, INT32_MIN, INT32_MAX, 0, 0};
  const int sx = st.sx, sy = st.sy;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < items; w += stride) {
    const int64_t gx = w % GX, t = w / GX;
    const int64_t j = DIM == 3 ? t % N : 0, ch = DIM == 3 ? t / N : t;
    const int m0 = (int)(ch * R);
    const int64_t o0 = gx * 4 + (DIM == 3 ? j * N : 0) + (int64_t)m0 * S;
    const int32_t* xp = (const int32_t*)op.sv().data + o0;
    const int32_t* yp = (const int32_t*)op.yv2().data + o0;
    int32_t* wp = (int32_t*)out.data + o0;
    st.xpad = gx == GX - 1;
    // the pad plane / row (index N-1 of the march axis, or row N-1 in 3-D) is written as zeros
    const int total = (int)std::min<int64_t>(R, NZ - m0);
    const bool rowpad = DIM == 3 && j == N - 1;
    const bool padplane = Z0 + m0 + total == N;  // last local plane is the global pad plane
    const int steps = rowpad ? 0 : (padplane ? total - 1 : total);
    if (rowpad || padplane) {
      const int first = rowpad ? 0 : total - 1;
      for (int s = first; s < total; ++s)
        *reinterpret_cast<int4*>(wp + (int64_t)s * S) = make_int4(0, 0, 0, 0);
      st.mx = 0 > st.mx ? 0 : st.mx;
      st.mn = 0 < st.mn ? 0 : st.mn;
    }
    if (steps == 0) continue;
    int X0[4], X1[4], X2[4], X3[4], Y0[4], Y1[4];
    int U0[4], U1[4], D0[4], D1[4];
    int l0 = 0, r0 = 0, l1 = 0, r1 = 0;
    ld4s(xp, -S, sx, X0);
    ld4s(xp, 0, sx, X1);
    ld4s(xp, S, sx, X2);
    ld4s(yp, 0, sy, Y0);
    if (DIM == 3) {
      ld4s(xp, -N, sx, U0);
      ld4s(xp, N, sx, D0);
    }
    if (st.lane == 0) l0 = __ldg(xp - 1) >> sx;
    if (st.lane == 31) r0 = __ldg(xp + 4) >> sx;
    // x buffers rotate with period 4, y / side buffers with period 2: unroll by 4
    int s = 0;
    for (;;) {
      if (s + 1 < steps) st.prefetch(xp, yp, X3, Y1, U1, D1, l1, r1);
      st.compute(wp, X0, X1, X2, Y0, U0, D0, l0, r0);
      if (++s >= steps) break;
      xp += S; yp += S; wp += S;
      if (s + 1 < steps) st.prefetch(xp, yp, X0, Y0, U0, D0, l0, r0);
      st.compute(wp, X1, X2, X3, Y1, U1, D1, l1, r1);
      if (++s >= steps) break;
      xp += S; yp += S; wp += S;
      if (s + 1 < steps) st.prefetch(xp, yp, X1, Y1, U1, D1, l1, r1);
      st.compute(wp, X2, X3, X0, Y0, U0, D0, l0, r0);
      if (++s >= steps) break;
      xp += S; yp += S; wp += S;
      if (s + 1 < steps) st.prefetch(xp, yp, X2, Y0, U0, D0, l0, r0);
      st.compute(wp, X3, X0, X1, Y1, U1, D1, l1, r1);
      if (++s >= steps) break;
      xp += S; yp += S; wp += S;
    }
  }
  r.olo |= st.olo;
  r.ohi |= st.ohi;
  r.mx = (int64_t)st.mx > r.mx ? (int64_t)st.mx : r.mx;
  r.mn = (int64_t)st.mn < r.mn ? (int64_t)st.mn : r.mn;
}

template <int MODE, int DIM, typename Op>
__global__ void __launch_bounds__(kThreads, DIM == 2 ? 3 : 2) march_win_kernel(Op op, Vec out, WinParams p,
                                                                int R) {
  griddep_wait();
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, int32_t>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  if (op.narrow && need <= 63) {
    if (op.swapped())
      march_loop<MODE, DIM, true>(op, out, p, c, r, R);
    else
      march_loop<MODE, DIM, false>(op, out, p, c, r, R);
  } else
    grid_body<MODE, int32_t>(op, out, p, c, r, need);  // exact generic fallback
  griddep_launch_dependents();
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// ---------------------------------------------------------------------------
// 2-D stencil ops through the bulk-async shared-memory pipeline (bfp_bulk.cuh)

// FW: the fast window of the common case -- pass 1 / recompute storing
// floor(z / 2^rs) with 0 <= rs < 32 and no left shift: the stored int32 is the low word
// of the shifted 64-bit row, one funnel shift (no range selects)
// Prologue of one item of the 2-D bulk pipeline (thread 0): x rows j0-1, j0 with group j0
// (x row j0+1, y row j0) on bar[j0 % YS]; then groups j0+1 .. j0+D.  Needs only the
// operands' addresses, so the kernel can issue the first item's before the op setup.
template <typename Op>
__device__ __forceinline__ int bulk_prologue(const Op& op, const Vec& out, int R, char* smem,
                                             int item) {
  const int64_t N = (int64_t)1 << out.l;
  const int strips = (int)(N / kBulkW);
  const int64_t NZ = out.nz;
  int32_t* xsl = reinterpret_cast<int32_t*>(smem);
  int32_t* ysl = xsl + kBulkXS * kBulkXW;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ysl + kBulkYS * kBulkW);
  const int32_t* X = (const int32_t*)op.sv().data;
  const int32_t* Y = (const int32_t*)op.yv2().data;
  const int strip = item % strips, ch = item / strips;
  const int64_t c0 = (int64_t)strip * kBulkW;
  const int j0 = ch * R;
  const int rows = (int)std::min<int64_t>(R, NZ - j0);
  auto xsrc = [&](int64_t row) { return X + (row > NZ ? NZ : row) * N + c0 - 4; };
  auto ysrc = [&](int64_t row) { return Y + (row > NZ ? NZ : row) * N + c0; };
  const uint32_t tx_bytes = (uint32_t)(kBulkXW + kBulkW) * 4;
  fence_proxy_async_smem();  // previous item's generic reads of the slots
  int g = 0;
  for (; g <= kBulkD && g < rows; ++g) {
    const int64_t tr = j0 + g;
    uint64_t* b = &bar[tr % kBulkYS];
    const uint32_t extra = g == 0 ? 2u * kBulkXW * 4 : 0u;
    mbar_expect_tx(b, tx_bytes + extra);
    if (g == 0) {
      bulk_g2s(xsl + ((tr - 1 + kBulkXS) % kBulkXS) * kBulkXW, xsrc(tr - 1), kBulkXW * 4, b);
      bulk_g2s(xsl + (tr % kBulkXS) * kBulkXW, xsrc(tr), kBulkXW * 4, b);
    }
    bulk_g2s(xsl + ((tr + 1) % kBulkXS) * kBulkXW, xsrc(tr + 1), kBulkXW * 4, b);
    bulk_g2s(ysl + (tr % kBulkYS) * kBulkW, ysrc(tr), kBulkW * 4, b);
  }
  return g;  // groups issued (one barrier phase each, on bar[(j0 + k) % YS])
}

template <int MODE, bool SHIFT, bool SWAP, bool FW, bool EARLY, typename Op>
__device__ __forceinline__ void bulk_loop(const Op& op, const Vec& out, const WinParams& p,
                                          const WinCtx& c, Red& r, int R, char* smem) {
  const int l = out.l;
  const int64_t N = (int64_t)1 << l;
  const int strips = (int)(N / kBulkW);
  const int64_t NZ = out.nz, Z0 = out.z0;
  const int chunks = (int)((NZ + R - 1) / R);
  int32_t* xsl = reinterpret_cast<int32_t*>(smem);                 // kBulkXS x (W+8)
  int32_t* ysl = xsl + kBulkXS * kBulkXW;                           // kBulkYS x W
  uint64_t* bar = reinterpret_cast<uint64_t*>(ysl + kBulkYS * kBulkW);
  uint64_t* ebar = bar + kBulkYS;  // empty: all warps done with the step's freed slots
  const int32_t* X = (const int32_t*)op.sv().data;
  const int32_t* Y = (const int32_t*)op.yv2().data;
  int32_t* O = (int32_t*)out.data;
  const int sx = SHIFT ? op.shs() : 0, sy = SHIFT ? op.shy() : 0;
  const int t = threadIdx.x;
  int32_t mx = INT32_MIN, mn = INT32_MAX;
  uint64_t olo = 0, ohi = 0;
  const bool store = c.store_tmp;
  const uint32_t tx_bytes = (uint32_t)(kBulkXW + kBulkW) * 4;
  uint32_t parity = 0;   // bit k: phase parity of bar[k]
  uint32_t eparity = 0;  // bit k: phase parity of ebar[k]
  for (int item = blockIdx.x; item < strips * chunks; item += gridDim.x) {
    const int strip = item % strips, ch = item / strips;
    const int64_t c0 = (int64_t)strip * kBulkW;
    const int j0 = ch * R;
    const int rows = (int)std::min<int64_t>(R, NZ - j0);
    // source row clamp: rows past the slab read its back halo row (zeros or exchanged)
    auto xsrc = [&](int64_t row) { return X + (row > NZ ? NZ : row) * N + c0 - 4; };
    auto ysrc = [&](int64_t row) { return Y + (row > NZ ? NZ : row) * N + c0; };
    // Warp 8 is the producer (lane 0 issues every bulk copy); warps 0..7 only consume.
    // The first item's prologue may have been issued before the op setup (EARLY, thread 0).
    if (t >= kBulkT) {
      if (t == kBulkT) {
        if (!(EARLY && item == (int)blockIdx.x)) bulk_prologue(op, out, R, smem, item);
        int fx = (int)((j0 - 1 + kBulkXS) % kBulkXS), fy = (int)(j0 % kBulkYS);
        for (int s = 0; s < rows; ++s) {
          // step j0 + s frees x row j - 1 (slot fx) and y row j / its barrier (slot fy)
          const uint32_t ep = (eparity >> fy) & 1u;
          eparity ^= 1u << fy;
          if (s + kBulkD + 1 < rows) {
            mbar_wait(&ebar[fy], ep);  // every consumer warp has finished step j
            const int64_t tr = j0 + s + kBulkD + 1;
            uint64_t* bb = &bar[fy];
            fence_proxy_async_smem();
            mbar_expect_tx(bb, tx_bytes);
            bulk_g2s(xsl + fx * kBulkXW, xsrc(tr + 1), kBulkXW * 4, bb);
            bulk_g2s(ysl + fy * kBulkW, ysrc(tr), kBulkW * 4, bb);
          }
          fx = fx + 1 == kBulkXS ? 0 : fx + 1;
          fy = fy + 1 == kBulkYS ? 0 : fy + 1;
        }
      }
      // the consumers' full-barrier phases of this item, for the bookkeeping below
      for (int s = 0; s < rows; ++s) parity ^= 1u << ((j0 + s) % kBulkYS);
      __syncthreads();
      continue;
    }
    const bool xpad = strip == strips - 1 && t == kBulkT - 1;  // c0 + 4 t + 3 == N - 1
    const int lane = t & 31;
    // the step of the grid's last (pad) row within this chunk, or -1
    const int64_t ps = N - 1 - Z0 - j0;
    const int pad_s = ps >= 0 && ps < rows ? (int)ps : -1;
    int32_t* orow = O + (int64_t)j0 * N + c0 + 4 * t;
    // running ring indices (no 64-bit modulo in the step loop)
    int sp = (int)((j0 - 1 + kBulkXS) % kBulkXS), sc = (int)(j0 % kBulkXS);
    int sn = (int)((j0 + 1) % kBulkXS), sy_ = (int)(j0 % kBulkYS);
    for (int s = 0; s < rows; ++s, orow += N) {
      mbar_wait(&bar[sy_], (parity >> sy_) & 1u);
      parity ^= 1u << sy_;
      const int32_t* xc = xsl + sc * kBulkXW + 4 + 4 * t;
      int4 a = *reinterpret_cast<const int4*>(xsl + sp * kBulkXW + 4 + 4 * t);
      int4 b = *reinterpret_cast<const int4*>(xc);
      int4 d = *reinterpret_cast<const int4*>(xsl + sn * kBulkXW + 4 + 4 * t);
      int4 y4 = *reinterpret_cast<const int4*>(ysl + sy_ * kBulkW + 4 * t);
      // edge lanes read their outer neighbour from the halo words (branch-free)
      const int lf0 = xc[-1], rt0 = xc[4];
      int lf = __shfl_up_sync(0xffffffffu, b.w, 1), rt = __shfl_down_sync(0xffffffffu, b.x, 1);
      lf = lane == 0 ? lf0 : lf;
      rt = lane == 31 ? rt0 : rt;
      const int C[4] = {b.x >> sx, b.y >> sx, b.z >> sx, b.w >> sx};
      const int U[4] = {a.x >> sx, a.y >> sx, a.z >> sx, a.w >> sx};
      const int Dn[4] = {d.x >> sx, d.y >> sx, d.z >> sx, d.w >> sx};
      const int Yv[4] = {y4.x >> sy, y4.y >> sy, y4.z >> sy, y4.w >> sy};
      const int nb[4] = {(lf >> sx) + C[1], C[0] + C[2], C[1] + C[3], C[2] + (rt >> sx)};
      int32_t tt[4] = {0, 0, 0, 0};
      if (s == pad_s) {  // the pad row: exact zeros (uniform branch, one row of the grid)
        mx = mx < 0 ? 0 : mx;
        mn = mn > 0 ? 0 : mn;
      } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int g = 4 * C[k] - (nb[k] + U[k] + Dn[k]);
        int64_t z = op.template point_t<SWAP>(g, C[k], Yv[k]);
        if (k == 3 && xpad) z = 0;
        if constexpr (FW) {
          if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
          tt[k] = (int32_t)__funnelshift_r((uint32_t)z, (uint32_t)((uint64_t)z >> 32), c.rs);
        } else if (MODE == MODE_NNQ) {
          tt[k] = (int32_t)shift_clamp<int64_t>(z, c.lam, p.w_out);
        } else {
          if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
          tt[k] = store ? store_shift<int32_t, int64_t>(z, c) : 0;
        }
        mx = tt[k] > mx ? tt[k] : mx;
        mn = tt[k] < mn ? tt[k] : mn;
      }
      }
      *reinterpret_cast<int4*>(orow) = make_int4(tt[0], tt[1], tt[2], tt[3]);
      // ring slots freed by this step: x row j-1 (slot sp) and y row j / its barrier (slot sy_)
      const int free_x = sp, free_y = sy_;
      sp = sc;
      sc = sn;
      sn = sn + 1 == kBulkXS ? 0 : sn + 1;
      sy_ = sy_ + 1 == kBulkYS ? 0 : sy_ + 1;
      // this warp is done with x row j-1 and y row j: the producer refills their slots
      (void)free_x;
      __syncwarp();
      if (lane == 0) mbar_arrive(&ebar[free_y]);
      eparity ^= 1u << free_y;
    }
    __syncthreads();
  }
  r.olo |= olo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

template <int MODE, typename Op>
__global__ void __launch_bounds__(kBulkT + 32, BFP_B2_MINB) bulk_win_kernel(Op op, Vec out, WinParams p, int R) {
  griddep_wait();
  extern __shared__ __align__(128) char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)(kBulkXS * kBulkXW + kBulkYS * kBulkW) * 4);
  // Early prologue: the first item's loads go out before the (one-thread, ~1.7 us) op
  // setup, which they then overlap; if the setup rules the pipeline out they are drained.
  constexpr bool EARLY = BFP_B2_EARLY && MODE != MODE_RECOMPUTE;
  const int64_t N = (int64_t)1 << out.l;
  const int items = (int)(N / kBulkW) * (int)((out.nz + R - 1) / R);
  int early_groups = 0;
  if (EARLY && threadIdx.x == 0) {
    for (int k = 0; k < kBulkYS; ++k) {
      mbar_init(&bar[k], 1);
      mbar_init(&bar[kBulkYS + k], kBulkT / 32);
    }
    mbar_fence_init();
    if ((int)blockIdx.x < items) early_groups = bulk_prologue(op, out, R, smem, blockIdx.x);
  }
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, int32_t>(op, out, p, c, need);
  if (c.skip) return;  // (RECOMPUTE only: no early prologue)
  Red r;
  r.init();
  if (op.narrow && need <= 63) {
    if (!EARLY && threadIdx.x == 0) {
      for (int k = 0; k < kBulkYS; ++k) {
        mbar_init(&bar[k], 1);
        mbar_init(&bar[kBulkYS + k], kBulkT / 32);
      }
      mbar_fence_init();
    }
    __syncthreads();
    const bool sh = (op.shs() | op.shy()) != 0, sw = op.swapped();
    const bool fw = MODE != MODE_NNQ && c.store_tmp && c.ls == 0 && c.rs < 32;
    if (fw) {
      if (!sh && !sw)
        bulk_loop<MODE, false, false, true, EARLY>(op, out, p, c, r, R, smem);
      else if (sh && !sw)
        bulk_loop<MODE, true, false, true, EARLY>(op, out, p, c, r, R, smem);
      else if (!sh)
        bulk_loop<MODE, false, true, true, EARLY>(op, out, p, c, r, R, smem);
      else
        bulk_loop<MODE, true, true, true, EARLY>(op, out, p, c, r, R, smem);
    } else if (!sh && !sw) {
      bulk_loop<MODE, false, false, false, EARLY>(op, out, p, c, r, R, smem);
    } else if (sh && !sw) {
      bulk_loop<MODE, true, false, false, EARLY>(op, out, p, c, r, R, smem);
    } else if (!sh) {
      bulk_loop<MODE, false, true, false, EARLY>(op, out, p, c, r, R, smem);
    } else {
      bulk_loop<MODE, true, true, false, EARLY>(op, out, p, c, r, R, smem);
    }
  } else {
    if (EARLY && threadIdx.x == 0) {  // drain the early prologue before leaving the smem
      const int j0 = ((int)blockIdx.x / (int)(N / kBulkW)) * R;
      for (int g = 0; g < early_groups; ++g) mbar_wait(&bar[(j0 + g) % kBulkYS], 0u);
    }
    grid_body<MODE, int32_t>(op, out, p, c, r, need);  // exact generic fallback
  }
  griddep_launch_dependents();
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// ---------------------------------------------------------------------------
// 3-D stencil ops through the bulk-async pipeline: a CTA owns a W3 x H3 tile of a
// plane (warp = one row of 128 columns) and marches R planes along z.  Each step
// streams the (H3+2) x (W3+8) x tile of plane k+1+D (y and x halos included) and
// the H3 x W3 y tile of plane k+D, one bulk copy per row issued by the lanes of
// warp 0, into rings of plane slots signalled by mbarriers.
#ifndef BFP_B3_EMPTY  // A/B switch: empty mbarriers (1) or a block barrier (0) per step
#define BFP_B3_EMPTY 0
#endif
#ifndef BFP_B3_SPLIT
#define BFP_B3_SPLIT 1  // int64 residual through SplitWin (A/B: -DBFP_B3_SPLIT=0)
#endif
constexpr int kB3W = 128, kB3H = 8, kB3T = kB3W / 4 * kB3H;  // 256 threads
// planes in flight (D; rings of D+3 x and D+1 y slots) and resident CTAs per SM the
// kernel is compiled for, per storage type and op, swept on the B200 after the balanced
// march depth (tools/ab_b3.sh, profiles/r1_ab_b3.txt; 3-D 511^3 int32 / 1023^3 int64):
// int32 residual D = 2 at 4 CTAs/SM (0.92 of HBM; D = 3: 0.81), int64 D = 3 at 2 CTAs/SM
// (residual 0.94, Jacobi 0.82; D = 2: 0.93 / 0.81, D = 4: 0.77 / 0.65).  The int32 Jacobi
// was D = 4 at 3 CTAs/SM in round 1; after its step loop shrank (two-IMAD.WIDE r term),
// D = 3 at 4 CTAs/SM: 0.89 -> 0.91 (tools/ab_b3j.sh, profiles/r2/r2j_ab_b3j.txt).
// -DBFP_B3_D / -DBFP_B3_MINB / -DBFP_B3_DJ / -DBFP_B3_MINBJ / -DBFP_B3_D64(J) override (A/B).
template <typename Op, typename = void> struct B3Tune {
  static constexpr int D = 2, MINB = 4;
};
template <typename Op> struct B3Tune<Op, decltype((void)Op::b3_depth)> {
  static constexpr int D = Op::b3_depth, MINB = Op::b3_minb;
};
#ifndef BFP_B3_D64
#define BFP_B3_D64 3
#endif
template <typename Op, typename = void> struct B3Tune64 {
  static constexpr int D = BFP_B3_D64;
};
template <typename Op> struct B3Tune64<Op, decltype((void)Op::b3_depth64)> {
  static constexpr int D = Op::b3_depth64;
};
template <typename T, typename Op> constexpr int b3_d() {
#ifdef BFP_B3_D
  return BFP_B3_D;
#else
  return sizeof(T) == 8 ? B3Tune64<Op>::D : B3Tune<Op>::D;
#endif
}
template <typename T, typename Op> constexpr int b3_minb() {
#ifdef BFP_B3_MINB
  return sizeof(T) == 8 ? 2 : BFP_B3_MINB;
#else
  return sizeof(T) == 8 ? 2 : B3Tune<Op>::MINB;
#endif
}
constexpr int kB3XW = kB3W + 8, kB3XR = kB3H + 2;             // x tile row width / rows
constexpr int kB3XT = kB3XW * kB3XR, kB3YT = kB3W * kB3H;     // elements per tile
// x-plane slots padded to 128 B (TMA destinations), 128 B of slack to align the base
template <typename T> constexpr int b3_xtp() {
  return (int)(((kB3XT * sizeof(T) + 127) / 128 * 128) / sizeof(T));
}
template <typename T, typename Op> constexpr size_t b3_smem() {
  constexpr int kB3XS = b3_d<T, Op>() + 3, kB3YS = b3_d<T, Op>() + 1;
  return (size_t)(kB3XS * b3_xtp<T>() + kB3YS * kB3YT) * sizeof(T) + 2 * kB3YS * 8 + 128 + 64;
}
// the x / y operands of a 3-D pipeline launch as tiled TMA descriptors: tensor
// (x, y, plane) over the whole allocation (2 halo planes each side), boxes of one
// x tile ((W+8) x (H+2)) and one y tile (W x H); out-of-range boxes fill zeros
struct B3Maps {
  CUtensorMap x, y;
};

// 4 consecutive elements of a shared-memory tile (16-B aligned)
template <typename T> struct S4;
template <> struct S4<int32_t> {
  using V = int;
  static constexpr int kLaneCols = 4;  // lane i owns columns 4i .. 4i+3
  __device__ static __forceinline__ void ld(const int32_t* p, int sh, V v[4]) {
    const int4 t = *reinterpret_cast<const int4*>(p);
    v[0] = t.x >> sh, v[1] = t.y >> sh, v[2] = t.z >> sh, v[3] = t.w >> sh;
  }
  __device__ static __forceinline__ void st(int32_t* p, const int32_t t[4]) {
    *reinterpret_cast<int4*>(p) = make_int4(t[0], t[1], t[2], t[3]);
  }
};
// int64 tiles use a split-pair lane layout: lane i owns columns (2i, 2i+1) and
// (64+2i, 64+2i+1) of the 128-wide tile, so each 16-B shared-memory load (and each
// 16-B global store) of a warp covers 512 contiguous bytes -- conflict-free, where
// four contiguous int64 per lane (32-B lane stride) would take two wavefronts per load.
template <> struct S4<int64_t> {
  using V = int64_t;
  static constexpr int kLaneCols = 2;  // column of lane i = 2i (pair A), 64 + 2i (pair B)
  __device__ static __forceinline__ void ld(const int64_t* p, int sh, V v[4]) {
    const longlong2 a = reinterpret_cast<const longlong2*>(p)[0];
    const longlong2 b = reinterpret_cast<const longlong2*>(p + 64)[0];
    v[0] = a.x >> sh, v[1] = a.y >> sh, v[2] = b.x >> sh, v[3] = b.y >> sh;
  }
  __device__ static __forceinline__ void st(int64_t* p, const int64_t t[4]) {
    reinterpret_cast<longlong2*>(p)[0] = make_longlong2(t[0], t[1]);
    reinterpret_cast<longlong2*>(p + 64)[0] = make_longlong2(t[2], t[3]);
  }
};
template <typename V> __device__ __forceinline__ V shfl_up1(V v) {
  return __shfl_up_sync(0xffffffffu, v, 1);
}
template <typename V> __device__ __forceinline__ V shfl_dn1(V v) {
  return __shfl_down_sync(0xffffffffu, v, 1);
}

// Split window for int64 storage (SP): with z = X 2^ad + Y (|X|, |Y| < 2^62, ad < 64) and
// the window shift rs < 64, the stored value is exact in 64-bit arithmetic,
//   t = floor(z / 2^rs) = X 2^(ad-rs) + (Y >> rs)        (ad >= rs)
//                       = (X + (Y >> ad)) >> (rs - ad)   (ad <  rs)
// (computed mod 2^64; exact because need - rs <= 63 bounds |t|), and mu* = max msb(z)
// follows from t: msb(z) = msb(t) + rs unless t is 0 or -1, in which case |z| < 2^rs
// and z = zl = X 2^ad + Y mod 2^64 exactly.  Each thread ORs t ^ sign and zl ^ sign and
// folds them into the usual 128-bit OR (a thread with any t outside {0, -1} dominates
// every row of every thread without one), so the finalize is unchanged.  Replaces the
// two-word rows of FW for the GemvOp residual: no 128-bit shifts, adds or compares.
// T = storage type, A = accumulator of the exact rows (int64 narrow for int32
// storage; int64 or __int128 through the ops' generic combine for int64 storage)
template <int MODE, bool SHIFT, bool SWAP, typename T, typename A, bool FW = false,
          bool SP = false, typename Op>
__device__ __forceinline__ void bulk3_loop(const Op& op, const Vec& out, const WinParams& p,
                                           const WinCtx& c, Red& r, int R, char* smem,
                                           const CUtensorMap* tmx, const CUtensorMap* tmy) {
  constexpr int XTP = b3_xtp<T>();
  constexpr int kB3D = b3_d<T, Op>(), kB3XS = kB3D + 3, kB3YS = kB3D + 1;
  using V = typename S4<T>::V;
  const int l = out.l;
  const int64_t N = (int64_t)1 << l, N2 = N * N;
  const int64_t NZ = out.nz, Z0 = out.z0;
  const int tx = (int)(N / kB3W), ty = (int)(N / kB3H);
  const int chunks = (int)((NZ + R - 1) / R);
  T* xsl = reinterpret_cast<T*>(smem);
  T* ysl = xsl + kB3XS * XTP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ysl + kB3YS * kB3YT);
  uint64_t* ebar = bar + kB3YS;  // empty: all warps done with the step's freed slots
  T* O = (T*)out.data;
  const int sx = SHIFT ? op.shs() : 0, sy = SHIFT ? op.shy() : 0;
  const int t = threadIdx.x, lane = t & 31, wy = t >> 5;  // row of the tile
  V mx = sizeof(T) == 4 ? (V)INT32_MIN : (V)INT64_MIN, mn = sizeof(T) == 4 ? (V)INT32_MAX : (V)INT64_MAX;
  uint64_t olo = 0, ohi = 0;
  const bool store = c.store_tmp;
  const uint32_t tx_bytes = (uint32_t)(kB3XT + kB3YT) * sizeof(T);
  SplitWin sw{};
  uint64_t ot = 0, oz = 0;  // SP: OR of t ^ sign, zl ^ sign
  if constexpr (SP) sw = op.b3_split_setup(c.rs);
  uint32_t parity = 0, eparity = 0;
  for (int item = blockIdx.x; item < tx * ty * chunks; item += gridDim.x) {
    const int tile = item % (tx * ty), ch = item / (tx * ty);
    const int64_t x0 = (int64_t)(tile % tx) * kB3W, y0 = (int64_t)(tile / tx) * kB3H;
    const int64_t k0 = (int64_t)ch * R;
    const int planes = (int)std::min<int64_t>(R, NZ - k0);
    // x plane kp (rows y0-1 .. y0+H3, columns x0-4 .. x0+W+3) and y plane ky on barrier
    // b, one tiled TMA box each (tensor plane = local plane + 2 halo planes); `first`
    // also streams x planes kp-2, kp-1 (the start of a march) on the same barrier
    auto issue = [&](int64_t kp, int xslot, int64_t ky, int yslot, uint64_t* b, bool first) {
      if (lane != 0) return;
      mbar_expect_tx(b, tx_bytes + (first ? 2u * kB3XT * sizeof(T) : 0u));
      auto xbox = [&](int64_t k, int slot) {
        tma_g2s_3d(xsl + slot * XTP, tmx, (int)x0 - 4, (int)y0 - 1, (int)((k > NZ ? NZ : k) + 2), b);
      };
      xbox(kp, xslot);
      if (first) {
        xbox(kp - 2, (int)((kp - 2 + kB3XS) % kB3XS));
        xbox(kp - 1, (int)((kp - 1 + kB3XS) % kB3XS));
      }
      tma_g2s_3d(ysl + yslot * kB3YT, tmy, (int)x0, (int)y0, (int)((ky > NZ ? NZ : ky) + 2), b);
    };
    if (wy == 0) {
      fence_proxy_async_smem();
      for (int g = 0; g <= kB3D && g < planes; ++g) {
        const int64_t tk = k0 + g;
        issue(tk + 1, (int)((tk + 1) % kB3XS), tk, (int)(tk % kB3YS), &bar[tk % kB3YS], g == 0);
      }
    }
    // column of the lane's point 3 (the only one that can be the x pad, column N-1)
    const int col3 = sizeof(T) == 4 ? 4 * lane + 3 : 64 + 2 * lane + 1;
    // 32-bit forms of the pad predicates (column 127 of the last tile column, row N-1 of
    // the last tile row, the step of plane N-1): cheaper to rematerialise in the step loop.
    // Measured per instantiation (ops_now.py): int64 residual 0.93 -> 0.94, int32 Jacobi
    // 0.88 -> 0.89, but the int32 residual (64 registers) 0.93 -> 0.87, which keeps the
    // 64-bit compares.
    constexpr bool kPad32 = !(sizeof(T) == 4 && HasSplit<Op>::value);
    const bool xpad = kPad32 ? tile % tx == tx - 1 && lane == 31 : x0 + col3 == N - 1;
    const bool ypad = kPad32 ? tile / tx == ty - 1 && wy == kB3H - 1 : y0 + wy == N - 1;
    const int64_t ps = N - 1 - Z0 - k0;
    const int pad_s = ps >= 0 && ps < planes ? (int)ps : -1;
    int sp = (int)((k0 - 1 + kB3XS) % kB3XS), sc = (int)(k0 % kB3XS);
    int sn = (int)((k0 + 1) % kB3XS), sy_ = (int)(k0 % kB3YS);
    for (int s = 0; s < planes; ++s) {
      const int64_t k = k0 + s;
      mbar_wait(&bar[sy_], (parity >> sy_) & 1u);
      parity ^= 1u << sy_;
      const int off = (wy + 1) * kB3XW + 4 + S4<T>::kLaneCols * lane;
      const T* xc = xsl + sc * XTP + off;
      V C[4], u[4], dn[4], zp[4], zn[4], Yv[4];
      S4<T>::ld(xc, sx, C);
      S4<T>::ld(xc - kB3XW, sx, u);
      S4<T>::ld(xc + kB3XW, sx, dn);
      S4<T>::ld(xsl + sp * XTP + off, sx, zp);
      S4<T>::ld(xsl + sn * XTP + off, sx, zn);
      S4<T>::ld(ysl + sy_ * kB3YT + wy * kB3W + S4<T>::kLaneCols * lane, sy, Yv);
      // x-neighbours of the lane's 4 points (tile halo columns -1 and 128 at the warp ends)
      V Lf[4], Rt[4];
      if constexpr (sizeof(T) == 4) {
        const V lf0 = (V)(xc[-1] >> sx), rt0 = (V)(xc[4] >> sx);
        V lf = shfl_up1(C[3]), rt = shfl_dn1(C[0]);
        Lf[0] = lane == 0 ? lf0 : lf;
        Rt[3] = lane == 31 ? rt0 : rt;
        Lf[1] = C[0], Lf[2] = C[1], Lf[3] = C[2];
        Rt[0] = C[1], Rt[1] = C[2], Rt[2] = C[3];
      } else {  // split pairs: columns 2i, 2i+1 | 64+2i, 64+2i+1
        const V lf0 = (V)(xc[-1] >> sx), rt0 = (V)(xc[66] >> sx);
        const V a = shfl_up1(C[1]), b = shfl_dn1(C[2]);
        // right of column 2i+1 is lane i+1's column 2i+2; lane 31's is column 64 (lane 0, B)
        const V r1 = __shfl_sync(0xffffffffu, lane == 0 ? C[2] : C[0], (lane + 1) & 31);
        // left of column 64+2i is lane i-1's column 64+2i-1; lane 0's is column 63 (lane 31, A)
        const V l2 = __shfl_sync(0xffffffffu, lane == 31 ? C[1] : C[3], (lane + 31) & 31);
        Lf[0] = lane == 0 ? lf0 : a, Rt[0] = C[1];
        Lf[1] = C[0], Rt[1] = r1;
        Lf[2] = l2, Rt[2] = C[3];
        Lf[3] = C[2], Rt[3] = lane == 31 ? rt0 : b;
      }
      T tt[4];
      const bool rowpad = ypad || (kPad32 ? s == pad_s : k + Z0 == N - 1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const V left = Lf[q], right = Rt[q];
        if constexpr (sizeof(T) == 8 && SP) {  // split window (SplitWin)
          const int64_t nb = left + right + u[q] + dn[q] + zp[q] + zn[q];
          int64_t tq, zl;
          op.template point_sp<SWAP>(6 * C[q] - nb, C[q], Yv[q], sw, tq, zl);
          if ((q == 3 && xpad) || rowpad) tq = zl = 0;
          if (MODE == MODE_QCOMP) {
            const uint64_t sg = (uint64_t)(tq >> 63);
            ot |= (uint64_t)tq ^ sg;
            oz |= (uint64_t)zl ^ sg;
          }
          tt[q] = (T)tq;
          mx = (V)tt[q] > mx ? (V)tt[q] : mx;
          mn = (V)tt[q] < mn ? (V)tt[q] : mn;
          continue;
        }
        if constexpr (sizeof(T) == 8 && FW) {  // two-word rows, window rs < 64
          const int64_t nb = left + right + u[q] + dn[q] + zp[q] + zn[q];
          W128 w = op.template point_fw<SWAP>(6 * C[q] - nb, C[q], Yv[q]);
          if ((q == 3 && xpad) || rowpad) w = W128{0, 0};
          if (MODE == MODE_QCOMP) w_or_mag(w, olo, ohi);
          tt[q] = (T)w_shr_lo(w, c.rs);
          mx = (V)tt[q] > mx ? (V)tt[q] : mx;
          mn = (V)tt[q] < mn ? (V)tt[q] : mn;
          continue;
        }
        A z;
        if constexpr (sizeof(T) == 4) {
          const int nb = left + right + u[q] + dn[q] + zp[q] + zn[q];
          z = op.template point_t<SWAP>(6 * C[q] - nb, C[q], Yv[q]);
        } else {
          const int64_t nb = left + right + u[q] + dn[q] + zp[q] + zn[q];  // |g| < 2^62 (w64)
          z = op.template point_w<A>(6 * C[q] - nb, C[q], Yv[q]);
        }
        if (q == 3 && xpad) z = 0;
        if (rowpad) z = 0;
        if constexpr (FW && sizeof(T) == 4) {
          if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
          tt[q] = (T)__funnelshift_r((uint32_t)z, (uint32_t)((uint64_t)z >> 32), c.rs);
        } else if (MODE == MODE_NNQ) {
          tt[q] = (T)shift_clamp<A>(z, c.lam, p.w_out);
        } else {
          if (MODE == MODE_QCOMP) or_mag<A>(z, olo, ohi);
          tt[q] = store ? store_shift<T, A>(z, c) : T(0);
        }
        mx = (V)tt[q] > mx ? (V)tt[q] : mx;
        mn = (V)tt[q] < mn ? (V)tt[q] : mn;
      }
      S4<T>::st(O + k * N2 + (y0 + wy) * N + x0 + S4<T>::kLaneCols * lane, tt);
      const int free_x = sp, free_y = sy_;
      sp = sc;
      sc = sn;
      sn = sn + 1 == kB3XS ? 0 : sn + 1;
      sy_ = sy_ + 1 == kB3YS ? 0 : sy_ + 1;
#if BFP_B3_EMPTY
      // this warp is done with x plane k-1 and y plane k
      __syncwarp();
      if (lane == 0) mbar_arrive(&ebar[free_y]);
      const uint32_t ep = (eparity >> free_y) & 1u;
      eparity ^= 1u << free_y;
      if (wy == 0 && s + kB3D + 1 < planes) {
        mbar_wait(&ebar[free_y], ep);  // every warp has finished step k
#else
      (void)ebar;
      (void)eparity;
      __syncthreads();  // slots of plane k-1 (x) and plane k (y) are free
      if (wy == 0 && s + kB3D + 1 < planes) {
#endif
        fence_proxy_async_smem();
        const int64_t tk = k + kB3D + 1;  // x plane tk+1 -> slot free_x, y plane tk -> free_y
        issue(tk + 1, free_x, tk, free_y, &bar[free_y], false);
      }
    }
    __syncthreads();
  }
  if constexpr (SP && MODE == MODE_QCOMP) {  // fold: msb(z) = msb(t) + rs, else zl
    const int rs = c.rs;
    if (ot) {
      olo |= ot << rs;
      ohi |= rs ? ot >> (64 - rs) : 0;
    } else {
      olo |= oz;
    }
  }
  r.olo |= olo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

// the four (SHIFT, SWAP) instantiations of one bulk3_loop flavour, chosen per launch
template <int MODE, typename T, typename A, bool FW, bool SP, typename Op>
__device__ __forceinline__ void b3_dispatch(bool sh, bool sw, const Op& op, const Vec& out,
                                            const WinParams& p, const WinCtx& c, Red& r, int R,
                                            char* smem, const B3Maps& tm) {
  if (sh && sw)
    bulk3_loop<MODE, true, true, T, A, FW, SP>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
  else if (sh)
    bulk3_loop<MODE, true, false, T, A, FW, SP>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
  else if (sw)
    bulk3_loop<MODE, false, true, T, A, FW, SP>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
  else
    bulk3_loop<MODE, false, false, T, A, FW, SP>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
}

template <int MODE, typename T, typename Op>
__global__ void __launch_bounds__(kB3T, b3_minb<T, Op>())
    bulk3_win_kernel(Op op, Vec out, WinParams p, int R, const __grid_constant__ B3Maps tm) {
  extern __shared__ __align__(128) char smem_raw[];
  char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  griddep_wait();
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, T>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  const bool fast = sizeof(T) == 4 ? (op.narrow && need <= 63) : (op.w64 && need <= 127);
  if (fast) {
    uint64_t* bar =
        reinterpret_cast<uint64_t*>(smem + (size_t)((b3_d<T, Op>() + 3) * b3_xtp<T>() +
                                                    (b3_d<T, Op>() + 1) * kB3YT) * sizeof(T));
    constexpr int kB3YS = b3_d<T, Op>() + 1;
    if (threadIdx.x == 0) {
      for (int k = 0; k < kB3YS; ++k) {
        mbar_init(&bar[k], 1);
        mbar_init(&bar[kB3YS + k], kB3T / 32);
      }
      mbar_fence_init();
    }
    __syncthreads();
    const bool sh = (op.shs() | op.shy()) != 0;
    if constexpr (sizeof(T) == 4) {
      const bool sw = op.swapped();
      const bool fw = MODE != MODE_NNQ && c.store_tmp && c.ls == 0 && c.rs < 32;
      if (fw) {
        if (!sh && !sw)
          bulk3_loop<MODE, false, false, T, int64_t, true>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
        else if (sh && !sw)
          bulk3_loop<MODE, true, false, T, int64_t, true>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
        else if (!sh)
          bulk3_loop<MODE, false, true, T, int64_t, true>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
        else
          bulk3_loop<MODE, true, true, T, int64_t, true>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
      } else if (!sh && !sw) {
        bulk3_loop<MODE, false, false, T, int64_t>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
      } else if (sh && !sw) {
        bulk3_loop<MODE, true, false, T, int64_t>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
      } else if (!sh) {
        bulk3_loop<MODE, false, true, T, int64_t>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
      } else {
        bulk3_loop<MODE, true, true, T, int64_t>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
      }
    } else {
      if (need <= 63) {
        if (sh)
          bulk3_loop<MODE, true, false, T, int64_t>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
        else
          bulk3_loop<MODE, false, false, T, int64_t>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
      } else if (MODE != MODE_NNQ && op.fwi && c.store_tmp && c.ls == 0 && c.rs < 64) {
        bool split = false;
        if constexpr (HasB3Split<Op>::value) {
          split = BFP_B3_SPLIT && op.b3_split_ok(need, c.rs);
          if (split)
            b3_dispatch<MODE, T, int64_t, false, true>(sh, op.fw_swap(), op, out, p, c, r, R, smem, tm);
        }
        if (!split)
          b3_dispatch<MODE, T, i128, true, false>(sh, op.fw_swap(), op, out, p, c, r, R, smem, tm);
      } else {
        if (sh)
          bulk3_loop<MODE, true, false, T, i128>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
        else
          bulk3_loop<MODE, false, false, T, i128>(op, out, p, c, r, R, smem, &tm.x, &tm.y);
      }
    }
  } else {
    grid_body<MODE, T>(op, out, p, c, r, need);  // exact generic path (or the width error)
  }
  griddep_launch_dependents();
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// ---------------------------------------------------------------------------
// 3-D prolongation (+ correction) through tiled TMA.  A CTA owns a 128 x 8 tile of
// the fine plane and marches fine planes in pairs (2K, 2K+1): both read the
// row sums S_K = sum over the two coarse rows of x-lines of coarse plane K, and
// fine plane 2K also reads S_{K-1}, so each coarse plane tile (72 x 5 box) is
// loaded and summed once per pair; P e_c (2K) = S_{K-1} + S_K, (2K+1) = 2 S_K.
// The correction operand y arrives as two 128 x 8 boxes per pair.
#ifdef BFP_P3_TIMING
__device__ long long g_p3_prof[8];
#define P3T(k)                                                                       \
  if (threadIdx.x == 0 && blockIdx.x == 0) {                                         \
    const long long _n = clock64();                                                  \
    atomicAdd((unsigned long long*)&g_p3_prof[k], (unsigned long long)(_n - _pt));   \
    _pt = _n;                                                                        \
  }
#else
#define P3T(k)
#endif
constexpr int kP3W = 128, kP3H = 8, kP3T = 256;
constexpr int kP3CW = kP3W / 2 + 8, kP3CH = kP3H / 2 + 1;  // coarse box 72 x 5
template <typename T> constexpr int p3_ct() {  // coarse slot in elements (128-B multiple)
  return (int)(((kP3CW * kP3CH * sizeof(T) + 127) / 128 * 128) / sizeof(T));
}
constexpr int kP3YT = kP3W * kP3H;                               // one y box
// Ring depth (fine-plane pairs in flight) and resident CTAs per SM, per op and storage type
// (tools/ab_p3.sh, profiles/r2/r2j_ab_p3.txt): the plain prolongation streams 1.4 / 2.9 KB
// coarse boxes and wants a deeper ring; prolong + correct moves two 4 / 8 KB fine boxes per
// pair and runs best with a shallow ring and more CTAs.
#ifndef BFP_P3_D
#define BFP_P3_D 3
#endif
#ifndef BFP_P3_DC
#define BFP_P3_DC 1
#endif
#ifndef BFP_P3_MINB  // int32 storage
#define BFP_P3_MINB 3
#endif
#ifndef BFP_P3_MINBC
#define BFP_P3_MINBC 4
#endif
#ifndef BFP_P3_MINB64  // int64 storage
#define BFP_P3_MINB64 2
#endif
#ifndef BFP_P3_MINBC64
#define BFP_P3_MINBC64 2
#endif
template <typename Op> constexpr int p3_d() { return Op::kCorr ? BFP_P3_DC : BFP_P3_D; }
template <typename Op> constexpr int p3_s() { return p3_d<Op>() + 1; }  // slots / barriers
template <typename T, typename Op> constexpr int p3_minb() {
  return sizeof(T) == 4 ? (Op::kCorr ? BFP_P3_MINBC : BFP_P3_MINB)
                        : (Op::kCorr ? BFP_P3_MINBC64 : BFP_P3_MINB64);
}
// the y part of a slot: two fine boxes (prolong + correct only)
template <typename Op> constexpr int p3_ys() { return Op::kCorr ? 2 * kP3YT : 0; }
template <typename T, typename Op> constexpr size_t p3_smem() {
  return (size_t)p3_s<Op>() * (p3_ct<T>() + p3_ys<Op>()) * sizeof(T) + 2 * p3_s<Op>() * 8 + 128 + 64;
}
struct P3Maps {
  CUtensorMap c, y;
};

// Warp-specialised: warps 0..7 (kP3T threads) are the consumers, warp 8 is the producer.
// Lane 0 of the producer streams the boxes into a ring of kP3S slots, waiting on the slot's
// EMPTY mbarrier (one arrival per consumer warp) and signalling its FULL mbarrier through
// complete_tx; the consumers never execute a block barrier, a proxy fence or a TMA issue
// (measured before: of ~2200 clk per step, 640 were the elected consumer thread's fence +
// issue with the other warps idle behind it, profiles/r2/r2c_p3_phases.txt).  Ring step j of
// an item: j = 0 loads coarse plane K0 - 1 alone (S_{K0-1}), j >= 1 loads coarse plane
// K0 + j - 1 and the two y boxes of pair K0 + j - 1.  The ring position runs on across
// items, so nothing drains between them.
template <int MODE, bool FW, typename T, typename Op>
__device__ __forceinline__ void pro3_loop(const Op& op, const Vec& out, const WinParams& p,
                                          const WinCtx& c, Red& r, int R, char* smem,
                                          const CUtensorMap* tmc, const CUtensorMap* tmy) {
  const int l = out.l;
  const int64_t N = (int64_t)1 << l, N2 = N * N;
  const int64_t NZ = out.nz, Z0 = out.z0;
  const int tx = (int)(N / kP3W), ty = (int)(N / kP3H);
  const int chunks = (int)((NZ + R - 1) / R);
  using V = typename std::conditional<sizeof(T) == 4, int, int64_t>::type;
  constexpr int kP3CT = p3_ct<T>();
  T* csl = reinterpret_cast<T*>(smem);
  constexpr int kP3S = p3_s<Op>();
  T* ysl = csl + kP3S * kP3CT;
  uint64_t* full = reinterpret_cast<uint64_t*>(ysl + kP3S * p3_ys<Op>());
  uint64_t* empty = full + kP3S;
  T* O = (T*)out.data;
  const int sc = op.shc(), sy = op.shy();
  const int kc_off = op.zp / 2;  // coarse local plane of fine local pair K
  const int t = threadIdx.x, lane = t & 31, wy = t >> 5;
  const bool producer = t >= kP3T;
  T mx = Lim<T>::lo, mn = Lim<T>::hi;
  uint64_t olo = 0, ohi = 0;
  uint32_t o32lo = 0, o32hi = 0;  // int32 fast window: OR of z ^ sign(z) in two words
  const bool store = c.store_tmp;
  const uint32_t cbytes = (uint32_t)(kP3CW * kP3CH * sizeof(T)), ybytes = (uint32_t)(kP3YT * sizeof(T));
  uint32_t ring = 0;  // ring position of the item's step 0 (both roles advance it alike)
  // local coarse rows of fine row y0 + wy and the coarse column of this thread's 4 points
  // (int32: fine columns 4 lane .. 4 lane + 3 from coarse 2 lane - 1 .. 2 lane + 1; int64:
  // split pairs, fine columns 2 lane, 2 lane + 1 | 64 + 2 lane, 64 + 2 lane + 1 from coarse
  // lane - 1, lane | 32 + lane - 1, 32 + lane, so that every 16-byte store and shared load
  // of the warp is contiguous)
  const int r0 = ((wy - 1) >> 1) + 1, r1 = (wy >> 1) + 1;
  const int col = (sizeof(T) == 4 ? 2 * lane : lane) + 4;
  const int xoff = sizeof(T) == 4 ? 4 * lane : 2 * lane;  // fine column of point 0
  // int32 fast window: z = g Pg + y Py as two IMAD.WIDE (no operand selects).  No pad
  // masking there: a fine pad index has both coarse taps on the coarse pad (index N/2 - 1,
  // stored zero) and y's own pad is zero, so its row is 0 Pg + 0 Py.
  [[maybe_unused]] int Pg = 1, Py = 0;
  if constexpr (Op::kCorr && sizeof(T) == 4) {
    Pg = op.swap ? 1 : op.P;
    Py = op.swap ? op.P : 1;
  }
  [[maybe_unused]] int sg64 = 0, sy64 = 0;  // int64 fast window: z = g 2^sg64 + y 2^sy64
  if constexpr (Op::kCorr && sizeof(T) == 8) {
    sg64 = op.swap ? 0 : op.AD;
    sy64 = op.swap ? op.AD : 0;
  }
  for (int item = blockIdx.x; item < tx * ty * chunks; item += gridDim.x) {
    const int tile = item % (tx * ty), ch = item / (tx * ty);
    const int64_t x0 = (int64_t)(tile % tx) * kP3W, y0 = (int64_t)(tile / tx) * kP3H;
    const int64_t k0 = (int64_t)ch * R;
    const int pairs = (int)(std::min<int64_t>(R, NZ - k0) / 2);
    const int64_t K0 = k0 / 2;
    if (producer) {
      if (lane == 0) {
        for (int j = 0; j <= pairs; ++j) {
          const uint32_t g = ring + (uint32_t)j, slot = g % kP3S;
          // the slot's previous user (ring step g - kP3S) has been read by every consumer warp
          mbar_wait(&empty[slot], ((g / kP3S) & 1u) ^ 1u);
          fence_proxy_async_smem();
          uint64_t* b = &full[slot];
          const int64_t K = K0 + j - 1;
          mbar_expect_tx(b, cbytes + (Op::kCorr && j > 0 ? 2 * ybytes : 0u));
          tma_g2s_3d(csl + slot * kP3CT, tmc, (int)(x0 / 2) - 4, (int)(y0 / 2) - 1,
                     (int)(K + kc_off + 2), b);
          if (Op::kCorr && j > 0)
            for (int h = 0; h < 2; ++h)
              tma_g2s_3d(ysl + (slot * 2 + h) * kP3YT, tmy, (int)x0, (int)y0, (int)(2 * K + h + 2), b);
        }
      }
      ring += (uint32_t)pairs + 1u;
      continue;
    }
    const bool xpad = x0 + (sizeof(T) == 4 ? 4 * lane + 3 : 64 + 2 * lane + 1) == N - 1;
    const bool ypad = y0 + wy == N - 1;
    T* dstp = O + 2 * K0 * N2 + (y0 + wy) * N + x0 + xoff;
    V Sp[4] = {0, 0, 0, 0};  // S_{K-1}
    for (int j = 0; j <= pairs; ++j) {
      const uint32_t g = ring + (uint32_t)j, slot = g % kP3S;
      mbar_wait(&full[slot], (g / kP3S) & 1u);
      V Sc[4];
      {
        const T* cb = csl + slot * kP3CT;
        V acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const T* row = cb + (rr ? r1 : r0) * kP3CW + col;
          if constexpr (sizeof(T) == 4) {
            const V a = row[-1] >> sc, b = row[0] >> sc, e = row[1] >> sc;
            acc[0] += a + b;
            acc[1] += 2 * b;
            acc[2] += b + e;
            acc[3] += 2 * e;
          } else {
            const V a = row[-1] >> sc, b = row[0] >> sc, a2 = row[31] >> sc, b2 = row[32] >> sc;
            acc[0] += a + b;
            acc[1] += 2 * b;
            acc[2] += a2 + b2;
            acc[3] += 2 * b2;
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) Sc[q] = acc[q];
      }
      if (j > 0) {
        const int s = j - 1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if constexpr (FW && sizeof(T) == 4) {
            int y4[4] = {0, 0, 0, 0};
            if constexpr (Op::kCorr) {
              const int4 yy = *reinterpret_cast<const int4*>(ysl + (slot * 2 + h) * kP3YT +
                                                             wy * kP3W + 4 * lane);
              y4[0] = yy.x >> sy, y4[1] = yy.y >> sy, y4[2] = yy.z >> sy, y4[3] = yy.w >> sy;
            }
            int tq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int gq = h ? 2 * Sc[q] : Sp[q] + Sc[q];
              if constexpr (Op::kCorr) {
                const int64_t z = mad_wide(gq, Pg, mul_wide(y4[q], Py));
                const uint32_t zl = (uint32_t)z, zh = (uint32_t)((uint64_t)z >> 32);
                if (MODE == MODE_QCOMP) {
                  const uint32_t sg = (uint32_t)((int)zh >> 31);
                  o32lo |= zl ^ sg;
                  o32hi |= zh ^ sg;
                }
                tq[q] = (int)__funnelshift_r(zl, zh, c.rs);
              } else {
                if (MODE == MODE_QCOMP) o32lo |= (uint32_t)(gq ^ (gq >> 31));
                tq[q] = gq >> c.rs;
              }
              mx = tq[q] > mx ? tq[q] : mx;
              mn = tq[q] < mn ? tq[q] : mn;
            }
            *reinterpret_cast<int4*>(dstp) = make_int4(tq[0], tq[1], tq[2], tq[3]);
            dstp += N2;
            continue;
          }
          if constexpr (FW && sizeof(T) == 8 && Op::kCorr) {
            // int64 fast window (need <= 63, rs < 64): the int32 loop's structure in 64-bit
            // words -- both alignment shifts uniform (one of them 0), no pad masks (same
            // argument: pad taps and y's pads are stored zeros), running store pointer.
            // Prolong + correct 0.97 -> 0.99 of the copy peak; the plain prolongation ran
            // SLOWER through it (0.875 -> 0.834, store bursts) and keeps the generic rows.
            int64_t y4[4] = {0, 0, 0, 0};
            if constexpr (Op::kCorr) {
              const T* yp = ysl + (slot * 2 + h) * kP3YT + wy * kP3W + xoff;
              const longlong2 a = *reinterpret_cast<const longlong2*>(yp);
              const longlong2 b = *reinterpret_cast<const longlong2*>(yp + 64);
              y4[0] = a.x >> sy, y4[1] = a.y >> sy, y4[2] = b.x >> sy, y4[3] = b.y >> sy;
            }
            int64_t tq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int64_t gq = h ? 2 * Sc[q] : Sp[q] + Sc[q];
              int64_t z = gq;
              if constexpr (Op::kCorr)
                z = (int64_t)(((uint64_t)gq << sg64) + ((uint64_t)y4[q] << sy64));
              if (MODE == MODE_QCOMP) olo |= (uint64_t)z ^ (uint64_t)(z >> 63);
              tq[q] = z >> c.rs;
              mx = tq[q] > mx ? tq[q] : mx;
              mn = tq[q] < mn ? tq[q] : mn;
            }
            *reinterpret_cast<longlong2*>(dstp) = make_longlong2(tq[0], tq[1]);
            *reinterpret_cast<longlong2*>(dstp + 64) = make_longlong2(tq[2], tq[3]);
            dstp += N2;
            continue;
          }
          const int64_t k = 2 * (K0 + s) + h;  // local fine plane
          V yv[4] = {0, 0, 0, 0};
          if (Op::kCorr) {
            const T* yp = ysl + (slot * 2 + h) * kP3YT + wy * kP3W + xoff;
            if constexpr (sizeof(T) == 4) {
              const int4 y4 = *reinterpret_cast<const int4*>(yp);
              yv[0] = y4.x >> sy, yv[1] = y4.y >> sy, yv[2] = y4.z >> sy, yv[3] = y4.w >> sy;
            } else {
              const longlong2 a = *reinterpret_cast<const longlong2*>(yp);
              const longlong2 b = *reinterpret_cast<const longlong2*>(yp + 64);
              yv[0] = a.x >> sy, yv[1] = a.y >> sy, yv[2] = b.x >> sy, yv[3] = b.y >> sy;
            }
          }
          const bool rowpad = ypad || k + Z0 == N - 1;
          T tt[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const V gq = h ? 2 * Sc[q] : Sp[q] + Sc[q];
            int64_t z;
            if constexpr (sizeof(T) == 4)
              z = op.corr(gq, yv[q]);
            else
              z = op.corr_w(gq, yv[q]);
            if ((q == 3 && xpad) || rowpad) z = 0;
            if constexpr (FW) {
              if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
              if constexpr (sizeof(T) == 4)
                tt[q] = (T)__funnelshift_r((uint32_t)z, (uint32_t)((uint64_t)z >> 32), c.rs);
              else
                tt[q] = (T)(z >> c.rs);
            } else if (MODE == MODE_NNQ) {
              tt[q] = (T)shift_clamp<int64_t>(z, c.lam, p.w_out);
            } else {
              if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
              tt[q] = store ? store_shift<T, int64_t>(z, c) : (T)0;
            }
            mx = tt[q] > mx ? tt[q] : mx;
            mn = tt[q] < mn ? tt[q] : mn;
          }
          T* dst = O + k * N2 + (y0 + wy) * N + x0 + xoff;
          if constexpr (sizeof(T) == 4) {
            *reinterpret_cast<int4*>(dst) = make_int4(tt[0], tt[1], tt[2], tt[3]);
          } else {
            *reinterpret_cast<longlong2*>(dst) = make_longlong2(tt[0], tt[1]);
            *reinterpret_cast<longlong2*>(dst + 64) = make_longlong2(tt[2], tt[3]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) Sp[q] = Sc[q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
    }
    ring += (uint32_t)pairs + 1u;
  }
  r.olo |= olo | ((uint64_t)o32hi << 32) | o32lo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

template <int MODE, typename T, typename Op>
__global__ void __launch_bounds__(kP3T + 32, p3_minb<T, Op>())
    pro3_win_kernel(Op op, Vec out, WinParams p, int R, const __grid_constant__ P3Maps tm) {
  extern __shared__ __align__(128) char smem_raw[];
  char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  griddep_wait();
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, T>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  const bool fast = sizeof(T) == 4 ? (op.narrow && need <= 63) : op.wide;
  if (fast) {
    constexpr int kP3S = p3_s<Op>();
    uint64_t* bar =
        reinterpret_cast<uint64_t*>(smem + (size_t)kP3S * (p3_ct<T>() + p3_ys<Op>()) * sizeof(T));
    if (threadIdx.x == 0) {
      for (int k = 0; k < kP3S; ++k) {
        mbar_init(&bar[k], 1);                    // full: the producer's expect_tx arrival
        mbar_init(&bar[kP3S + k], kP3T / 32);     // empty: one arrival per consumer warp
      }
      mbar_fence_init();
    }
    __syncthreads();
    if (MODE != MODE_NNQ && c.store_tmp && c.ls == 0 && c.rs < (sizeof(T) == 4 ? 32 : 64))
      pro3_loop<MODE, true, T>(op, out, p, c, r, R, smem, &tm.c, &tm.y);
    else
      pro3_loop<MODE, false, T>(op, out, p, c, r, R, smem, &tm.c, &tm.y);
  } else {
    grid_body<MODE, T>(op, out, p, c, r, need);  // exact generic path
  }
  griddep_launch_dependents();
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// ---------------------------------------------------------------------------
// 3-D full-weighting restriction through tiled TMA.  A CTA owns a 64 x 8 tile of the
// coarse plane (4 coarse points per thread) and marches coarse planes K; fine plane p
// contributes the row sums T_p = sum_{rows 2J..2J+2} w_y (f[2I] + 2 f[2I+1] + f[2I+2])
// and coarse K = T_{2K} + 2 T_{2K+1} + T_{2K+2}: each fine plane tile (136 x 17 box)
// is loaded once and T_{2K+2} is kept in registers for the next step.
constexpr int kR3W = 64, kR3H = 8, kR3T = kR3W / 4 * kR3H;           // 128 threads
constexpr int kR3FW = 2 * kR3W + 8, kR3FH = 2 * kR3H + 1;            // fine box 136 x 17
constexpr int kR3D = 1;                                              // steps in flight
constexpr int kR3FS = 2 * kR3D + 3, kR3B = kR3D + 1;                 // plane slots, barriers
// plane slot in elements of the storage type (128-B multiple)
template <typename T> constexpr int r3_ft() {
  return (int)(((kR3FW * kR3FH * sizeof(T) + 127) / 128 * 128) / sizeof(T));
}
template <typename T> constexpr size_t r3_smem() {
  return (size_t)kR3FS * r3_ft<T>() * sizeof(T) + kR3B * 8 + 128 + 64;
}
// one fine row segment of 9 values (columns 2 I0 - ... of 4 coarse points), shifted
__device__ __forceinline__ void r3_row(const int32_t* row, int sh, int v[9]) {
  const int4 a = *reinterpret_cast<const int4*>(row);
  const int4 b = *reinterpret_cast<const int4*>(row + 4);
  v[0] = a.x >> sh, v[1] = a.y >> sh, v[2] = a.z >> sh, v[3] = a.w >> sh;
  v[4] = b.x >> sh, v[5] = b.y >> sh, v[6] = b.z >> sh, v[7] = b.w >> sh;
  v[8] = row[8] >> sh;
}
__device__ __forceinline__ void r3_row(const int64_t* row, int sh, int64_t v[9]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const longlong2 a = reinterpret_cast<const longlong2*>(row)[k];
    v[2 * k] = a.x >> sh, v[2 * k + 1] = a.y >> sh;
  }
  v[8] = row[8] >> sh;
}
struct R3Maps {
  CUtensorMap f;
};

// T = storage type: int32 (plane sums in int32, need <= 35) or int64 (C5; plane sums in
// int64, need <= 63); the box and the march are the same, the slot holds T elements
template <int MODE, bool FW, typename T>
__device__ __forceinline__ void rst3_loop(const RestrictOp& op, const Vec& out,
                                          const WinParams& p, const WinCtx& c, Red& r, int R,
                                          char* smem, const CUtensorMap* tmf) {
  using V = typename std::conditional<sizeof(T) == 4, int, int64_t>::type;
  constexpr int kR3FT = r3_ft<T>();
  const int lc = out.l;  // coarse level
  const int64_t Nc = (int64_t)1 << lc, Nc2 = Nc * Nc;
  const int64_t NZ = out.nz, Z0 = out.z0;
  const int tx = (int)(Nc / kR3W), ty = (int)(Nc / kR3H);
  const int chunks = (int)((NZ + R - 1) / R);
  T* fsl = reinterpret_cast<T*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(fsl + kR3FS * kR3FT);
  T* O = (T*)out.data;
  const int sh = (int)op.sr;
  const int t = threadIdx.x, cy = t >> 4, cxq = t & 15;  // coarse row in tile, 4-group
  T mx = Lim<T>::lo, mn = Lim<T>::hi;
  uint64_t olo = 0, ohi = 0;
  const bool store = c.store_tmp;
  const uint32_t pbytes = (uint32_t)(kR3FW * kR3FH * sizeof(T));
  uint32_t parity = 0;
  for (int item = blockIdx.x; item < tx * ty * chunks; item += gridDim.x) {
    const int tile = item % (tx * ty), ch = item / (tx * ty);
    const int64_t x0 = (int64_t)(tile % tx) * kR3W, y0 = (int64_t)(tile / tx) * kR3H;
    const int64_t K0 = (int64_t)ch * R;
    const int steps = (int)std::min<int64_t>(R, NZ - K0);
    // step s: fine planes 2(K0+s)+1, +2 (and 2 K0 at s = 0); fine plane f -> slot
    // (f - 2 K0) % FS, barrier s % B
    auto issue = [&](int s) {
      uint64_t* b = &bar[s % kR3B];
      mbar_expect_tx(b, pbytes * (s == 0 ? 3u : 2u));
      for (int j = (s == 0 ? 0 : 1); j <= 2; ++j) {
        const int64_t f = 2 * (K0 + s) + j;  // local fine plane
        tma_g2s_3d(fsl + (int)((f - 2 * K0) % kR3FS) * kR3FT, tmf, (int)(2 * x0) - 4,
                   (int)(2 * y0), (int)(f + 2), b);
      }
    };
    if (t == 0) {
      fence_proxy_async_smem();
      for (int s = 0; s <= kR3D && s < steps; ++s) issue(s);
    }
    // fine columns 2 I0 .. 2 I0 + 8 of this thread's 4 coarse points, rows 2 cy .. 2 cy + 2
    const int fcol = 8 * cxq + 4, frow = 2 * cy;
    auto T_of = [&](int64_t f, V Ts[4]) {
      const T* base = fsl + (int)((f - 2 * K0) % kR3FS) * kR3FT + fcol;
      V acc[4] = {0, 0, 0, 0};
#pragma unroll
      for (int py = 0; py < 3; ++py) {
        V v[9];
        r3_row(base + (frow + py) * kR3FW, sh, v);
        const V wy = py == 1 ? 2 : 1;
        acc[0] += wy * (v[0] + 2 * v[1] + v[2]);
        acc[1] += wy * (v[2] + 2 * v[3] + v[4]);
        acc[2] += wy * (v[4] + 2 * v[5] + v[6]);
        acc[3] += wy * (v[6] + 2 * v[7] + v[8]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) Ts[q] = acc[q];
    };
    // int64 storage: the thread's 4 coarse points are columns cxq + 16 q (not 4 cxq + q), so
    // that the 16-byte shared loads of a half-warp are contiguous (the 4-consecutive layout
    // strides them by 64 bytes: 4-way bank conflicts, short-scoreboard-bound at 0.75 of
    // HBM).  Per plane: A = sum_py w_py f(2I), B = sum_py w_py f(2I + 1) from one longlong2
    // per row and point; T(I) = A(I) + 2 B(I) + A(I + 1), A(I + 1) from lane + 1 by shuffle
    // (lane 15 of the half-warp: lane 0's next point, or the tile's halo column 128).
    [[maybe_unused]] auto T_of64 = [&](int64_t f, V Ts[4]) {
      const T* base = fsl + (int)((f - 2 * K0) % kR3FS) * kR3FT + 4 + 2 * cxq;
      V A[5] = {0, 0, 0, 0, 0}, Bs[4] = {0, 0, 0, 0};
#pragma unroll
      for (int py = 0; py < 3; ++py) {
        const T* row = base + (frow + py) * kR3FW;
        const V wy = py == 1 ? 2 : 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const longlong2 a = *reinterpret_cast<const longlong2*>(row + 32 * q);
          A[q] += wy * (V)(a.x >> sh);
          Bs[q] += wy * (V)(a.y >> sh);
        }
        A[4] += wy * (V)(row[128 - 2 * cxq] >> sh);  // fine column 128 of the row (broadcast)
      }
      const int src = (t & 16) | ((cxq + 1) & 15);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const V nxt = __shfl_sync(0xffffffffu, cxq == 0 ? A[q + 1] : A[q], src);
        Ts[q] = A[q] + 2 * Bs[q] + nxt;
      }
    };
    const bool xpad = sizeof(T) == 4 ? x0 + 4 * cxq + 3 == Nc - 1 : x0 + cxq + 48 == Nc - 1;
    const bool ypad = y0 + cy == Nc - 1;
    V Tp[4] = {0, 0, 0, 0};  // T_{2K}
    for (int s = 0; s < steps; ++s) {
      const int64_t Kc = K0 + s;
      mbar_wait(&bar[s % kR3B], (parity >> (s % kR3B)) & 1u);
      parity ^= 1u << (s % kR3B);
      V T1[4], T2[4];
      if constexpr (sizeof(T) == 4) {
        if (s == 0) T_of(2 * Kc, Tp);
        T_of(2 * Kc + 1, T1);
        T_of(2 * Kc + 2, T2);
      } else {
        if (s == 0) T_of64(2 * Kc, Tp);
        T_of64(2 * Kc + 1, T1);
        T_of64(2 * Kc + 2, T2);
      }
      const bool rowpad = ypad || Kc + Z0 == Nc - 1;
      T tt[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t z = (int64_t)Tp[q] + 2 * (int64_t)T1[q] + (int64_t)T2[q];
        if ((q == 3 && xpad) || rowpad) z = 0;
        if constexpr (FW) {
          if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
          if constexpr (sizeof(T) == 4)
            tt[q] = (T)__funnelshift_r((uint32_t)z, (uint32_t)((uint64_t)z >> 32), c.rs);
          else
            tt[q] = (T)(z >> c.rs);
        } else if (MODE == MODE_NNQ) {
          tt[q] = (T)shift_clamp<int64_t>(z, c.lam, p.w_out);
        } else {
          if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
          tt[q] = store ? store_shift<T, int64_t>(z, c) : (T)0;
        }
        mx = tt[q] > mx ? tt[q] : mx;
        mn = tt[q] < mn ? tt[q] : mn;
      }
      if constexpr (sizeof(T) == 4) {
        T* dst = O + Kc * Nc2 + (y0 + cy) * Nc + x0 + 4 * cxq;
        *reinterpret_cast<int4*>(dst) = make_int4(tt[0], tt[1], tt[2], tt[3]);
      } else {
        T* dst = O + Kc * Nc2 + (y0 + cy) * Nc + x0 + cxq;
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[16 * q] = tt[q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) Tp[q] = T2[q];
      __syncthreads();  // fine planes 2Kc, 2Kc + 1 are free
      if (t == 0 && s + kR3D + 1 < steps) {
        fence_proxy_async_smem();
        issue(s + kR3D + 1);
      }
    }
    __syncthreads();
  }
  r.olo |= olo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

template <int MODE, typename T>
__global__ void __launch_bounds__(kR3T, sizeof(T) == 4 ? 8 : 2)
    rst3_win_kernel(RestrictOp op, Vec out, WinParams p, int R, const __grid_constant__ R3Maps tm) {
  extern __shared__ __align__(128) char smem_raw[];
  char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  griddep_wait();
  int64_t need = 0;
  WinCtx c;
  block_setup<RestrictOp, T>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  // plane sums T_p (weights 16) in int32 need eff_bits(r) <= 27, i.e. need <= 35 in 3-D;
  // int64 storage sums in int64 (need <= 63); the final combination is 64-bit
  const bool fast = sizeof(T) == 4 ? (op.sr < 32 && need <= 35) : (op.sr < 64 && need <= 63);
  if (fast && op.gs == 0) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)kR3FS * r3_ft<T>() * sizeof(T));
    if (threadIdx.x == 0) {
      for (int k = 0; k < kR3B; ++k) mbar_init(&bar[k], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (MODE != MODE_NNQ && c.store_tmp && c.ls == 0 && c.rs < (sizeof(T) == 4 ? 32 : 64))
      rst3_loop<MODE, true, T>(op, out, p, c, r, R, smem, &tm.f);
    else
      rst3_loop<MODE, false, T>(op, out, p, c, r, R, smem, &tm.f);
  } else {
    grid_body<MODE, T>(op, out, p, c, r, need);  // exact generic path
  }
  griddep_launch_dependents();
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// ---------------------------------------------------------------------------
// 2-D transfers through the bulk-async row pipeline (the 2-D analogues of pro3 /
// rst3, rows instead of planes, one cp.async.bulk per row).
// Prolong (+ correct): a CTA owns 1024 fine columns and marches fine-row pairs
// (2J, 2J+1) over the coarse row sums S_J (P e_c: 2J -> S_{J-1} + S_J, 2J+1 -> 2 S_J).
constexpr int kP2T = 256, kP2W = 4 * kP2T;                       // fine strip
constexpr int kP2CW = kP2W / 2 + 8;                              // coarse row slot (words)
#ifndef BFP_P2_D
#define BFP_P2_D 2
#endif
#ifndef BFP_P2_MINB
#define BFP_P2_MINB 4
#endif
constexpr int kP2D = BFP_P2_D, kP2S = kP2D + 1;                   // pairs in flight, slots
constexpr size_t kP2Smem = (size_t)kP2S * (kP2CW + 2 * kP2W) * 4 + kP2S * 8 + 128 + 64;

template <int MODE, bool FW, typename Op>
__device__ __forceinline__ void pro2_loop(const Op& op, const Vec& out, const WinParams& p,
                                          const WinCtx& c, Red& r, int R, char* smem) {
  const int l = out.l;
  const int64_t N = (int64_t)1 << l, Nc = N >> 1;
  const int64_t NZ = out.nz, Z0 = out.z0;
  const int strips = (int)(N / kP2W);
  const int chunks = (int)((NZ + R - 1) / R);
  int32_t* csl = reinterpret_cast<int32_t*>(smem);
  int32_t* ysl = csl + kP2S * kP2CW;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ysl + kP2S * 2 * kP2W);
  const int32_t* Cd = (const int32_t*)op.cv().data;
  const int32_t* Yd = (const int32_t*)op.yv().data;
  int32_t* O = (int32_t*)out.data;
  const int sc = op.shc(), sy = op.shy();
  const int kc_off = op.zp / 2;
  const int t = threadIdx.x, col = 2 * t + 4;
  int32_t mx = INT32_MIN, mn = INT32_MAX;
  uint64_t olo = 0, ohi = 0;
  uint32_t o32lo = 0, o32hi = 0;  // fast window: OR of z ^ sign(z) in two words
  const bool store = c.store_tmp;
  uint32_t parity = 0;
  for (int item = blockIdx.x; item < strips * chunks; item += gridDim.x) {
    const int strip = item % strips, ch = item / strips;
    const int64_t x0 = (int64_t)strip * kP2W, cx0 = x0 / 2;
    const int64_t k0 = (int64_t)ch * R;
    const int pairs = (int)(std::min<int64_t>(R, NZ - k0) / 2);
    const int64_t J0 = k0 / 2;
    auto crow = [&](int64_t J) { return Cd + (J + kc_off) * Nc + cx0 - 4; };
    auto issue = [&](int s) {
      const int slot = s % kP2S;
      uint64_t* b = &bar[slot];
      const int64_t J = J0 + s;
      const uint32_t cb = kP2CW * 4, yb = kP2W * 4;
      mbar_expect_tx(b, cb + (s == 0 ? cb : 0u) + (Op::kCorr ? 2 * yb : 0u));
      bulk_g2s(csl + slot * kP2CW, crow(J), cb, b);
      if (s == 0) bulk_g2s(csl + (kP2S - 1) * kP2CW, crow(J - 1), cb, b);
      if (Op::kCorr)
        for (int h = 0; h < 2; ++h)
          bulk_g2s(ysl + (slot * 2 + h) * kP2W, Yd + (2 * J + h) * N + x0, yb, b);
    };
    if (t == 0) {
      fence_proxy_async_smem();
      for (int s = 0; s < kP2D && s < pairs; ++s) issue(s);
    }
    const bool xpad = x0 + 4 * t + 3 == N - 1;
    // fast window: z = g Pg + y Py as two IMAD.WIDE, output pointer advanced per row, no pad
    // masking (a fine pad index has both coarse taps on the coarse pad; see pro3_loop)
    [[maybe_unused]] int Pg = 1, Py = 0;
    if constexpr (Op::kCorr) {
      Pg = op.swap ? 1 : op.P;
      Py = op.swap ? op.P : 1;
    }
    int32_t* dstp = O + 2 * J0 * N + x0 + 4 * t;
    int Sp[4] = {0, 0, 0, 0};
    auto S_of = [&](int sl, int S[4]) {
      const int32_t* row = csl + sl * kP2CW + col;
      const int a = row[-1] >> sc, b = row[0] >> sc, e = row[1] >> sc;
      S[0] = a + b;
      S[1] = 2 * b;
      S[2] = b + e;
      S[3] = 2 * e;
    };
    for (int s = 0; s < pairs; ++s) {
      const int slot = s % kP2S;
      mbar_wait(&bar[slot], (parity >> slot) & 1u);
      parity ^= 1u << slot;
      if (s == 0) S_of(kP2S - 1, Sp);
      int Sc[4];
      S_of(slot, Sc);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if constexpr (FW) {
          int y4[4] = {0, 0, 0, 0};
          if constexpr (Op::kCorr) {
            const int4 yy = *reinterpret_cast<const int4*>(ysl + (slot * 2 + h) * kP2W + 4 * t);
            y4[0] = yy.x >> sy, y4[1] = yy.y >> sy, y4[2] = yy.z >> sy, y4[3] = yy.w >> sy;
          }
          int tq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int g = h ? 2 * Sc[q] : Sp[q] + Sc[q];
            if constexpr (Op::kCorr) {
              const int64_t z = mad_wide(g, Pg, mul_wide(y4[q], Py));
              const uint32_t zl = (uint32_t)z, zh = (uint32_t)((uint64_t)z >> 32);
              if (MODE == MODE_QCOMP) {
                const uint32_t sg = (uint32_t)((int)zh >> 31);
                o32lo |= zl ^ sg;
                o32hi |= zh ^ sg;
              }
              tq[q] = (int)__funnelshift_r(zl, zh, c.rs);
            } else {
              if (MODE == MODE_QCOMP) o32lo |= (uint32_t)(g ^ (g >> 31));
              tq[q] = g >> c.rs;
            }
            mx = tq[q] > mx ? tq[q] : mx;
            mn = tq[q] < mn ? tq[q] : mn;
          }
          *reinterpret_cast<int4*>(dstp) = make_int4(tq[0], tq[1], tq[2], tq[3]);
          dstp += N;
          continue;
        }
        const int64_t j = 2 * (J0 + s) + h;  // local fine row
        int yv[4] = {0, 0, 0, 0};
        if (Op::kCorr) {
          const int4 y4 = *reinterpret_cast<const int4*>(ysl + (slot * 2 + h) * kP2W + 4 * t);
          yv[0] = y4.x >> sy, yv[1] = y4.y >> sy, yv[2] = y4.z >> sy, yv[3] = y4.w >> sy;
        }
        const bool rowpad = j + Z0 == N - 1;
        int32_t tt[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int g = h ? 2 * Sc[q] : Sp[q] + Sc[q];
          int64_t z = op.corr(g, yv[q]);
          if ((q == 3 && xpad) || rowpad) z = 0;
          if constexpr (FW) {
            if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
            tt[q] = (int32_t)__funnelshift_r((uint32_t)z, (uint32_t)((uint64_t)z >> 32), c.rs);
          } else if (MODE == MODE_NNQ) {
            tt[q] = (int32_t)shift_clamp<int64_t>(z, c.lam, p.w_out);
          } else {
            if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
            tt[q] = store ? store_shift<int32_t, int64_t>(z, c) : 0;
          }
          mx = tt[q] > mx ? tt[q] : mx;
          mn = tt[q] < mn ? tt[q] : mn;
        }
        *reinterpret_cast<int4*>(O + j * N + x0 + 4 * t) = make_int4(tt[0], tt[1], tt[2], tt[3]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) Sp[q] = Sc[q];
      __syncthreads();
      if (t == 0 && s + kP2D < pairs) {
        fence_proxy_async_smem();
        issue(s + kP2D);
      }
    }
    __syncthreads();
  }
  r.olo |= olo | ((uint64_t)o32hi << 32) | o32lo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

template <int MODE, typename Op>
__global__ void __launch_bounds__(kP2T, BFP_P2_MINB) pro2_win_kernel(Op op, Vec out, WinParams p, int R) {
  extern __shared__ __align__(128) char smem_raw[];
  char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  griddep_wait();
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, int32_t>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  if (op.narrow && need <= 63) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)kP2S * (kP2CW + 2 * kP2W) * 4);
    if (threadIdx.x == 0) {
      for (int k = 0; k < kP2S; ++k) mbar_init(&bar[k], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (MODE != MODE_NNQ && c.store_tmp && c.ls == 0 && c.rs < 32)
      pro2_loop<MODE, true>(op, out, p, c, r, R, smem);
    else
      pro2_loop<MODE, false>(op, out, p, c, r, R, smem);
  } else {
    grid_body<MODE, int32_t>(op, out, p, c, r, need);
  }
  griddep_launch_dependents();
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// Full weighting: a CTA owns 512 coarse columns and marches coarse rows K over the
// fine-row sums T_p (coarse K = T_{2K} + 2 T_{2K+1} + T_{2K+2}, T_{2K+2} carried).
constexpr int kR2T = 128, kR2W = 4 * kR2T;                       // coarse strip
constexpr int kR2FW = 2 * kR2W + 8;                              // fine row slot (words)
constexpr int kR2D = 2, kR2FS = 2 * kR2D + 3, kR2B = kR2D + 1;
constexpr size_t kR2Smem = (size_t)kR2FS * kR2FW * 4 + kR2B * 8 + 128 + 64;

template <int MODE, bool FW>
__device__ __forceinline__ void rst2_loop(const RestrictOp& op, const Vec& out,
                                          const WinParams& p, const WinCtx& c, Red& r, int R,
                                          char* smem) {
  const int lc = out.l;
  const int64_t Nc = (int64_t)1 << lc, Nf = Nc << 1;
  const int64_t NZ = out.nz, Z0 = out.z0;
  const int strips = (int)(Nc / kR2W);
  const int chunks = (int)((NZ + R - 1) / R);
  int32_t* fsl = reinterpret_cast<int32_t*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(fsl + kR2FS * kR2FW);
  const int32_t* F = (const int32_t*)op.r.data;
  int32_t* O = (int32_t*)out.data;
  const int sh = (int)op.sr;
  const int t = threadIdx.x;
  int32_t mx = INT32_MIN, mn = INT32_MAX;
  uint64_t olo = 0, ohi = 0;
  const bool store = c.store_tmp;
  uint32_t parity = 0;
  for (int item = blockIdx.x; item < strips * chunks; item += gridDim.x) {
    const int strip = item % strips, ch = item / strips;
    const int64_t cx0 = (int64_t)strip * kR2W;
    const int64_t K0 = (int64_t)ch * R;
    const int steps = (int)std::min<int64_t>(R, NZ - K0);
    auto issue = [&](int s) {
      uint64_t* b = &bar[s % kR2B];
      mbar_expect_tx(b, (uint32_t)kR2FW * 4 * (s == 0 ? 3u : 2u));
      for (int j = (s == 0 ? 0 : 1); j <= 2; ++j) {
        const int64_t f = 2 * (K0 + s) + j;  // local fine row
        bulk_g2s(fsl + (int)((f - 2 * K0) % kR2FS) * kR2FW, F + f * Nf + 2 * cx0 - 4,
                 kR2FW * 4, b);
      }
    };
    if (t == 0) {
      fence_proxy_async_smem();
      for (int s = 0; s <= kR2D && s < steps; ++s) issue(s);
    }
    auto T_of = [&](int64_t f, int T[4]) {
      const int32_t* row = fsl + (int)((f - 2 * K0) % kR2FS) * kR2FW + 8 * t + 4;
      const int4 a = *reinterpret_cast<const int4*>(row);
      const int4 b = *reinterpret_cast<const int4*>(row + 4);
      const int e = row[8] >> sh;
      const int v0 = a.x >> sh, v1 = a.y >> sh, v2 = a.z >> sh, v3 = a.w >> sh;
      const int v4 = b.x >> sh, v5 = b.y >> sh, v6 = b.z >> sh, v7 = b.w >> sh;
      T[0] = v0 + 2 * v1 + v2;
      T[1] = v2 + 2 * v3 + v4;
      T[2] = v4 + 2 * v5 + v6;
      T[3] = v6 + 2 * v7 + e;
    };
    const bool xpad = cx0 + 4 * t + 3 == Nc - 1;
    int Tp[4] = {0, 0, 0, 0};
    for (int s = 0; s < steps; ++s) {
      const int64_t Kc = K0 + s;
      mbar_wait(&bar[s % kR2B], (parity >> (s % kR2B)) & 1u);
      parity ^= 1u << (s % kR2B);
      if (s == 0) T_of(2 * Kc, Tp);
      int T1[4], T2[4];
      T_of(2 * Kc + 1, T1);
      T_of(2 * Kc + 2, T2);
      const bool rowpad = Kc + Z0 == Nc - 1;
      int32_t tt[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t z = (int64_t)Tp[q] + 2 * (int64_t)T1[q] + (int64_t)T2[q];
        if ((q == 3 && xpad) || rowpad) z = 0;
        if constexpr (FW) {
          if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
          tt[q] = (int32_t)__funnelshift_r((uint32_t)z, (uint32_t)((uint64_t)z >> 32), c.rs);
        } else if (MODE == MODE_NNQ) {
          tt[q] = (int32_t)shift_clamp<int64_t>(z, c.lam, p.w_out);
        } else {
          if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
          tt[q] = store ? store_shift<int32_t, int64_t>(z, c) : 0;
        }
        mx = tt[q] > mx ? tt[q] : mx;
        mn = tt[q] < mn ? tt[q] : mn;
      }
      *reinterpret_cast<int4*>(O + Kc * Nc + cx0 + 4 * t) = make_int4(tt[0], tt[1], tt[2], tt[3]);
#pragma unroll
      for (int q = 0; q < 4; ++q) Tp[q] = T2[q];
      __syncthreads();
      if (t == 0 && s + kR2D + 1 < steps) {
        fence_proxy_async_smem();
        issue(s + kR2D + 1);
      }
    }
    __syncthreads();
  }
  r.olo |= olo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

template <int MODE>
__global__ void __launch_bounds__(kR2T, 8) rst2_win_kernel(RestrictOp op, Vec out, WinParams p,
                                                           int R) {
  extern __shared__ __align__(128) char smem_raw[];
  char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  griddep_wait();
  int64_t need = 0;
  WinCtx c;
  block_setup<RestrictOp, int32_t>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  // row sums T_p (weights 4) in int32: eff_bits(r) <= 29, need = eff + 6 <= 35 in 2-D
  if (op.sr < 32 && need <= 35 && op.gs == 0) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)kR2FS * kR2FW * 4);
    if (threadIdx.x == 0) {
      for (int k = 0; k < kR2B; ++k) mbar_init(&bar[k], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (MODE != MODE_NNQ && c.store_tmp && c.ls == 0 && c.rs < 32)
      rst2_loop<MODE, true>(op, out, p, c, r, R, smem);
    else
      rst2_loop<MODE, false>(op, out, p, c, r, R, smem);
  } else {
    grid_body<MODE, int32_t>(op, out, p, c, r, need);
  }
  griddep_launch_dependents();
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// one exact row per thread, __int128 accumulation (generic CSR / fixed rows)
template <typename M, typename Op>
__global__ void __launch_bounds__(kThreads) flat_win_kernel(Op op, Vec out, WinParams p) {
  griddep_wait();
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, M>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  if (need > 127) {
    r.err = ERR_WIDTH;
  } else {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < out.nlog; i += stride) {
      i128 z = op.template eval1<M>(i);
      M t;
      if (p.mode == MODE_NNQ) {
        t = (M)shift_clamp<i128>(z, c.lam, p.w_out);
      } else {
        if (p.mode == MODE_QCOMP) or_mag<i128>(z, r.olo, r.ohi);
        t = c.store_tmp ? store_shift<M, i128>(z, c) : (M)0;
      }
      ((M*)out.data)[i] = t;
      r.val((int64_t)t);
    }
  }
  griddep_launch_dependents();
  window_reduce(r, out.hdr, p, c, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}


namespace bfp {

static inline int check_window(const WinParams& p, const bfp_vec_s* out) {
  const int sb = out->ebytes * 8;
  if (p.w_out < 1 || p.w_out > sb) return BFP_ERR_ARG;
  if (p.mode == MODE_QCOMP && (p.w_tmp < p.w_out || p.w_tmp > 64)) return BFP_ERR_ARG;
  if (p.gamma.literal && p.gamma.lm <= 0) return BFP_ERR_ARG;
  return BFP_OK;
}

// tiny levels run as one block (finalize and qcomp recompute in the same launch); above
// two 4-groups per thread a multi-block pass plus the deferred finalize is faster
// (measured: tools/op_latency.py)
#ifndef BFP_SINGLE_BLOCK_GROUPS
#define BFP_SINGLE_BLOCK_GROUPS 512
#endif
constexpr int64_t kSingleBlockGroups = BFP_SINGLE_BLOCK_GROUPS;
// up to this many 4-groups, a multi-block qcomp pass 1 is finished by grid_finish_kernel
#ifndef BFP_FINISH_GROUPS
#define BFP_FINISH_GROUPS (1 << 13)  // (a one-block recompute of 32k points: ~20 us, rare)
#endif
constexpr int64_t kFinishGroups = BFP_FINISH_GROUPS;

// launch a grid-windowed op: nnqcomp (one pass) or qcomp (pass 1 + recompute)
template <typename Op>
static inline int launch_grid(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  // tiny levels: one block (finalized without cross-block atomics)
  const int64_t groups = out->span / 4;
  const int b = groups <= kSingleBlockGroups ? 1 : blocks_for(groups);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    const int nb = pp.mode == MODE_RECOMPUTE ? std::min(b, 2 * sm_count()) : b;
    if (out->ebytes == 4) {
      if (pp.mode == MODE_QCOMP)
        launch_pdl(grid_win_kernel<MODE_QCOMP, int32_t, Op>, nb, kThreads, 0, s, op, o, pp);
      else if (pp.mode == MODE_NNQ)
        launch_pdl(grid_win_kernel<MODE_NNQ, int32_t, Op>, nb, kThreads, 0, s, op, o, pp);
      else
        launch_pdl(grid_win_kernel<MODE_RECOMPUTE, int32_t, Op>, nb, kThreads, 0, s, op, o, pp);
    } else {
      if (pp.mode == MODE_QCOMP)
        launch_pdl(grid_win_kernel<MODE_QCOMP, int64_t, Op>, nb, kThreads, 0, s, op, o, pp);
      else if (pp.mode == MODE_NNQ)
        launch_pdl(grid_win_kernel<MODE_NNQ, int64_t, Op>, nb, kThreads, 0, s, op, o, pp);
      else
        launch_pdl(grid_win_kernel<MODE_RECOMPUTE, int64_t, Op>, nb, kThreads, 0, s, op, o, pp);
    }
    count_launch();
    count_family(FAM_GRID);
  };
  p.defer = defer_ok(p, b);
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p);
    cudaEventRecord(ev.second, s);
  } else {
    go(p);
  }
  // mid-size grids: finalize + (rare) recompute by one block in one launch
  if (p.defer && p.mode == MODE_QCOMP && !g_skip_recompute && !p.part && groups <= kFinishGroups) {
    p.defer = 0;
    if (out->ebytes == 4)
      launch_pdl(grid_finish_kernel<int32_t, Op>, 1, kThreads, 0, s, op, o, p);
    else
      launch_pdl(grid_finish_kernel<int64_t, Op>, 1, kThreads, 0, s, op, o, p);
    count_launch();
    return last_launch();
  }
  if (p.defer) launch_deferred_finalize(o, p, out->ebytes * 8, s);
  p.defer = 0;
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part && b > 1) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}


// tiled TMA descriptor of a 3-D grid vector (driver entry point through the runtime)
static inline bool encode_b3(CUtensorMap* m, const Vec& v, int bw, int bh) {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return false;
    fn = reinterpret_cast<EncodeFn>(f);
  }
  const uint64_t N = (uint64_t)1 << v.l, eb = (uint64_t)v.ebytes;
  char* base = (char*)v.data - 2 * N * N * eb;  // two halo planes before plane 0
  const cuuint64_t dims[3] = {N, N, (cuuint64_t)v.nz + 4};
  const cuuint64_t strides[2] = {N * eb, N * N * eb};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, eb == 4 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_INT64, 3, base,
            dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, typename Op>
static inline int launch_bulk3(const Op& op, bfp_vec_s* out, const WinParams& p0,
                               cudaStream_t s) {
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  B3Maps tm;
  if (!encode_b3(&tm.x, op.sv(), kB3XW, kB3XR) || !encode_b3(&tm.y, op.yv2(), kB3W, kB3H))
    return BFP_ERR_CUDA;
  const int64_t N = int64_t(1) << out->l;
  constexpr size_t smem = b3_smem<T, Op>();
  static std::atomic<int> occ_dev[kMaxDev];  // per instantiation and device
  const int occ = per_device(occ_dev, [&] {
    int o = 0;
    for (auto fn : {bulk3_win_kernel<MODE_QCOMP, T, Op>, bulk3_win_kernel<MODE_NNQ, T, Op>,
                    bulk3_win_kernel<MODE_RECOMPUTE, T, Op>})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, bulk3_win_kernel<MODE_QCOMP, T, Op>, kB3T,
                                                  smem);
    return std::max(o, 1);
  });
  const int64_t tiles = (N / kB3W) * (N / kB3H), ctas = (int64_t)sm_count() * occ, NZ = out->nz;
  const int R = march_R(tiles, NZ, ctas, 4, 1, 2);
  const int64_t items = tiles * ((NZ + R - 1) / R);
  const int b = (int)std::min<int64_t>(items, ctas);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    if (pp.mode == MODE_QCOMP)
      launch_pdl(bulk3_win_kernel<MODE_QCOMP, T, Op>, b, kB3T, smem, s, op, o, pp, R, tm);
    else if (pp.mode == MODE_NNQ)
      launch_pdl(bulk3_win_kernel<MODE_NNQ, T, Op>, b, kB3T, smem, s, op, o, pp, R, tm);
    else
      launch_pdl(bulk3_win_kernel<MODE_RECOMPUTE, T, Op>, b, kB3T, smem, s, op, o, pp, R, tm);
    count_launch();
    count_family(FAM_BULK3);
  };
  p.defer = defer_ok(p, b);
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p);
    cudaEventRecord(ev.second, s);
  } else {
    go(p);
  }
  if (p.defer) launch_deferred_finalize(o, p, out->ebytes * 8, s);
  p.defer = 0;
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}

// 3-D prolongation (+ correction), int32 storage, N >= 128: the tiled-TMA pair march
template <typename T, typename Op>
static inline int launch_pro3(const Op& op, bfp_vec_s* out, const WinParams& p0,
                              cudaStream_t s) {
  constexpr size_t kP3Smem = p3_smem<T, Op>();
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  P3Maps tm;
  if (!encode_b3(&tm.c, op.cv(), kP3CW, kP3CH)) return BFP_ERR_CUDA;
  if (Op::kCorr) {
    if (!encode_b3(&tm.y, op.yv(), kP3W, kP3H)) return BFP_ERR_CUDA;
  } else {
    tm.y = tm.c;  // unused
  }
  const int64_t N = int64_t(1) << out->l;
  static std::atomic<int> occ_dev[kMaxDev];  // per instantiation and device
  const int occ = per_device(occ_dev, [&] {
    int o = 0;
    for (auto fn : {pro3_win_kernel<MODE_QCOMP, T, Op>, pro3_win_kernel<MODE_NNQ, T, Op>,
                    pro3_win_kernel<MODE_RECOMPUTE, T, Op>})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kP3Smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, pro3_win_kernel<MODE_QCOMP, T, Op>, kP3T + 32,
                                                  kP3Smem);
    return std::max(o, 1);
  });
  const int64_t tiles = (N / kP3W) * (N / kP3H), ctas = (int64_t)sm_count() * occ, NZ = out->nz;
  const int R = march_R(tiles, NZ, ctas, 4, 2, 1);  // whole fine-plane pairs
  const int64_t items = tiles * ((NZ + R - 1) / R);
  const int b = (int)std::min<int64_t>(items, ctas);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    if (pp.mode == MODE_QCOMP)
      launch_pdl(pro3_win_kernel<MODE_QCOMP, T, Op>, b, kP3T + 32, kP3Smem, s, op, o, pp, R, tm);
    else if (pp.mode == MODE_NNQ)
      launch_pdl(pro3_win_kernel<MODE_NNQ, T, Op>, b, kP3T + 32, kP3Smem, s, op, o, pp, R, tm);
    else
      launch_pdl(pro3_win_kernel<MODE_RECOMPUTE, T, Op>, b, kP3T + 32, kP3Smem, s, op, o, pp, R, tm);
    count_launch();
    count_family(FAM_PRO3);
  };
  p.defer = defer_ok(p, b);
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p);
    cudaEventRecord(ev.second, s);
  } else {
    go(p);
  }
  if (p.defer) launch_deferred_finalize(o, p, out->ebytes * 8, s);
  p.defer = 0;
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}

// 3-D full-weighting restriction, int32 storage, coarse N >= 64: the tiled-TMA march
template <typename T>
static inline int launch_rst3(const RestrictOp& op, bfp_vec_s* out, const WinParams& p0,
                              cudaStream_t s) {
  constexpr size_t kR3Smem = r3_smem<T>();
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  R3Maps tm;
  if (!encode_b3(&tm.f, op.r, kR3FW, kR3FH)) return BFP_ERR_CUDA;
  const int64_t Nc = int64_t(1) << out->l;
  static std::atomic<int> occ_dev[kMaxDev];  // per instantiation and device
  const int occ = per_device(occ_dev, [&] {
    int o = 0;
    for (auto fn : {rst3_win_kernel<MODE_QCOMP, T>, rst3_win_kernel<MODE_NNQ, T>,
                    rst3_win_kernel<MODE_RECOMPUTE, T>})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kR3Smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, rst3_win_kernel<MODE_QCOMP, T>, kR3T,
                                                  kR3Smem);
    return std::max(o, 1);
  });
  const int64_t tiles = (Nc / kR3W) * (Nc / kR3H), ctas = (int64_t)sm_count() * occ, NZ = out->nz;
  const int R = march_R(tiles, NZ, ctas, 2, 1, 1);
  const int64_t items = tiles * ((NZ + R - 1) / R);
  const int b = (int)std::min<int64_t>(items, ctas);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    if (pp.mode == MODE_QCOMP)
      launch_pdl(rst3_win_kernel<MODE_QCOMP, T>, b, kR3T, kR3Smem, s, op, o, pp, R, tm);
    else if (pp.mode == MODE_NNQ)
      launch_pdl(rst3_win_kernel<MODE_NNQ, T>, b, kR3T, kR3Smem, s, op, o, pp, R, tm);
    else
      launch_pdl(rst3_win_kernel<MODE_RECOMPUTE, T>, b, kR3T, kR3Smem, s, op, o, pp, R, tm);
    count_launch();
    count_family(FAM_RST3);
  };
  p.defer = defer_ok(p, b);
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p);
    cudaEventRecord(ev.second, s);
  } else {
    go(p);
  }
  if (p.defer) launch_deferred_finalize(o, p, out->ebytes * 8, s);
  p.defer = 0;
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}

// one-wave launch of a row/plane-march transfer kernel (pass 1 + recompute unless partial)
template <typename K0, typename K1, typename K2, typename... Args>
static inline int launch_wave(int fam, K0 kq, K1 kn, K2 kr, int threads, size_t smem,
                              int64_t units, int64_t NZ, int Rmin, bool even, bfp_vec_s* out,
                              const WinParams& p0, cudaStream_t s, Args... args) {
  int rc = check_window(p0, out);
  if (rc) return rc;
  static_assert(sizeof...(Args) >= 1, "kernel arguments");
  static std::atomic<int> occ_dev[kMaxDev];  // per instantiation and device
  const int occ = per_device(occ_dev, [&] {
    int o = 0;
    cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kq, threads, smem);
    return std::max(o, 1);
  });
  const int64_t ctas = (int64_t)sm_count() * occ;
  const int R = march_R(units, NZ, ctas, Rmin, even ? 2 : 1, 1);
  const int64_t items = units * ((NZ + R - 1) / R);
  const int b = (int)std::min<int64_t>(items, ctas);
  Vec o = view(out);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    if (pp.mode == MODE_QCOMP)
      launch_pdl(kq, b, threads, smem, s, args..., o, pp, R);
    else if (pp.mode == MODE_NNQ)
      launch_pdl(kn, b, threads, smem, s, args..., o, pp, R);
    else
      launch_pdl(kr, b, threads, smem, s, args..., o, pp, R);
    count_launch();
    count_family(fam);
  };
  p.defer = defer_ok(p, b);
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p);
    cudaEventRecord(ev.second, s);
  } else {
    go(p);
  }
  if (p.defer) launch_deferred_finalize(o, p, out->ebytes * 8, s);
  p.defer = 0;
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}
template <typename Op>
static inline int launch_pro2(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
  const int64_t N = int64_t(1) << out->l;
  return launch_wave(FAM_PRO2, pro2_win_kernel<MODE_QCOMP, Op>, pro2_win_kernel<MODE_NNQ, Op>,
                     pro2_win_kernel<MODE_RECOMPUTE, Op>, kP2T, kP2Smem, N / kP2W, out->nz, 4,
                     true, out, p0, s, op);
}
static inline int launch_rst2(const RestrictOp& op, bfp_vec_s* out, const WinParams& p0,
                              cudaStream_t s) {
  const int64_t Nc = int64_t(1) << out->l;
  return launch_wave(FAM_RST2, rst2_win_kernel<MODE_QCOMP>, rst2_win_kernel<MODE_NNQ>,
                     rst2_win_kernel<MODE_RECOMPUTE>, kR2T, kR2Smem, Nc / kR2W, out->nz, 2,
                     false, out, p0, s, op);
}

// stencil ops on int32 grids of 2-D / 3-D with N >= 128 use the register march
template <typename Op>
static inline int launch_bulk(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  const int64_t N = int64_t(1) << out->l;
  static std::atomic<int> occ_dev[kMaxDev];  // per instantiation and device
  const int occ = per_device(occ_dev, [&] {
    int o = 0;
    for (auto fn : {bulk_win_kernel<MODE_QCOMP, Op>, bulk_win_kernel<MODE_NNQ, Op>,
                    bulk_win_kernel<MODE_RECOMPUTE, Op>})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBulkSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, bulk_win_kernel<MODE_QCOMP, Op>, kBulkT + 32,
                                                  kBulkSmem);
    return std::max(o, 1);
  });
  const int64_t strips = N / kBulkW, ctas = (int64_t)sm_count() * occ;
  const int64_t NZ = out->nz;
  const int R = march_R(strips, NZ, ctas, 8, 1, 2);
  const int64_t items = strips * ((NZ + R - 1) / R);
  const int b = (int)std::min<int64_t>(items, ctas);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    if (pp.mode == MODE_QCOMP)
      launch_pdl(bulk_win_kernel<MODE_QCOMP, Op>, b, kBulkT + 32, kBulkSmem, s, op, o, pp, R);
    else if (pp.mode == MODE_NNQ)
      launch_pdl(bulk_win_kernel<MODE_NNQ, Op>, b, kBulkT + 32, kBulkSmem, s, op, o, pp, R);
    else
      launch_pdl(bulk_win_kernel<MODE_RECOMPUTE, Op>, b, kBulkT + 32, kBulkSmem, s, op, o, pp, R);
    count_launch();
    count_family(FAM_BULK2);
  };
  p.defer = defer_ok(p, b);
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p);
    cudaEventRecord(ev.second, s);
  } else {
    go(p);
  }
  if (p.defer) launch_deferred_finalize(o, p, out->ebytes * 8, s);
  p.defer = 0;
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}



template <typename Op>
static inline int launch_march(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
  // level 7 (2M points, L2-resident) is faster on the one-group-per-thread grid kernel
  static const int b3_min = min_level("BFP_B3_MIN_L", 8);  // kB3W = 128 columns
  if (g_use_bulk && out->dim == 3 && (int64_t(1) << out->l) >= kB3W && out->l >= b3_min)
    return out->ebytes == 4 ? launch_bulk3<int32_t>(op, out, p0, s)
                            : launch_bulk3<int64_t>(op, out, p0, s);
  if (out->ebytes != 4 || out->dim < 2 || (int64_t(1) << out->l) < kMarchMinN)
    return launch_grid(op, out, p0, s);
  static const int b2_min = min_level("BFP_B2_MIN_L", 10);  // kBulkW = 1024 columns
  if (g_use_bulk && out->dim == 2 && (int64_t(1) << out->l) >= kBulkW && out->l >= b2_min)
    return launch_bulk(op, out, p0, s);
  // below the bulk pipeline's size a resident wave holds every 4-group with one group per
  // thread: the generic grid kernel issues all of a group's loads at once, where the march
  // (>= 4 dependent steps per thread) is latency-bound on these L2-resident levels
#ifdef BFP_AB_ENV
  static const bool march_mid = getenv("BFP_MARCH_MID") != nullptr;  // A/B switch
#else
  constexpr bool march_mid = false;
#endif
  if (!march_mid && out->dim == 2) return launch_grid(op, out, p0, s);
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  const int64_t N = int64_t(1) << out->l, GX = N / 4, rows = out->dim == 3 ? N : 1;
  static std::atomic<int> occ2_dev[kMaxDev], occ3_dev[kMaxDev];
  const int occ = out->dim == 2 ? per_device(occ2_dev, [] {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, march_win_kernel<MODE_QCOMP, 2, Op>,
                                                kThreads, 0);
    return std::max(o, 1);
  }) : per_device(occ3_dev, [] {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, march_win_kernel<MODE_QCOMP, 3, Op>,
                                                kThreads, 0);
    return std::max(o, 1);
  });
  // one balanced resident wave: every thread marches R steps (last chunk shorter)
  const int64_t slots = (int64_t)sm_count() * occ * kThreads;
  const int64_t NZ = out->nz;
  int R = (int)std::max<int64_t>(4, (GX * rows * NZ + slots - 1) / slots);
  const int64_t items = GX * rows * ((NZ + R - 1) / R);
  const int b = (int)std::max<int64_t>(1, std::min<int64_t>((items + kThreads - 1) / kThreads,
                                                            (int64_t)sm_count() * occ));
  WinParams p = p0;
  auto go = [&](const WinParams& pp, int nb) {
    if (out->dim == 2) {
      if (pp.mode == MODE_QCOMP)
        launch_pdl(march_win_kernel<MODE_QCOMP, 2, Op>, nb, kThreads, 0, s, op, o, pp, R);
      else if (pp.mode == MODE_NNQ)
        launch_pdl(march_win_kernel<MODE_NNQ, 2, Op>, nb, kThreads, 0, s, op, o, pp, R);
      else
        launch_pdl(march_win_kernel<MODE_RECOMPUTE, 2, Op>, nb, kThreads, 0, s, op, o, pp, R);
    } else {
      if (pp.mode == MODE_QCOMP)
        launch_pdl(march_win_kernel<MODE_QCOMP, 3, Op>, nb, kThreads, 0, s, op, o, pp, R);
      else if (pp.mode == MODE_NNQ)
        launch_pdl(march_win_kernel<MODE_NNQ, 3, Op>, nb, kThreads, 0, s, op, o, pp, R);
      else
        launch_pdl(march_win_kernel<MODE_RECOMPUTE, 3, Op>, nb, kThreads, 0, s, op, o, pp, R);
    }
    count_launch();
    count_family(FAM_MARCH);
  };
  p.defer = defer_ok(p, b);
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p, b);
    cudaEventRecord(ev.second, s);
  } else {
    go(p, b);
  }
  if (p.defer) launch_deferred_finalize(o, p, out->ebytes * 8, s);
  p.defer = 0;
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p, b);
  }
  return last_launch();
}

template <typename Op>
static inline int launch_flat(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  const int b = blocks_for(out->nlog);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    if (out->ebytes == 4)
      launch_pdl(flat_win_kernel<int32_t, Op>, b, kThreads, 0, s, op, o, pp);
    else
      launch_pdl(flat_win_kernel<int64_t, Op>, b, kThreads, 0, s, op, o, pp);
    count_launch();
    count_family(FAM_FLAT);
  };
  p.defer = defer_ok(p, b);
  go(p);
  if (p.defer) launch_deferred_finalize(o, p, out->ebytes * 8, s);
  p.defer = 0;
  if (p.mode == MODE_QCOMP && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}

static inline bool same_grid(const bfp_vec_s* a, const bfp_vec_s* b) {
  return a->dim == b->dim && a->l == b->l && a->ebytes == b->ebytes && a->span == b->span &&
         a->nlog == b->nlog && a->z0 == b->z0 && a->nz == b->nz;
}
static inline bool full_grid(const bfp_vec_s* a) { return a->dim == 0 || a->nz == (1 << a->l); }

}  // namespace bfp
