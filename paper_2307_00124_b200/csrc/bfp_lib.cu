// bfp_lib.cu -- sm_100a kernels of the BFP hot path and the C-ABI
// (include/bfpmg_b200.h).  No CPU fallback: every entry point either launches
// device work or fails with a status code.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "bfp_internal.h"
#include "bfp_bulk.cuh"

using namespace bfpdev;

namespace {
std::atomic<int64_t> g_launches{0};
bool g_pdl = true;  // programmatic dependent launch for the windowed kernels
bool g_skip_recompute = false;  // measurement only: pass-1 alone (flags must be clear)

// Launch with Programmatic Dependent Launch: the grid may be scheduled while the
// previous kernel in the stream drains; the kernel executes griddepcontrol.wait
// before touching any data, so stream semantics are unchanged.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
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
// measurement hooks: (start, end) event pairs around pass-1 / nnqcomp kernels
bool g_prof = false;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_ev;
size_t g_ev_used = 0;
std::pair<cudaEvent_t, cudaEvent_t> prof_pair() {
  if (g_ev_used == g_ev.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    g_ev.emplace_back(a, b);
  }
  return g_ev[g_ev_used++];
}
constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 8;

int blocks_for(int64_t work) {
  int64_t b = (work + kThreads - 1) / kThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, kMaxBlocks));
}
int cuda_status(cudaError_t e) { return e == cudaSuccess ? BFP_OK : BFP_ERR_CUDA; }
int last_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "bfpmg_b200: launch failed: %s\n", cudaGetErrorString(e));
    return BFP_ERR_CUDA;
  }
  return BFP_OK;
}
}  // namespace

// ===========================================================================
// kernels

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
template <int MODE, typename M, typename Op, typename A, bool NC = true>
__device__ __forceinline__ void grid_loop(Op& op, const Vec& out, const WinParams& p,
                                          const WinCtx& c, Red& r) {
  const int64_t ngroups = out.n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  M mx = Lim<M>::lo, mn = Lim<M>::hi;
  uint64_t olo = 0, ohi = 0;
  const bool store = c.store_tmp;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += stride) {
    A z[4];
    op.template eval4<M, A, NC>(g * 4, z);
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
  }
  r.olo |= olo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;  // sentinels stay neutral
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

template <int MODE, typename M, typename Op, bool NC = true>
__device__ __forceinline__ void grid_body(Op& op, const Vec& out, const WinParams& p,
                                          const WinCtx& c, Red& r, int64_t need) {
  if (need > 127)
    r.err = ERR_WIDTH;
  else if (need <= 63)
    grid_loop<MODE, M, Op, int64_t, NC>(op, out, p, c, r);
  else
    grid_loop<MODE, M, Op, i128, NC>(op, out, p, c, r);
}

// One windowed pass over a grid (or 4-padded flat) output: qcomp pass 1,
// nnqcomp, or the qcomp recompute pass, selected by p.mode.
// The op setup and the gamma rule are uniform per launch: one thread evaluates
// them from the device headers and broadcasts through shared memory.
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
  if (threadIdx.x == 0) {
    int64_t e_star = 0, nd = 0;
    Op o = op;
    o.setup(e_star, nd);
    WinCtx cc;
    win_setup(p, out.hdr, e_star, 8 * (int)sizeof(M), cc);
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
  griddep_wait();
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, M>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  grid_body<MODE, M>(op, out, p, c, r, need);
  griddep_launch_dependents();
  reduce_and_finalize(r, out.hdr, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
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
template <int MODE, int DIM, typename Op>
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
      int64_t z = op.point(g, C[k], Y[k]);
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

template <int MODE, int DIM, typename Op>
__device__ __forceinline__ void march_loop(const Op& op, const Vec& out, const WinParams& p,
                                           const WinCtx& c, Red& r, int R) {
  const int l = out.l;
  const int64_t N = (int64_t)1 << l, GX = N >> 2;
  const int64_t S = DIM == 2 ? N : N * N;  // march stride
  const int64_t rows = DIM == 3 ? N : 1;
  const int64_t NZ = out.nz, Z0 = out.z0;  // local planes along the march axis, slab offset
  const int64_t chunks = (NZ + R - 1) / R;
  const int64_t items = GX * rows * chunks;
  MarchStep<MODE, DIM, Op> st{op, p, c, S, N, op.shs(), op.shy(), (int)(threadIdx.x & 31),
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
  if (op.narrow && need <= 63)
    march_loop<MODE, DIM>(op, out, p, c, r, R);
  else
    grid_body<MODE, int32_t>(op, out, p, c, r, need);  // exact generic fallback
  griddep_launch_dependents();
  reduce_and_finalize(r, out.hdr, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// ---------------------------------------------------------------------------
// 2-D stencil ops through the bulk-async shared-memory pipeline (bfp_bulk.cuh)

template <int MODE, bool SHIFT, bool SWAP, typename Op>
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
  const int32_t* X = (const int32_t*)op.sv().data;
  const int32_t* Y = (const int32_t*)op.yv2().data;
  int32_t* O = (int32_t*)out.data;
  const int sx = SHIFT ? op.shs() : 0, sy = SHIFT ? op.shy() : 0;
  const int t = threadIdx.x;
  int32_t mx = INT32_MIN, mn = INT32_MAX;
  uint64_t olo = 0, ohi = 0;
  const bool store = c.store_tmp;
  const uint32_t tx_bytes = (uint32_t)(kBulkXW + kBulkW) * 4;
  uint32_t parity = 0;  // bit k: phase parity of bar[k]
  for (int item = blockIdx.x; item < strips * chunks; item += gridDim.x) {
    const int strip = item % strips, ch = item / strips;
    const int64_t c0 = (int64_t)strip * kBulkW;
    const int j0 = ch * R;
    const int rows = (int)std::min<int64_t>(R, NZ - j0);
    // source row clamp: rows past the slab read its back halo row (zeros or exchanged)
    auto xsrc = [&](int64_t row) { return X + (row > NZ ? NZ : row) * N + c0 - 4; };
    auto ysrc = [&](int64_t row) { return Y + (row > NZ ? NZ : row) * N + c0; };
    if (t == 0) {
      fence_proxy_async_smem();  // previous item's generic reads of the slots
      // prologue: x rows j0-1, j0 with group j0 (x row j0+1, y row j0) on bar[j0 % YS];
      // then groups j0+1 .. j0+D
      for (int g = 0; g <= kBulkD && g < rows; ++g) {
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
    }
    const bool xpad = c0 + 4 * t + 3 == N - 1;
    const int lane = t & 31;
    // running ring indices (no 64-bit modulo in the step loop)
    int sp = (int)((j0 - 1 + kBulkXS) % kBulkXS), sc = (int)(j0 % kBulkXS);
    int sn = (int)((j0 + 1) % kBulkXS), sy_ = (int)(j0 % kBulkYS);
    for (int s = 0; s < rows; ++s) {
      const int64_t j = j0 + s;
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
      int32_t tt[4];
      const bool rowpad = j + Z0 == N - 1;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int g = 4 * C[k] - (nb[k] + U[k] + Dn[k]);
        int64_t z = op.template point_t<SWAP>(g, C[k], Yv[k]);
        if (k == 3 && xpad) z = 0;
        if (rowpad) z = 0;
        if (MODE == MODE_NNQ) {
          tt[k] = (int32_t)shift_clamp<int64_t>(z, c.lam, p.w_out);
        } else {
          if (MODE == MODE_QCOMP) or_mag<int64_t>(z, olo, ohi);
          tt[k] = store ? store_shift<int32_t, int64_t>(z, c) : 0;
        }
        mx = tt[k] > mx ? tt[k] : mx;
        mn = tt[k] < mn ? tt[k] : mn;
      }
      *reinterpret_cast<int4*>(O + j * N + c0 + 4 * t) = make_int4(tt[0], tt[1], tt[2], tt[3]);
      // ring slots freed by this step: x row j-1 (slot sp) and y row j / its barrier (slot sy_)
      const int free_x = sp, free_y = sy_;
      sp = sc;
      sc = sn;
      sn = sn + 1 == kBulkXS ? 0 : sn + 1;
      sy_ = sy_ + 1 == kBulkYS ? 0 : sy_ + 1;
      __syncthreads();  // slots of x row j-1 and y row j are free
      if (t == 0 && s + kBulkD + 1 < rows) {
        // next group: x row tr+1 -> slot (j-1) % XS, y row tr -> slot j % YS, tr = j+D+1
        const int64_t tr = j + kBulkD + 1;
        uint64_t* bb = &bar[free_y];
        fence_proxy_async_smem();
        mbar_expect_tx(bb, tx_bytes);
        bulk_g2s(xsl + free_x * kBulkXW, xsrc(tr + 1), kBulkXW * 4, bb);
        bulk_g2s(ysl + free_y * kBulkW, ysrc(tr), kBulkW * 4, bb);
      }
    }
    __syncthreads();
  }
  r.olo |= olo;
  r.ohi |= ohi;
  r.mx = (int64_t)mx > r.mx ? (int64_t)mx : r.mx;
  r.mn = (int64_t)mn < r.mn ? (int64_t)mn : r.mn;
}

template <int MODE, typename Op>
__global__ void __launch_bounds__(kBulkT, 4) bulk_win_kernel(Op op, Vec out, WinParams p, int R) {
  griddep_wait();
  extern __shared__ __align__(128) char smem[];
  int64_t need = 0;
  WinCtx c;
  block_setup<Op, int32_t>(op, out, p, c, need);
  if (c.skip) return;
  Red r;
  r.init();
  if (op.narrow && need <= 63) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)(kBulkXS * kBulkXW + kBulkYS * kBulkW) * 4);
    if (threadIdx.x == 0) {
      for (int k = 0; k < kBulkYS; ++k) mbar_init(&bar[k], 1);
      mbar_fence_init();
    }
    __syncthreads();
    const bool sh = (op.shs() | op.shy()) != 0, sw = op.swapped();
    if (!sh && !sw)
      bulk_loop<MODE, false, false>(op, out, p, c, r, R, smem);
    else if (sh && !sw)
      bulk_loop<MODE, true, false>(op, out, p, c, r, R, smem);
    else if (!sh)
      bulk_loop<MODE, false, true>(op, out, p, c, r, R, smem);
    else
      bulk_loop<MODE, true, true>(op, out, p, c, r, R, smem);
  } else {
    grid_body<MODE, int32_t>(op, out, p, c, r, need);  // exact generic fallback
  }
  griddep_launch_dependents();
  reduce_and_finalize(r, out.hdr, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// ---------------------------------------------------------------------------
// Fused coarse levels: one CTA interprets a list of windowed ops (the part of a
// V-cycle / FMG on levels below the fusion threshold) with block-level
// reductions and finalizers instead of one or two kernel launches per op.  The
// per-op semantics are the same functions as the multi-block kernels
// (setup, win_setup, eval4, win_finalize), so results are bit-identical.

template <typename Fin>
__device__ inline void block_reduce_finalize(Red& r, Fin fin) {
  __shared__ unsigned long long s_lo[32], s_hi[32];
  __shared__ int s_err[32];
  __shared__ long long s_mx[32], s_mn[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  uint64_t lo = shfl_or64(r.olo), hi = shfl_or64(r.ohi);
  int err = __reduce_or_sync(0xffffffffu, r.err);
  int64_t mx = shfl_max64(r.mx), mn = shfl_min64(r.mn);
  if (lane == 0) {
    s_lo[wid] = lo;
    s_hi[wid] = hi;
    s_err[wid] = err;
    s_mx[wid] = mx;
    s_mn[wid] = mn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) {
      lo |= s_lo[w];
      hi |= s_hi[w];
      err |= s_err[w];
      mx = s_mx[w] > mx ? s_mx[w] : mx;
      mn = s_mn[w] < mn ? s_mn[w] : mn;
    }
    const int bits = (hi ? 64 + bitlen64(hi) : bitlen64(lo)) + 1;
    fin(bits, mx, mn, err);
  }
  __syncthreads();
}

template <int MODE, typename M, typename Op>
__device__ __forceinline__ void fused_pass(Op& op, const Vec& out, const WinParams& p,
                                           const WinCtx& c, int64_t need) {
  Red r;
  r.init();
  grid_body<MODE, M, Op, false>(op, out, p, c, r, need);
  block_reduce_finalize(r, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

template <typename M, typename Op>
__device__ __noinline__ void fused_run(Op op, const Vec& out, WinParams p) {
  __shared__ WinCtx s_c;
  __shared__ int64_t s_need;
  __shared__ alignas(16) char s_op[sizeof(Op)];
  if (threadIdx.x == 0) {
    int64_t e_star = 0, nd = 0;
    Op o = op;
    o.setup(e_star, nd);
    WinCtx cc;
    win_setup(p, out.hdr, e_star, 8 * (int)sizeof(M), cc);
    *reinterpret_cast<Op*>(s_op) = o;
    s_c = cc;
    s_need = nd;
  }
  __syncthreads();
  op = *reinterpret_cast<const Op*>(s_op);
  WinCtx c = s_c;
  const int64_t need = s_need;
  if (p.mode == MODE_NNQ) {
    fused_pass<MODE_NNQ, M>(op, out, p, c, need);
    return;
  }
  fused_pass<MODE_QCOMP, M>(op, out, p, c, need);
  // header finalized by thread 0 and published by the barrier in block_reduce_finalize
  WinParams p2 = p;
  p2.mode = MODE_RECOMPUTE;
  WinCtx c2;
  win_setup(p2, out.hdr, 0, 8 * (int)sizeof(M), c2);
  if (!c2.skip) fused_pass<MODE_RECOMPUTE, M>(op, out, p2, c2, need);
}

template <typename M>
__device__ __noinline__ void fused_zero(const Vec& v, int64_t q) {
  for (int64_t o = threadIdx.x; o < v.n; o += blockDim.x) ((M*)v.data)[o] = 0;
  if (threadIdx.x == 0) {
    Hdr* h = v.hdr;
    h->q = q;
    h->e = 0;
    h->shift = 0;
    h->max_m = 0;
    h->min_m = 0;
    h->flags = 0;
    h->need_recompute = 0;
  }
  __syncthreads();
}

template <typename M>
__global__ void __launch_bounds__(kFusedThreads) fused_kernel(const FusedOp* ops, int n) {
  griddep_wait();
  for (int i = 0; i < n; ++i) {
    const int kind = ops[i].kind;
    switch (kind) {
      case FK_GEMV: fused_run<M>(ops[i].u.gemv, ops[i].out, ops[i].p); break;
      case FK_JACOBI: fused_run<M>(ops[i].u.jac, ops[i].out, ops[i].p); break;
      case FK_SCAL: fused_run<M>(ops[i].u.scal, ops[i].out, ops[i].p); break;
      case FK_AXPBY: fused_run<M>(ops[i].u.axpby, ops[i].out, ops[i].p); break;
      case FK_RESTRICT: fused_run<M>(ops[i].u.rst, ops[i].out, ops[i].p); break;
      case FK_PROLONG: fused_run<M>(ops[i].u.pro, ops[i].out, ops[i].p); break;
      case FK_PCORR: fused_run<M>(ops[i].u.pc, ops[i].out, ops[i].p); break;
      case FK_ZERO: fused_zero<M>(ops[i].out, ops[i].q); break;
    }
    __syncthreads();
  }
}

// multi-rank finalize: apply the all-reduced partials {mu*, max, -min, err} with the
// window context recorded by pass 1 (exactly the single-rank win_finalize)
__global__ void window_finalize_kernel(Vec out, WinParams p, const int64_t* part, int storage_bits) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  griddep_wait();
  Hdr* h = out.hdr;
  if (p.mode == MODE_RECOMPUTE && !h->need_recompute) return;  // fast path: nothing ran
  WinCtx c;
  c.e_star = h->st_estar;
  c.mu_tmp = h->st_mutmp;
  c.lam = p.mode == MODE_RECOMPUTE ? h->lam_out : h->st_lam;
  c.gm = h->st_gm;
  c.ge = h->st_ge;
  c.store_tmp = p.mode == MODE_QCOMP ? (p.w_tmp <= storage_bits && !p.force) : 1;
  c.skip = 0;
  p.part = nullptr;
  win_finalize(p, c, h, (int)part[0], part[1], part[2] == INT64_MAX ? INT64_MIN : -part[2],
               (int)part[3]);
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
  reduce_and_finalize(r, out.hdr, [&](int bits, int64_t mx, int64_t mn, int err) {
    win_finalize(p, c, out.hdr, bits, mx, mn, err);
  });
}

// logical index <-> storage offset
// local logical index (interior points of the vector / slab, x fastest); for slabs the
// slowest axis starts at global plane z0
__device__ __forceinline__ int64_t logical_of(const Vec& v, int64_t o, bool& pad) {
  if (v.dim == 0) {
    pad = o >= v.nlog;
    return o;
  }
  const int64_t N = (int64_t)1 << v.l, m = N - 1, n = N - 1;
  const int64_t ix = o & m;
  if (v.dim == 1) {
    pad = ix == m;
    return ix;
  }
  if (v.dim == 2) {
    const int64_t s = o >> v.l;  // local row
    pad = ix == m || s + v.z0 == m;
    return ix + n * s;
  }
  const int64_t iy = (o >> v.l) & m, s = o >> (2 * v.l);  // local plane
  pad = ix == m || iy == m || s + v.z0 == m;
  return ix + n * (iy + n * s);
}
__device__ __forceinline__ int64_t storage_of(const Vec& v, int64_t i) {
  if (v.dim == 0) return i;
  const int64_t n = ((int64_t)1 << v.l) - 1;
  int64_t ix = i % n, t = i / n;
  int64_t iy = v.dim >= 2 ? (v.dim == 2 ? t : t % n) : 0, iz = v.dim >= 3 ? t / n : 0;
  if (v.dim == 2) return ix + (iy << v.l);
  return ix + ((iy + (iz << v.l)) << v.l);
}
// global logical index (generators: slab data equals the corresponding part of the
// full vector)
__device__ __forceinline__ int64_t global_logical(const Vec& v, int64_t local) {
  if (v.dim < 2) return local;
  const int64_t n = ((int64_t)1 << v.l) - 1;
  return local + (int64_t)v.z0 * (v.dim == 2 ? n : n * n);
}

// host logical array (staged) -> padded storage, header (q, e) with T_q / storage checks
template <typename M, typename S>
__global__ void __launch_bounds__(kThreads) scatter_kernel(Vec v, const S* src, int64_t q,
                                                           int64_t e) {
  Red r;
  r.init();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < v.n; o += stride) {
    bool pad;
    int64_t i = logical_of(v, o, pad);
    int64_t val = pad ? 0 : (int64_t)src[i];
    if (sizeof(M) == 4 && (val > INT32_MAX || val < INT32_MIN)) r.err |= ERR_STORAGE;
    ((M*)v.data)[o] = (M)val;
    r.val(val);
  }
  reduce_and_finalize(r, v.hdr, [&](int, int64_t mx, int64_t mn, int err) {
    Hdr* h = v.hdr;
    h->q = q;
    h->e = e;
    h->shift = 0;
    h->max_m = mx;
    h->min_m = mn;
    h->flags = 0;
    h->need_recompute = 0;
    int fits = q >= 64 || (msb(mx) <= q && msb(mn) <= q);
    h->err = err | (fits ? 0 : 3 /* BFP_ERR_DOMAIN */);
  });
}

// padded storage -> logical staged array, pending shift applied
template <typename M, typename D>
__global__ void __launch_bounds__(kThreads) gather_kernel(Vec v, D* dst) {
  const int64_t sh = v.hdr->shift;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < v.nlog; i += stride)
    dst[i] = (D)(((int64_t)((const M*)v.data)[storage_of(v, i)]) >> sh);
}

// zero_vec: all zero (pads included), q given, e = 0
template <typename M> __global__ void zero_kernel(Vec v, int64_t q) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < v.n; o += stride)
    ((M*)v.data)[o] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Hdr* h = v.hdr;
    h->q = q;
    h->e = 0;
    h->shift = 0;
    h->max_m = 0;
    h->min_m = 0;
    h->flags = 0;
    h->need_recompute = 0;
  }
}

// normalize (mode 0) / quantize to w (mode 1), src/bfp.cpp:97-122.  Pointwise,
// in place allowed.  Every block derives the same shift from the header.
template <typename M>
__global__ void __launch_bounds__(kThreads) renorm_kernel(Vec x, Vec out, int mode, int64_t w) {
  const Hdr* hx = x.hdr;
  const int64_t sx = hx->shift;
  const bool zero = max_abs(hx) == 0;
  const int64_t mu = zero ? 0 : eff_bits(hx);
  // shift s: value-space right shift (negative = left)
  const int64_t s = zero ? 0 : (mode == 0 ? -(hx->q - mu) : mu - w);
  Red r;
  r.init();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < x.n; o += stride) {
    int64_t v = ((int64_t)((const M*)x.data)[o]) >> sx;
    int64_t t = s >= 0 ? (s >= 63 ? (v < 0 ? -1 : 0) : (v >> s)) : (int64_t)((uint64_t)v << (-s));
    ((M*)out.data)[o] = (M)t;
    r.val(t);
  }
  // all blocks must have read hx before the finalizer rewrites it (in place):
  // the finalizer runs after every block's atomics, i.e. after their reads.
  reduce_and_finalize(r, out.hdr, [&](int, int64_t mx, int64_t mn, int err) {
    Hdr* h = out.hdr;
    int64_t e_new = zero ? 0 : hx->e + s;  // hx may alias h: read before writing
    int64_t q_new = mode == 0 ? hx->q : w;
    h->q = q_new;
    h->e = e_new;
    h->shift = 0;
    h->max_m = mx;
    h->min_m = mn;
    h->flags = 0;
    h->need_recompute = 0;
    h->err |= err;
  });
}

// uniform generator: m uniform in T_p at e = -(p-1)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
template <typename M>
__global__ void __launch_bounds__(kThreads) uniform_kernel(Vec v, int64_t p, uint64_t key) {
  Red r;
  r.init();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < v.n; o += stride) {
    bool pad;
    int64_t i = global_logical(v, logical_of(v, o, pad));
    int64_t m = 0;
    if (!pad) m = (int64_t)(splitmix64(key + (uint64_t)i) >> (64 - p)) - ((int64_t)1 << (p - 1));
    ((M*)v.data)[o] = (M)m;
    r.val(m);
  }
  reduce_and_finalize(r, v.hdr, [&](int, int64_t mx, int64_t mn, int) {
    Hdr* h = v.hdr;
    h->q = p;
    h->e = -(p - 1);
    h->shift = 0;
    h->max_m = mx;
    h->min_m = mn;
    h->flags = 0;
    h->need_recompute = 0;
  });
}

// sine rhs: v = ((C s_x) s_y) s_z in IEEE double (no contraction), then
// quantize_exact at p bits (src/bfp.cpp:163-187).  Pass 1 finds the top
// binade (bits field of Red), pass 2 writes mantissas.
__device__ __forceinline__ double sine_val(const Vec& v, const double* tab, double C, int64_t o,
                                           bool& pad) {
  int64_t i = logical_of(v, o, pad);
  (void)i;
  if (pad) return 0.0;
  const int64_t N = (int64_t)1 << v.l, m = N - 1;
  double r = __dmul_rn(C, tab[o & m]);
  if (v.dim == 2) r = __dmul_rn(r, tab[(o >> v.l) + v.z0]);
  if (v.dim == 3) {
    r = __dmul_rn(r, tab[(o >> v.l) & m]);
    r = __dmul_rn(r, tab[(o >> (2 * v.l)) + v.z0]);
  }
  return r;
}
__device__ __forceinline__ void split_double(double v, int64_t& z, int64_t& k) {
  int ex;
  double fr = frexp(v, &ex);
  z = (int64_t)ldexp(fr, 53);
  k = (int64_t)ex - 53;
}
__global__ void set_i64_kernel(int64_t* p, int64_t v) { *p = v; }

template <typename M>
__global__ void __launch_bounds__(kThreads) sine_top_kernel(Vec v, const double* tab, double C,
                                                            int64_t* top) {
  int64_t t = INT64_MIN;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < v.n; o += stride) {
    bool pad;
    double d = sine_val(v, tab, C, o, pad);
    if (pad || d == 0.0) continue;
    int64_t z, k;
    split_double(d, z, k);
    int64_t b = msb(z) + k;
    t = b > t ? b : t;
  }
  t = shfl_max64(t);
  if ((threadIdx.x & 31) == 0 && t != INT64_MIN) atomicMax((long long*)top, (long long)t);
}
template <typename M>
__global__ void __launch_bounds__(kThreads) sine_write_kernel(Vec v, const double* tab, double C,
                                                              const int64_t* top, int64_t p) {
  const int64_t tp = *top;
  const bool any = tp != INT64_MIN;
  const int64_t e_out = any ? tp - p : 0;
  Red r;
  r.init();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < v.n; o += stride) {
    bool pad;
    double d = sine_val(v, tab, C, o, pad);
    int64_t m = 0;
    if (!pad && d != 0.0) {
      int64_t z, k;
      split_double(d, z, k);
      int64_t s = e_out - k;
      m = s >= 0 ? (s >= 63 ? (z < 0 ? -1 : 0) : (z >> s)) : (int64_t)((uint64_t)z << (-s));
    }
    ((M*)v.data)[o] = (M)m;
    r.val(m);
  }
  reduce_and_finalize(r, v.hdr, [&](int, int64_t mx, int64_t mn, int) {
    Hdr* h = v.hdr;
    h->q = p;
    h->e = e_out;
    h->shift = 0;
    h->max_m = mx;
    h->min_m = mn;
    h->flags = 0;
    h->need_recompute = 0;
  });
}

// exact dot: per-block int128 partials, then one block sums them
template <typename M>
__global__ void __launch_bounds__(kThreads) dot_partial_kernel(Vec x, Vec y, i128* part) {
  const int64_t sx = x.hdr->shift, sy = y.hdr->shift;
  i128 acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < x.n; o += stride)
    acc += (i128)(((int64_t)((const M*)x.data)[o]) >> sx) *
           (i128)(((int64_t)((const M*)y.data)[o]) >> sy);
  // warp reduce (two 64-bit halves with carry via 128-bit adds)
  for (int off = 16; off > 0; off >>= 1) {
    uint64_t lo = __shfl_xor_sync(0xffffffffu, (uint64_t)acc, off);
    int64_t hi = __shfl_xor_sync(0xffffffffu, (int64_t)(acc >> 64), off);
    acc += (i128)(((u128)(uint64_t)hi << 64) | lo);
  }
  __shared__ i128 s[kThreads / 32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    part[blockIdx.x] = t;
  }
}
__global__ void dot_final_kernel(const i128* part, int n, i128* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    i128 t = 0;
    for (int i = 0; i < n; ++i) t += part[i];
    *out = t;
  }
}

// ===========================================================================
// host side

namespace bfp {

void count_launch(int n) { g_launches += n; }
int64_t launches() { return g_launches.load(); }

Vec view(const bfp_vec_s* v) {
  Vec d;
  d.data = v->data;
  d.hdr = v->hdr;
  d.ebytes = v->ebytes;
  d.dim = v->dim;
  d.l = v->l;
  d.z0 = v->z0;
  d.n = v->span;
  d.nlog = v->nlog;
  d.nz = v->nz;
  d.pad = 0;
  return d;
}

int vec_alloc(int dim, int level, int64_t n, int ebytes, bfp_vec_s** out) {
  return vec_alloc_slab(dim, level, n, 0, -1, ebytes, out);
}

// z_hi < 0: full grid.  Otherwise a slab of planes [z_lo, z_hi) of the padded global grid
// along the slowest axis (2-D rows, 3-D planes), with the usual halo planes around it.
int vec_alloc_slab(int dim, int level, int64_t n, int z_lo, int z_hi, int ebytes, bfp_vec_s** out) {
  if (ebytes != 4 && ebytes != 8) return BFP_ERR_ARG;
  if (dim < 0 || dim > 3) return BFP_ERR_ARG;
  if (z_hi >= 0 && (dim < 2 || z_lo < 0 || z_hi <= z_lo || z_hi > (1 << level)))
    return BFP_ERR_ARG;
  bfp_vec_s* v = new bfp_vec_s();
  v->dim = dim;
  v->l = level;
  v->ebytes = ebytes;
  if (dim == 0) {
    if (n < 0) {
      delete v;
      return BFP_ERR_ARG;
    }
    v->nlog = n;
    v->span = (n + 3) / 4 * 4;
    v->halo = 4;
  } else {
    if (level < 2 || level > 30 || (int64_t)dim * level > 36) {
      delete v;
      return BFP_ERR_ARG;
    }
    const int64_t N = (int64_t)1 << level, nn = N - 1;
    v->z0 = z_hi >= 0 ? z_lo : 0;
    v->nz = z_hi >= 0 ? z_hi - z_lo : (int)N;
    const int64_t interior = std::min<int64_t>(v->z0 + v->nz, nn) - v->z0;  // planes < N-1
    v->nlog = interior;
    v->span = v->nz;
    for (int a = 1; a < dim; ++a) {
      v->nlog *= nn;
      v->span *= N;
    }
    v->halo = dim == 1 ? 4 : 2 * (v->span / v->nz);
  }
  size_t bytes = (size_t)(v->span + 2 * v->halo) * ebytes;
  if (cudaMalloc(&v->base, bytes) != cudaSuccess) {
    delete v;
    cudaGetLastError();
    return BFP_ERR_NOMEM;
  }
  cudaMemset(v->base, 0, bytes);
  v->data = v->base + (size_t)v->halo * ebytes;
  if (cudaMalloc(&v->hdr, sizeof(Hdr)) != cudaSuccess) {
    cudaFree(v->base);
    delete v;
    cudaGetLastError();
    return BFP_ERR_NOMEM;
  }
  Hdr h;
  memset(&h, 0, sizeof(h));
  h.q = 1;
  h.acc_max = INT64_MIN;
  h.acc_min = INT64_MAX;
  h.acc_or_lo = h.acc_or_hi = 0;
  cudaMemcpy(v->hdr, &h, sizeof(h), cudaMemcpyHostToDevice);
  *out = v;
  return BFP_OK;
}

void vec_free(bfp_vec_s* v) {
  if (!v) return;
  cudaFree(v->base);
  cudaFree(v->hdr);
  if (v->stage) cudaFree(v->stage);
  if (v->tab) cudaFree(v->tab);
  delete v;
}

static int ensure_stage(bfp_vec_s* v, size_t bytes) {
  if (v->stage_bytes >= bytes) return BFP_OK;
  if (v->stage) cudaFree(v->stage);
  v->stage = nullptr;
  v->stage_bytes = 0;
  if (cudaMalloc(&v->stage, std::max<size_t>(bytes, 16)) != cudaSuccess) {
    cudaGetLastError();
    return BFP_ERR_NOMEM;
  }
  v->stage_bytes = bytes;
  return BFP_OK;
}

int set_zero(bfp_vec_s* v, int64_t q, cudaStream_t s) {
  Vec d = view(v);
  int b = blocks_for(v->span);
  if (v->ebytes == 4)
    zero_kernel<int32_t><<<b, kThreads, 0, s>>>(d, q);
  else
    zero_kernel<int64_t><<<b, kThreads, 0, s>>>(d, q);
  count_launch();
  return last_launch();
}

WinParams win_params(int mode, int64_t w_out, int64_t w_tmp, int force) {
  WinParams p;
  memset(&p, 0, sizeof(p));
  p.w_out = w_out;
  p.w_tmp = mode == MODE_QCOMP ? w_tmp : w_out;
  p.mode = mode;
  p.force = force;
  p.trace_slot = -1;
  p.trace = nullptr;
  p.hist_slot = -1;
  p.hist = nullptr;
  p.part = nullptr;
  return p;
}
GammaRule gamma_literal(int64_t m, int64_t e) {
  GammaRule g;
  memset(&g, 0, sizeof(g));
  g.literal = 1;
  g.lm = m;
  g.le = e;
  return g;
}

static int check_window(const WinParams& p, const bfp_vec_s* out) {
  const int sb = out->ebytes * 8;
  if (p.w_out < 1 || p.w_out > sb) return BFP_ERR_ARG;
  if (p.mode == MODE_QCOMP && (p.w_tmp < p.w_out || p.w_tmp > 64)) return BFP_ERR_ARG;
  if (p.gamma.literal && p.gamma.lm <= 0) return BFP_ERR_ARG;
  return BFP_OK;
}

// launch a grid-windowed op: nnqcomp (one pass) or qcomp (pass 1 + recompute)
template <typename Op>
static int launch_grid(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  const int b = blocks_for(out->span / 4);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    const int nb = pp.mode == MODE_RECOMPUTE ? std::min(b, 2 * 148) : b;
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
  };
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p);
    cudaEventRecord(ev.second, s);
  } else {
    go(p);
  }
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}

// stencil ops on int32 grids of 2-D / 3-D with N >= 128 use the register march
template <typename Op>
static int launch_bulk(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  const int64_t N = int64_t(1) << out->l;
  static int occ = 0;
  if (!occ) {
    for (auto fn : {bulk_win_kernel<MODE_QCOMP, Op>, bulk_win_kernel<MODE_NNQ, Op>,
                    bulk_win_kernel<MODE_RECOMPUTE, Op>})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBulkSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bulk_win_kernel<MODE_QCOMP, Op>, kBulkT,
                                                  kBulkSmem);
    occ = std::max(occ, 1);
  }
  const int64_t strips = N / kBulkW, ctas = (int64_t)148 * occ;
  const int64_t NZ = out->nz;
  const int R = (int)std::max<int64_t>(8, (strips * NZ + ctas - 1) / ctas);
  const int64_t items = strips * ((NZ + R - 1) / R);
  const int b = (int)std::min<int64_t>(items, ctas);
  WinParams p = p0;
  auto go = [&](const WinParams& pp) {
    if (pp.mode == MODE_QCOMP)
      launch_pdl(bulk_win_kernel<MODE_QCOMP, Op>, b, kBulkT, kBulkSmem, s, op, o, pp, R);
    else if (pp.mode == MODE_NNQ)
      launch_pdl(bulk_win_kernel<MODE_NNQ, Op>, b, kBulkT, kBulkSmem, s, op, o, pp, R);
    else
      launch_pdl(bulk_win_kernel<MODE_RECOMPUTE, Op>, b, kBulkT, kBulkSmem, s, op, o, pp, R);
    count_launch();
  };
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p);
    cudaEventRecord(ev.second, s);
  } else {
    go(p);
  }
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}

static bool g_use_bulk = true;

template <typename Op>
static int launch_march(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
  if (out->ebytes != 4 || out->dim < 2 || (int64_t(1) << out->l) < kMarchMinN)
    return launch_grid(op, out, p0, s);
  if (g_use_bulk && out->dim == 2 && (int64_t(1) << out->l) >= kBulkW)
    return launch_bulk(op, out, p0, s);
  int rc = check_window(p0, out);
  if (rc) return rc;
  Vec o = view(out);
  const int64_t N = int64_t(1) << out->l, GX = N / 4, rows = out->dim == 3 ? N : 1;
  static int occ2 = 0, occ3 = 0;
  if (!occ2) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, march_win_kernel<MODE_QCOMP, 2, Op>,
                                                  kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, march_win_kernel<MODE_QCOMP, 3, Op>,
                                                  kThreads, 0);
    occ2 = std::max(occ2, 1);
    occ3 = std::max(occ3, 1);
  }
  const int occ = out->dim == 2 ? occ2 : occ3;
  // one balanced resident wave: every thread marches R steps (last chunk shorter)
  const int64_t slots = (int64_t)148 * occ * kThreads;
  const int64_t NZ = out->nz;
  int R = (int)std::max<int64_t>(4, (GX * rows * NZ + slots - 1) / slots);
  const int64_t items = GX * rows * ((NZ + R - 1) / R);
  const int b = (int)std::max<int64_t>(1, std::min<int64_t>((items + kThreads - 1) / kThreads,
                                                            (int64_t)148 * occ));
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
  };
  if (g_prof) {
    auto ev = prof_pair();
    cudaEventRecord(ev.first, s);
    go(p, b);
    cudaEventRecord(ev.second, s);
  } else {
    go(p, b);
  }
  if (p.mode == MODE_QCOMP && !g_skip_recompute && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p, b);
  }
  return last_launch();
}

template <typename Op>
static int launch_flat(const Op& op, bfp_vec_s* out, const WinParams& p0, cudaStream_t s) {
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
  };
  go(p);
  if (p.mode == MODE_QCOMP && !p.part) {
    p.mode = MODE_RECOMPUTE;
    go(p);
  }
  return last_launch();
}

static bool same_grid(const bfp_vec_s* a, const bfp_vec_s* b) {
  return a->dim == b->dim && a->l == b->l && a->ebytes == b->ebytes && a->span == b->span &&
         a->nlog == b->nlog && a->z0 == b->z0 && a->nz == b->nz;
}
static bool full_grid(const bfp_vec_s* a) { return a->dim == 0 || a->nz == (1 << a->l); }

int op_gemv(bfp_vec_s* x, bfp_vec_s* y, Scal al, Scal be, const WinParams& p, bfp_vec_s* out,
            cudaStream_t s) {
  if (x->dim < 1 || !same_grid(x, y) || !same_grid(x, out)) return BFP_ERR_ARG;
  if (out == x || out == y) return BFP_ERR_ALIAS;
  GemvOp op;
  op.x = view(x);
  op.y = view(y);
  op.al = al;
  op.be = be;
  op.dim = x->dim;
  op.l = x->l;
  op.z0 = x->z0;
  return launch_march(op, out, p, s);
}

int op_jacobi(bfp_vec_s* x, bfp_vec_s* b, Scal c, const WinParams& p, bfp_vec_s* out,
              cudaStream_t s) {
  if (x->dim < 1 || !same_grid(x, b) || !same_grid(x, out)) return BFP_ERR_ARG;
  if (out == x || out == b) return BFP_ERR_ALIAS;
  JacobiOp op;
  op.x = view(x);
  op.b = view(b);
  op.c = c;
  op.dim = x->dim;
  op.l = x->l;
  op.z0 = x->z0;
  return launch_march(op, out, p, s);
}

int op_scal(bfp_vec_s* r, Scal c, const WinParams& p, bfp_vec_s* out, cudaStream_t s) {
  if (!same_grid(r, out)) return BFP_ERR_ARG;
  if (out == r) return BFP_ERR_ALIAS;
  ScalOp op;
  op.r = view(r);
  op.c = c;
  return launch_grid(op, out, p, s);
}

int op_axpby(bfp_vec_s* x, bfp_vec_s* y, Scal al, Scal be, const WinParams& p, bfp_vec_s* out,
             cudaStream_t s) {
  if (!same_grid(x, y) || !same_grid(x, out)) return BFP_ERR_ARG;
  if (out == x || out == y) return BFP_ERR_ALIAS;
  AxpbyOp op;
  op.x = view(x);
  op.y = view(y);
  op.al = al;
  op.be = be;
  return launch_grid(op, out, p, s);
}

int op_restrict(bfp_vec_s* r, const WinParams& p, bfp_vec_s* out, cudaStream_t s) {
  if (!full_grid(r) || !full_grid(out)) return BFP_ERR_ARG;  // transfers: full grids only
  if (r->dim < 1 || out->dim != r->dim || out->l != r->l - 1 || out->ebytes != r->ebytes)
    return BFP_ERR_ARG;
  RestrictOp op;
  op.r = view(r);
  op.dim = r->dim;
  op.l = r->l;
  return launch_grid(op, out, p, s);
}

int op_prolong(bfp_vec_s* xc, const WinParams& p, bfp_vec_s* out, cudaStream_t s) {
  if (!full_grid(xc) || !full_grid(out)) return BFP_ERR_ARG;
  if (xc->dim < 1 || out->dim != xc->dim || out->l != xc->l + 1 || out->ebytes != xc->ebytes)
    return BFP_ERR_ARG;
  ProlongOp op;
  op.xc = view(xc);
  op.dim = out->dim;
  op.l = out->l;
  return launch_grid(op, out, p, s);
}

int op_prolong_correct(bfp_vec_s* ec, bfp_vec_s* y, const WinParams& p, bfp_vec_s* out,
                       cudaStream_t s) {
  if (!full_grid(ec) || !full_grid(y)) return BFP_ERR_ARG;
  if (ec->dim < 1 || !same_grid(y, out) || y->dim != ec->dim || y->l != ec->l + 1 ||
      y->ebytes != ec->ebytes)
    return BFP_ERR_ARG;
  if (out == y) return BFP_ERR_ALIAS;
  ProlongCorrectOp op;
  op.ec = view(ec);
  op.y = view(y);
  op.dim = y->dim;
  op.l = y->l;
  return launch_grid(op, out, p, s);
}

int gen_uniform(bfp_vec_s* v, int64_t p, uint64_t seed, uint64_t stream_id, cudaStream_t s) {
  if (p < 2 || p > std::min(62, v->ebytes * 8)) return BFP_ERR_ARG;
  auto sm = [](uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  uint64_t key = sm(sm(seed) ^ stream_id);
  Vec d = view(v);
  int b = blocks_for(v->span);
  if (v->ebytes == 4) {
    uniform_kernel<int32_t><<<b, kThreads, 0, s>>>(d, p, key);
    renorm_kernel<int32_t><<<b, kThreads, 0, s>>>(d, d, 0, 0);
  } else {
    uniform_kernel<int64_t><<<b, kThreads, 0, s>>>(d, p, key);
    renorm_kernel<int64_t><<<b, kThreads, 0, s>>>(d, d, 0, 0);
  }
  count_launch(2);
  return last_launch();
}

int gen_sine(bfp_vec_s* v, int64_t p, cudaStream_t s) {
  if (v->dim < 1 || p < 2 || p > std::min(62, v->ebytes * 8)) return BFP_ERR_ARG;
  const int64_t N = (int64_t)1 << v->l, n = N - 1;
  if (!v->tab) {
    std::vector<double> t((size_t)N + 1, 0.0);
    const double h = std::ldexp(1.0, -v->l);
    for (int64_t i = 0; i < n; ++i) t[(size_t)i] = std::sin(M_PI * ((double)(i + 1) * h));
    if (cudaMalloc(&v->tab, sizeof(double) * (N + 1)) != cudaSuccess) {
      cudaGetLastError();
      return BFP_ERR_NOMEM;
    }
    cudaMemcpy(v->tab, t.data(), sizeof(double) * (N + 1), cudaMemcpyHostToDevice);
    // slot N holds the top-binade scratch (int64)
  }
  const double C = (double)v->dim * (M_PI * M_PI);
  int64_t* top = reinterpret_cast<int64_t*>(v->tab + N);
  set_i64_kernel<<<1, 1, 0, s>>>(top, INT64_MIN);
  count_launch();
  Vec d = view(v);
  int b = blocks_for(v->span);
  if (v->ebytes == 4) {
    sine_top_kernel<int32_t><<<b, kThreads, 0, s>>>(d, v->tab, C, top);
    sine_write_kernel<int32_t><<<b, kThreads, 0, s>>>(d, v->tab, C, top, p);
  } else {
    sine_top_kernel<int64_t><<<b, kThreads, 0, s>>>(d, v->tab, C, top);
    sine_write_kernel<int64_t><<<b, kThreads, 0, s>>>(d, v->tab, C, top, p);
  }
  count_launch(2);
  return last_launch();
}

void jacobi_coeff(int dim, int level, int64_t qc, int64_t* cm, int64_t* ce) {
  // omega_d/(2d) = 1/3, 1/5, 1/7 floor-quantised at qc bits
  const int64_t den = dim == 1 ? 3 : (dim == 2 ? 5 : 7);
  int64_t fl = 0;
  while ((((int64_t)1) << (-fl)) < den) --fl;
  const int64_t top = fl + 2;
  *cm = (int64_t)((((__int128)1) << (qc - top)) / den);
  *ce = top - qc - 2 * (int64_t)level;
}

}  // namespace bfp


namespace bfp {

int fused_make(int kind, bfp_vec_s* a, bfp_vec_s* b, Scal s1, Scal s2, const WinParams& p,
               int64_t q, bfp_vec_s* out, FusedOp* f) {
  memset(f, 0, sizeof(*f));
  f->kind = kind;
  f->out = view(out);
  f->p = p;
  f->q = q;
  switch (kind) {
    case FK_GEMV:
      f->u.gemv.x = view(a); f->u.gemv.y = view(b); f->u.gemv.al = s1; f->u.gemv.be = s2;
      f->u.gemv.dim = a->dim; f->u.gemv.l = a->l; f->u.gemv.z0 = a->z0;
      break;
    case FK_JACOBI:
      f->u.jac.x = view(a); f->u.jac.b = view(b); f->u.jac.c = s1;
      f->u.jac.dim = a->dim; f->u.jac.l = a->l; f->u.jac.z0 = a->z0;
      break;
    case FK_SCAL: f->u.scal.r = view(a); f->u.scal.c = s1; break;
    case FK_AXPBY:
      f->u.axpby.x = view(a); f->u.axpby.y = view(b); f->u.axpby.al = s1; f->u.axpby.be = s2;
      break;
    case FK_RESTRICT: f->u.rst.r = view(a); f->u.rst.dim = a->dim; f->u.rst.l = a->l; break;
    case FK_PROLONG: f->u.pro.xc = view(a); f->u.pro.dim = out->dim; f->u.pro.l = out->l; break;
    case FK_PCORR:
      f->u.pc.ec = view(a); f->u.pc.y = view(b); f->u.pc.dim = out->dim; f->u.pc.l = out->l;
      break;
    case FK_ZERO: break;
    default: return BFP_ERR_ARG;
  }
  return BFP_OK;
}

int fused_launch(const FusedOp* d_ops, int n, int ebytes, cudaStream_t s) {
  if (ebytes == 4)
    launch_pdl(fused_kernel<int32_t>, 1, kFusedThreads, 0, s, d_ops, n);
  else
    launch_pdl(fused_kernel<int64_t>, 1, kFusedThreads, 0, s, d_ops, n);
  count_launch();
  return last_launch();
}

}  // namespace bfp

// ===========================================================================
// C-ABI

using namespace bfp;

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static Scal SC(bfp_scalar_t s) { return Scal{s.m, s.q, s.e}; }

extern "C" {

const char* bfp_status_string(int st) {
  switch (st) {
    case BFP_OK: return "ok";
    case BFP_ERR_ARG: return "invalid argument";
    case BFP_ERR_WIDTH: return "exact row exceeds 127 bits";
    case BFP_ERR_DOMAIN: return "mantissa does not fit T_q";
    case BFP_ERR_CUDA: return "CUDA error";
    case BFP_ERR_ALIAS: return "output aliases an input";
    case BFP_ERR_NOMEM: return "out of device memory";
    case BFP_ERR_STORAGE: return "value does not fit the mantissa storage";
  }
  return "unknown";
}

int64_t bfp_launch_count(void) { return launches(); }

int bfp_profile_enable(int on) {
  g_prof = on != 0;
  return BFP_OK;
}
int bfp_set_kernel_path(int bulk) {
  g_use_bulk = (bulk & 1) != 0;
  g_pdl = (bulk & 2) == 0;             // bit 1 disables programmatic dependent launch
  g_skip_recompute = (bulk & 4) != 0;  // bit 2: measurement of pass 1 alone
  return BFP_OK;
}
int bfp_profile_read(double* total_ms, int64_t* count, int reset) {
  double t = 0;
  for (size_t i = 0; i < g_ev_used; ++i) {
    if (cudaEventSynchronize(g_ev[i].second) != cudaSuccess) return BFP_ERR_CUDA;
    float ms = 0;
    cudaEventElapsedTime(&ms, g_ev[i].first, g_ev[i].second);
    t += ms;
  }
  if (total_ms) *total_ms = t;
  if (count) *count = (int64_t)g_ev_used;
  if (reset) g_ev_used = 0;
  return BFP_OK;
}

int bfp_device_sync(void* stream) { return cuda_status(cudaStreamSynchronize(S(stream))); }

int bfp_vec_create(int64_t n, int mant_bytes, bfp_vec_t* out) {
  return vec_alloc(0, 0, n, mant_bytes, out);
}
int bfp_vec_create_grid(int dim, int level, int mant_bytes, bfp_vec_t* out) {
  if (dim < 1) return BFP_ERR_ARG;
  return vec_alloc(dim, level, 0, mant_bytes, out);
}
int bfp_vec_destroy(bfp_vec_t v) {
  vec_free(v);
  return BFP_OK;
}
int64_t bfp_vec_size(bfp_vec_t v) { return v ? v->nlog : -1; }

}  // extern "C"
template <typename S_>
static int upload_impl(bfp_vec_t v, const S_* m, int64_t q, int64_t e, void* stream) {
  if (!v || q < 1 || (q > 64)) return BFP_ERR_ARG;
  int rc = ensure_stage(v, sizeof(S_) * (size_t)std::max<int64_t>(v->nlog, 1));
  if (rc) return rc;
  if (v->nlog)
    if (cudaMemcpyAsync(v->stage, m, sizeof(S_) * v->nlog, cudaMemcpyHostToDevice, S(stream)) !=
        cudaSuccess)
      return BFP_ERR_CUDA;
  Vec d = view(v);
  int b = blocks_for(v->span);
  if (v->ebytes == 4)
    scatter_kernel<int32_t, S_><<<b, kThreads, 0, S(stream)>>>(d, (const S_*)v->stage, q, e);
  else
    scatter_kernel<int64_t, S_><<<b, kThreads, 0, S(stream)>>>(d, (const S_*)v->stage, q, e);
  count_launch();
  return last_launch();
}
extern "C" {
int bfp_vec_upload(bfp_vec_t v, const int64_t* m, int64_t q, int64_t e, void* stream) {
  return upload_impl<int64_t>(v, m, q, e, stream);
}
int bfp_vec_upload_i32(bfp_vec_t v, const int32_t* m, int64_t q, int64_t e, void* stream) {
  return upload_impl<int32_t>(v, m, q, e, stream);
}

int bfp_vec_header(bfp_vec_t v, bfp_header_t* hdr, void* stream) {
  if (!v || !hdr) return BFP_ERR_ARG;
  Hdr h;
  if (cudaMemcpyAsync(&h, v->hdr, sizeof(h), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess)
    return BFP_ERR_CUDA;
  if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return BFP_ERR_CUDA;
  int64_t a = h.max_m >> h.shift, b = h.min_m >> h.shift;
  uint64_t ua = a < 0 ? (uint64_t)0 - (uint64_t)a : (uint64_t)a;
  uint64_t ub = b < 0 ? (uint64_t)0 - (uint64_t)b : (uint64_t)b;
  hdr->q = h.q;
  hdr->e = h.e;
  hdr->n = v->nlog;
  hdr->max_abs = (int64_t)(ua > ub ? ua : ub);
  hdr->flags = h.flags;
  hdr->err = h.err;
  return h.err ? h.err : BFP_OK;
}

}  // extern "C"
template <typename D_>
static int download_impl(bfp_vec_t v, D_* m, bfp_header_t* hdr, void* stream) {
  if (!v) return BFP_ERR_ARG;
  int rc = ensure_stage(v, sizeof(D_) * (size_t)std::max<int64_t>(v->nlog, 1));
  if (rc) return rc;
  Vec d = view(v);
  int b = blocks_for(v->nlog);
  if (v->ebytes == 4)
    gather_kernel<int32_t, D_><<<b, kThreads, 0, S(stream)>>>(d, (D_*)v->stage);
  else
    gather_kernel<int64_t, D_><<<b, kThreads, 0, S(stream)>>>(d, (D_*)v->stage);
  count_launch();
  if ((rc = last_launch())) return rc;
  if (v->nlog && m)
    if (cudaMemcpyAsync(m, v->stage, sizeof(D_) * v->nlog, cudaMemcpyDeviceToHost, S(stream)) !=
        cudaSuccess)
      return BFP_ERR_CUDA;
  bfp_header_t tmp;
  return bfp_vec_header(v, hdr ? hdr : &tmp, stream);
}
extern "C" {
int bfp_vec_download(bfp_vec_t v, int64_t* m, bfp_header_t* hdr, void* stream) {
  return download_impl<int64_t>(v, m, hdr, stream);
}
int bfp_vec_download_async_i32(bfp_vec_t v, int32_t* m, void* stream) {
  if (!v || v->ebytes != 4) return BFP_ERR_ARG;
  int rc = ensure_stage(v, sizeof(int32_t) * (size_t)std::max<int64_t>(v->nlog, 1));
  if (rc) return rc;
  Vec d = view(v);
  gather_kernel<int32_t, int32_t><<<blocks_for(v->nlog), kThreads, 0, S(stream)>>>(d, (int32_t*)v->stage);
  count_launch();
  if ((rc = last_launch())) return rc;
  if (v->nlog && m &&
      cudaMemcpyAsync(m, v->stage, sizeof(int32_t) * v->nlog, cudaMemcpyDeviceToHost, S(stream)) !=
          cudaSuccess)
    return BFP_ERR_CUDA;
  return BFP_OK;
}
int bfp_vec_download_i32(bfp_vec_t v, int32_t* m, bfp_header_t* hdr, void* stream) {
  if (v && v->ebytes != 4) return BFP_ERR_ARG;
  return download_impl<int32_t>(v, m, hdr, stream);
}

int bfp_vec_zero(bfp_vec_t v, int64_t q, void* stream) {
  if (!v || q < 1 || q > v->ebytes * 8) return BFP_ERR_ARG;
  return set_zero(v, q, S(stream));
}

int64_t bfp_vec_dump(bfp_vec_t v, char* buf, int64_t cap, void* stream) {
  if (!v) return -1;
  std::vector<int64_t> m((size_t)v->nlog);
  bfp_header_t h;
  int rc = bfp_vec_download(v, m.data(), &h, stream);
  if (rc) return -rc;
  std::ostringstream os;
  os << h.q << ' ' << h.e << ' ' << v->nlog << '\n';  // Layout::vector (src/bfp.cpp:230-241)
  for (int64_t x : m) os << x << '\n';
  std::string s = os.str();
  if (buf && cap > 0) {
    size_t k = std::min<size_t>((size_t)cap - 1, s.size());
    memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return (int64_t)s.size() + 1;
}

int bfp_vec_parse(const char* text, bfp_vec_t* out, void* stream) {
  if (!text || !out) return BFP_ERR_ARG;
  std::istringstream is(text);
  int64_t q, e;
  std::string d;
  if (!(is >> q >> e >> d)) return BFP_ERR_ARG;
  int64_t rows = 1, cols = 1;
  if (d != "scalar") {
    auto xp = d.find('x');
    try {
      if (xp == std::string::npos) {
        rows = std::stoll(d);
      } else {
        rows = std::stoll(d.substr(0, xp));
        cols = std::stoll(d.substr(xp + 1));
      }
    } catch (...) {
      return BFP_ERR_ARG;
    }
  }
  std::vector<int64_t> m;
  std::string tok;
  while (is >> tok) {
    try {
      size_t pos = 0;
      long long v = std::stoll(tok, &pos);
      if (pos != tok.size()) return BFP_ERR_ARG;
      m.push_back(v);
    } catch (...) {
      return BFP_ERR_DOMAIN;  // beyond int64 storage
    }
  }
  if ((int64_t)m.size() != rows * cols) return BFP_ERR_ARG;
  bfp_vec_t v;
  int rc = bfp_vec_create((int64_t)m.size(), 8, &v);
  if (rc) return rc;
  rc = bfp_vec_upload(v, m.data(), q, e, stream);
  if (!rc) {
    bfp_header_t h;
    rc = bfp_vec_header(v, &h, stream);
  }
  if (rc) {
    bfp_vec_destroy(v);
    return rc;
  }
  *out = v;
  return BFP_OK;
}

static int renorm(bfp_vec_t x, bfp_vec_t out, int mode, int64_t w, void* stream) {
  if (!x || !out || x->span != out->span || x->dim != out->dim || x->l != out->l ||
      x->ebytes != out->ebytes)
    return BFP_ERR_ARG;
  if (mode == 1 && (w < 1 || w > out->ebytes * 8)) return BFP_ERR_ARG;
  Vec a = view(x), b = view(out);
  int nb = blocks_for(x->span);
  if (x->ebytes == 4)
    renorm_kernel<int32_t><<<nb, kThreads, 0, S(stream)>>>(a, b, mode, w);
  else
    renorm_kernel<int64_t><<<nb, kThreads, 0, S(stream)>>>(a, b, mode, w);
  count_launch();
  return last_launch();
}
int bfp_normalize(bfp_vec_t x, bfp_vec_t out, void* stream) { return renorm(x, out, 0, 0, stream); }
int bfp_quantize(bfp_vec_t x, int64_t w, bfp_vec_t out, void* stream) {
  return renorm(x, out, 1, w, stream);
}

int bfp_inf_norm_upper(bfp_vec_t x, int64_t q_gamma, int64_t* m, int64_t* q, int64_t* e,
                       void* stream) {
  // src/bfp.cpp:124-148 on the device header's exact max |m|
  if (q_gamma < 2 || q_gamma > 62) return BFP_ERR_ARG;
  bfp_header_t h;
  int rc = bfp_vec_header(x, &h, stream);
  if (rc) return rc;
  uint64_t mx = (uint64_t)h.max_abs;
  *q = q_gamma;
  if (mx == 0) {
    *m = (int64_t)1 << (q_gamma - 2);
    *e = h.e - (q_gamma - 2);
    return BFP_OK;
  }
  int64_t s = (int64_t)msb_h((int64_t)mx) - q_gamma;
  if (mx >> 63) s = 65 - q_gamma;  // |INT64_MIN|
  uint64_t mm;
  if (s <= 0) {
    mm = mx << (-s);
  } else {
    mm = (mx >> s) + ((mx & ((1ull << s) - 1)) != 0);
    if (msb_h((int64_t)mm) > q_gamma) {
      mm >>= 1;
      ++s;
    }
  }
  *m = (int64_t)mm;
  *e = h.e + s;
  return BFP_OK;
}

int bfp_dot_exact(bfp_vec_t x, bfp_vec_t y, int64_t* hi, uint64_t* lo, int64_t* e, void* stream) {
  if (!x || !y || x->span != y->span || x->ebytes != y->ebytes || x->dim != y->dim) return BFP_ERR_ARG;
  const int nb = blocks_for(x->span);
  i128* part = nullptr;
  if (cudaMalloc(&part, sizeof(i128) * (nb + 1)) != cudaSuccess) return BFP_ERR_NOMEM;
  Vec a = view(x), b = view(y);
  if (x->ebytes == 4)
    dot_partial_kernel<int32_t><<<nb, kThreads, 0, S(stream)>>>(a, b, part);
  else
    dot_partial_kernel<int64_t><<<nb, kThreads, 0, S(stream)>>>(a, b, part);
  dot_final_kernel<<<1, 32, 0, S(stream)>>>(part, nb, part + nb);
  count_launch(2);
  i128 r = 0;
  cudaMemcpyAsync(&r, part + nb, sizeof(r), cudaMemcpyDeviceToHost, S(stream));
  Hdr hx, hy;
  cudaMemcpyAsync(&hx, x->hdr, sizeof(Hdr), cudaMemcpyDeviceToHost, S(stream));
  cudaMemcpyAsync(&hy, y->hdr, sizeof(Hdr), cudaMemcpyDeviceToHost, S(stream));
  cudaError_t err = cudaStreamSynchronize(S(stream));
  cudaFree(part);
  if (err != cudaSuccess) return BFP_ERR_CUDA;
  *hi = (int64_t)(r >> 64);
  *lo = (uint64_t)r;
  *e = hx.e + hy.e;
  return BFP_OK;
}

static WinParams mkp(int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t g, int force) {
  WinParams p = win_params(mode == 1 ? MODE_NNQ : MODE_QCOMP, w_out, w_tmp, force);
  p.gamma = gamma_literal(g.m, g.e);
  return p;
}

int bfp_axpby(bfp_vec_t x, bfp_vec_t y, bfp_scalar_t alpha, bfp_scalar_t beta, int mode,
              int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma, int force, bfp_vec_t out,
              void* stream) {
  if (!x || !y || !out || gamma.m <= 0) return BFP_ERR_ARG;
  return op_axpby(x, y, SC(alpha), SC(beta), mkp(mode, w_out, w_tmp, gamma, force), out,
                  S(stream));
}

int bfp_csr_create(int64_t rows, int64_t cols, const int64_t* rowptr, const int64_t* col,
                   const int64_t* m, int64_t q, int64_t e, bfp_csr_t* out) {
  if (rows < 0 || cols < 0 || !rowptr) return BFP_ERR_ARG;
  const int64_t nnz = rowptr[rows];
  int64_t mx = 0;
  for (int64_t i = 0; i < rows; ++i) {
    if (rowptr[i + 1] < rowptr[i]) return BFP_ERR_ARG;
    mx = std::max(mx, rowptr[i + 1] - rowptr[i]);
  }
  for (int64_t k = 0; k < nnz; ++k) {
    if (col[k] < 0 || col[k] >= cols) return BFP_ERR_ARG;
    if (msb_h(m[k]) > q) return BFP_ERR_DOMAIN;  // check_fits (src/bfp.cpp:11-14)
  }
  bfp_csr_s* a = new bfp_csr_s();
  size_t words = (size_t)(rows + 1 + 2 * nnz + 1);
  if (cudaMalloc(&a->buf, words * 8) != cudaSuccess) {
    delete a;
    return BFP_ERR_NOMEM;
  }
  cudaMemcpy(a->buf, rowptr, 8 * (rows + 1), cudaMemcpyHostToDevice);
  if (nnz) {
    cudaMemcpy(a->buf + rows + 1, col, 8 * nnz, cudaMemcpyHostToDevice);
    cudaMemcpy(a->buf + rows + 1 + nnz, m, 8 * nnz, cudaMemcpyHostToDevice);
  }
  a->d = CsrDev{rows, cols, q, e, mx, a->buf, a->buf + rows + 1, a->buf + rows + 1 + nnz};
  *out = a;
  return BFP_OK;
}
int bfp_csr_destroy(bfp_csr_t a) {
  if (a) {
    cudaFree(a->buf);
    delete a;
  }
  return BFP_OK;
}

int bfp_spmv_csr(bfp_csr_t a, bfp_vec_t x, int64_t m_a, int mode, int64_t w_out, int64_t w_tmp,
                 bfp_scalar_t gamma, int force, bfp_vec_t out, void* stream) {
  if (!a || !x || !out || gamma.m <= 0) return BFP_ERR_ARG;
  if (a->d.cols != x->nlog || out->nlog != a->d.rows || x->dim || out->dim) return BFP_ERR_ARG;
  if (out == x) return BFP_ERR_ALIAS;
  if (m_a == 0) m_a = a->d.max_row_nnz;
  if (m_a < a->d.max_row_nnz) return BFP_ERR_ARG;  // src/blas.cpp:78-79
  if (x->ebytes != out->ebytes) return BFP_ERR_ARG;
  CsrSpmvOp op;
  op.a = a->d;
  op.x = view(x);
  op.m_a = m_a;
  return launch_flat(op, out, mkp(mode, w_out, w_tmp, gamma, force), S(stream));
}

int bfp_gemv_csr(bfp_csr_t a, bfp_vec_t x, bfp_vec_t y, bfp_scalar_t alpha, bfp_scalar_t beta,
                 int64_t m_a, int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                 int force, bfp_vec_t out, void* stream) {
  if (!a || !x || !y || !out || gamma.m <= 0) return BFP_ERR_ARG;
  if (a->d.cols != x->nlog || a->d.rows != y->nlog || out->nlog != a->d.rows || x->dim || y->dim ||
      out->dim)
    return BFP_ERR_ARG;  // src/blas.cpp:101-103
  if (out == x || out == y) return BFP_ERR_ALIAS;
  if (m_a == 0) m_a = a->d.max_row_nnz;
  if (m_a < a->d.max_row_nnz) return BFP_ERR_ARG;
  if (x->ebytes != out->ebytes || y->ebytes != out->ebytes) return BFP_ERR_ARG;
  CsrGemvOp op;
  op.a = a->d;
  op.x = view(x);
  op.y = view(y);
  op.al = SC(alpha);
  op.be = SC(beta);
  op.m_a = m_a;
  return launch_flat(op, out, mkp(mode, w_out, w_tmp, gamma, force), S(stream));
}

int bfp_qcomp_rows(int64_t n, const int64_t* hi, const uint64_t* lo, int64_t q, int64_t e, int mode,
                   int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma, int force, bfp_vec_t out,
                   void* stream) {
  (void)q;
  if (!out || out->nlog != n || out->dim || gamma.m <= 0) return BFP_ERR_ARG;
  int64_t* buf = nullptr;
  if (cudaMalloc(&buf, 16 * (size_t)std::max<int64_t>(n, 1)) != cudaSuccess) return BFP_ERR_NOMEM;
  if (n) {
    cudaMemcpyAsync(buf, hi, 8 * n, cudaMemcpyHostToDevice, S(stream));
    cudaMemcpyAsync(buf + n, lo, 8 * n, cudaMemcpyHostToDevice, S(stream));
  }
  RowsOp op;
  op.hi = buf;
  op.lo = (const uint64_t*)(buf + n);
  op.e = e;
  int rc = launch_flat(op, out, mkp(mode, w_out, w_tmp, gamma, force), S(stream));
  cudaStreamSynchronize(S(stream));
  cudaFree(buf);
  return rc;
}

int bfp_stencil_gemv(bfp_vec_t x, bfp_vec_t y, bfp_scalar_t alpha, bfp_scalar_t beta, int mode,
                     int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma, int force, bfp_vec_t out,
                     void* stream) {
  if (!x || !y || !out || gamma.m <= 0) return BFP_ERR_ARG;
  return op_gemv(x, y, SC(alpha), SC(beta), mkp(mode, w_out, w_tmp, gamma, force), out,
                 S(stream));
}
int bfp_stencil_jacobi(bfp_vec_t x, bfp_vec_t b, bfp_scalar_t c, int mode, int64_t w_out,
                       int64_t w_tmp, bfp_scalar_t gamma, bfp_vec_t out, void* stream) {
  if (!x || !b || !out || gamma.m <= 0) return BFP_ERR_ARG;
  return op_jacobi(x, b, SC(c), mkp(mode, w_out, w_tmp, gamma, 0), out, S(stream));
}
int bfp_scal(bfp_vec_t r, bfp_scalar_t c, int mode, int64_t w_out, int64_t w_tmp,
             bfp_scalar_t gamma, bfp_vec_t out, void* stream) {
  if (!r || !out || gamma.m <= 0) return BFP_ERR_ARG;
  return op_scal(r, SC(c), mkp(mode, w_out, w_tmp, gamma, 0), out, S(stream));
}
int bfp_restrict_fw(bfp_vec_t r, int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                    bfp_vec_t out, void* stream) {
  if (!r || !out || gamma.m <= 0) return BFP_ERR_ARG;
  return op_restrict(r, mkp(mode, w_out, w_tmp, gamma, 0), out, S(stream));
}
int bfp_prolong(bfp_vec_t xc, int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                bfp_vec_t out, void* stream) {
  if (!xc || !out || gamma.m <= 0) return BFP_ERR_ARG;
  return op_prolong(xc, mkp(mode, w_out, w_tmp, gamma, 0), out, S(stream));
}
int bfp_prolong_correct(bfp_vec_t ec, bfp_vec_t y, int mode, int64_t w_out, int64_t w_tmp,
                        bfp_scalar_t gamma, bfp_vec_t out, void* stream) {
  if (!ec || !y || !out || gamma.m <= 0) return BFP_ERR_ARG;
  return op_prolong_correct(ec, y, mkp(mode, w_out, w_tmp, gamma, 0), out, S(stream));
}
int bfp_vec_create_slab(int dim, int level, int z_lo, int z_hi, int mant_bytes, bfp_vec_t* out) {
  if (dim < 2) return BFP_ERR_ARG;
  return vec_alloc_slab(dim, level, 0, z_lo, z_hi, mant_bytes, out);
}

int bfp_vec_planes(bfp_vec_t v, void** first, void** last, void** halo_lo, void** halo_hi,
                   int64_t* plane_bytes) {
  if (!v || v->dim < 2) return BFP_ERR_ARG;
  const int64_t pe = v->span / v->nz, pb = pe * v->ebytes;
  char* d = (char*)v->data;
  if (first) *first = d;
  if (last) *last = d + (v->nz - 1) * pb;
  if (halo_lo) *halo_lo = d - pb;
  if (halo_hi) *halo_hi = d + v->nz * pb;
  if (plane_bytes) *plane_bytes = pb;
  return BFP_OK;
}

static WinParams mkp_part(int mode, int stage, int64_t w_out, int64_t w_tmp, bfp_scalar_t g,
                          int64_t* d_part) {
  WinParams p = mkp(mode, w_out, w_tmp, g, 0);
  if (stage == 1) p.mode = MODE_RECOMPUTE;
  p.part = d_part;
  return p;
}

int bfp_stencil_gemv_part(bfp_vec_t x, bfp_vec_t y, bfp_scalar_t alpha, bfp_scalar_t beta,
                          int mode, int stage, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                          bfp_vec_t out, int64_t* d_part, void* stream) {
  if (!x || !y || !out || !d_part || gamma.m <= 0 || stage < 0 || stage > 1) return BFP_ERR_ARG;
  return op_gemv(x, y, SC(alpha), SC(beta), mkp_part(mode, stage, w_out, w_tmp, gamma, d_part),
                 out, S(stream));
}

int bfp_stencil_jacobi_part(bfp_vec_t x, bfp_vec_t b, bfp_scalar_t c, int mode, int stage,
                            int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma, bfp_vec_t out,
                            int64_t* d_part, void* stream) {
  if (!x || !b || !out || !d_part || gamma.m <= 0 || stage < 0 || stage > 1) return BFP_ERR_ARG;
  return op_jacobi(x, b, SC(c), mkp_part(mode, stage, w_out, w_tmp, gamma, d_part), out,
                   S(stream));
}

int bfp_window_finalize(bfp_vec_t out, int mode, int stage, int64_t w_out, int64_t w_tmp,
                        const int64_t* d_part, void* stream) {
  if (!out || !d_part || stage < 0 || stage > 1) return BFP_ERR_ARG;
  WinParams p = win_params(stage == 1 ? MODE_RECOMPUTE : (mode == 1 ? MODE_NNQ : MODE_QCOMP),
                           w_out, w_tmp, 0);
  launch_pdl(window_finalize_kernel, 1, 32, 0, S(stream), view(out), p, d_part,
             out->ebytes * 8);
  count_launch();
  return last_launch();
}

int bfp_jacobi_coeff(int dim, int level, int64_t qc, bfp_scalar_t* c) {
  if (dim < 1 || dim > 3 || qc < 2 || qc > 60 || !c) return BFP_ERR_ARG;
  int64_t cm, ce;
  jacobi_coeff(dim, level, qc, &cm, &ce);
  c->m = cm;
  c->q = qc;
  c->e = ce;
  return BFP_OK;
}

int bfp_gen_uniform(bfp_vec_t v, int64_t p, uint64_t seed, uint64_t stream_id, void* stream) {
  if (!v) return BFP_ERR_ARG;
  return gen_uniform(v, p, seed, stream_id, S(stream));
}
int bfp_gen_sine(bfp_vec_t v, int64_t p, void* stream) {
  if (!v) return BFP_ERR_ARG;
  return gen_sine(v, p, S(stream));
}

}  // extern "C"
