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

#include "bfp_kernels.cuh"

using namespace bfpdev;


namespace {
std::atomic<int64_t> g_launches{0};
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_ev;
size_t g_ev_used = 0;
int cuda_status(cudaError_t e) { return e == cudaSuccess ? BFP_OK : BFP_ERR_CUDA; }
}  // namespace

namespace bfp {
bool g_pdl = true;
bool g_skip_recompute = false;
bool g_prof = false;
bool g_use_bulk = true;
std::pair<cudaEvent_t, cudaEvent_t> prof_pair() {
  if (g_ev_used == g_ev.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    g_ev.emplace_back(a, b);
  }
  return g_ev[g_ev_used++];
}
}  // namespace bfp
using bfp::g_prof;
using bfp::g_pdl;
using bfp::g_skip_recompute;
using bfp::g_use_bulk;
using bfp::blocks_for;
using bfp::last_launch;

// multi-rank finalize: apply the all-reduced partials {mu*, max, -min, err} with the
// window context recorded by pass 1 (exactly the single-rank win_finalize)
__global__ void window_finalize_kernel(Vec out, WinParams p, const int64_t* part, int storage_bits) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  griddep_wait();
  finalize_from_partials(out, p, part, storage_bits);
}

// deferred finalize of a multi-block pass 1 (bfpdev::window_reduce): the blocks'
// accumulated {OR, max, min, err} and block 0's window context -> win_finalize, then the
// accumulators are reset for the next op writing this vector
__global__ void deferred_finalize_kernel(Vec out, WinParams p, int storage_bits) {
  griddep_wait();
  griddep_launch_dependents();  // dependents still wait for this grid's completion
  if (threadIdx.x != 0) return;
  deferred_finalize(out, p, storage_bits);
}

namespace bfp {
int launch_deferred_finalize(const Vec& out, const WinParams& p, int storage_bits, cudaStream_t s) {
  launch_pdl(deferred_finalize_kernel, 1, 32, 0, s, out, p, storage_bits);
  count_launch();
  return BFP_OK;
}
}  // namespace bfp

#ifdef BFP_TIMING
static long long* g_dbg = nullptr;  // record 0: launch counter; 4095 ring records of 8 stamps
extern "C" int bfp_dbg_stamps(long long* out, int n) {
  cudaDeviceSynchronize();
  if (!g_dbg) return 0;
  cudaMemcpy(out, g_dbg, sizeof(long long) * 8 * (size_t)n, cudaMemcpyDeviceToHost);
  cudaMemset(g_dbg, 0, sizeof(long long) * 8 * 4096);
  return 1;
}
#endif

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
    pad = ix == m || o > m;  // o > m: storage padding of the 1-D level 1 (N = 2)
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

// ===========================================================================
// host side

namespace bfp {

void count_launch(int n) { g_launches += n; }
static std::atomic<int64_t> g_family[FAM_N];
void count_family(int fam) { g_family[fam] += 1; }
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
    if (level < (dim == 3 ? 2 : 1) || level > 30 || (int64_t)dim * level > 36) {  // 2-D level 1: ref mode
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
    if (dim == 1 && v->span < 4) v->span = 4;  // level 1: one point + pad, padded to a 4-group
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
  if (v->dot_acc) cudaFree(v->dot_acc);
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

// finalize of a partial (multi-rank) window from all-reduced partials; p carries the
// op's trace / history slots (stage 1 = the recompute pass)
int window_finalize(bfp_vec_s* out, WinParams p, int stage, const int64_t* part, cudaStream_t s) {
  if (stage == 1) p.mode = MODE_RECOMPUTE;
  p.part = nullptr;
  launch_pdl(window_finalize_kernel, 1, 32, 0, s, view(out), p, part, out->ebytes * 8);
  count_launch();
  return last_launch();
}

WinParams win_params(int mode, int64_t w_out, int64_t w_tmp, int force) {
  WinParams p;
  memset(&p, 0, sizeof(p));
#ifdef BFP_TIMING
  if (!g_dbg) {
    cudaMalloc(&g_dbg, sizeof(long long) * 8 * 4096);
    cudaMemset(g_dbg, 0, sizeof(long long) * 8 * 4096);
  }
  p.dbg = g_dbg;
#endif
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

// quantize_exact (src/bfp.cpp:163-187) over entries z_i * 2^k_i given per logical index
// by a source: top = max msb(z_i) + k_i over nonzero entries, e_out = top - w,
// m_i = floor(z_i * 2^(k_i - e_out)); an all-zero input gives e_out = 0
struct SrcZK {  // mantissa / exponent pairs
  const int64_t *z, *k;
  __device__ bool get(int64_t i, int64_t& zz, int64_t& kk) const {
    zz = z[i];
    kk = k[i];
    return zz != 0;
  }
};
struct SrcDbl {  // IEEE doubles (from_extfloat, src/bfp.cpp:189-194): v = z * 2^k exactly
  const double* v;
  __device__ bool get(int64_t i, int64_t& zz, int64_t& kk) const {
    const double d = v[i];
    if (d == 0.0) return false;
    split_double(d, zz, kk);
    return true;
  }
};
template <typename Src>
__global__ void __launch_bounds__(kThreads) qe_top_kernel(Vec v, Src src, int64_t* top) {
  int64_t t = INT64_MIN;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < v.n; o += stride) {
    bool pad;
    const int64_t i = logical_of(v, o, pad);
    int64_t z, k;
    if (pad || !src.get(i, z, k)) continue;
    const int64_t b = msb(z) + k;
    t = b > t ? b : t;
  }
  t = shfl_max64(t);
  if ((threadIdx.x & 31) == 0 && t != INT64_MIN) atomicMax((long long*)top, (long long)t);
}
template <typename M, typename Src>
__global__ void __launch_bounds__(kThreads) qe_write_kernel(Vec v, Src src, const int64_t* top,
                                                            int64_t w) {
  const int64_t tp = *top;
  const int64_t e_out = tp != INT64_MIN ? tp - w : 0;
  Red r;
  r.init();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < v.n; o += stride) {
    bool pad;
    const int64_t i = logical_of(v, o, pad);
    int64_t z, k, m = 0;
    if (!pad && src.get(i, z, k)) {
      const int64_t s = e_out - k;  // shift_floor(z, s), src/wideint.cpp:94-99
      m = s >= 0 ? (s >= 63 ? (z < 0 ? -1 : 0) : (z >> s)) : (int64_t)((uint64_t)z << (-s));
    }
    ((M*)v.data)[o] = (M)m;
    r.val(m);
  }
  reduce_and_finalize(r, v.hdr, [&](int, int64_t mx, int64_t mn, int) {
    Hdr* h = v.hdr;
    h->q = w;
    h->e = e_out;
    h->shift = 0;
    h->max_m = mx;
    h->min_m = mn;
    h->flags = 0;
    h->need_recompute = 0;
    h->err = 0;
  });
}
template <typename Src>
static int quantize_exact_impl(bfp_vec_s* v, Src src, int64_t w, int64_t* top, cudaStream_t s) {
  set_i64_kernel<<<1, 1, 0, s>>>(top, INT64_MIN);
  Vec d = view(v);
  const int b = blocks_for(v->span);
  qe_top_kernel<Src><<<b, kThreads, 0, s>>>(d, src, top);
  if (v->ebytes == 4)
    qe_write_kernel<int32_t, Src><<<b, kThreads, 0, s>>>(d, src, top, w);
  else
    qe_write_kernel<int64_t, Src><<<b, kThreads, 0, s>>>(d, src, top, w);
  count_launch(3);
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

int bfp_kernel_family_counts(int64_t* counts, int n) {
  if (!counts || n < 0) return BFP_ERR_ARG;
  for (int i = 0; i < n && i < FAM_N; ++i) counts[i] = g_family[i].load();
  return BFP_OK;
}

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
  // One contiguous H2D copy into a staging buffer at the full PCIe rate, then a scatter
  // kernel into the padded layout (HBM speed, hidden behind the next copy).  A pitched DMA
  // (cudaMemcpy3DAsync) straight into the padded layout was measured 3.2x slower end to
  // end: 2 KB rows run the copy engine at a quarter of its rate
  // (profiles/r2/r2h_upload_ab.txt).
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

int bfp_quantize_exact(const int64_t* z, const int64_t* k, int64_t n, int64_t w, bfp_vec_t out,
                       void* stream) {
  if (!out || n != out->nlog || (n > 0 && (!z || !k)) || w < 1 || w > out->ebytes * 8)
    return BFP_ERR_ARG;
  cudaStream_t s = S(stream);
  int64_t* buf = nullptr;  // top scratch + z + k
  if (cudaMallocAsync((void**)&buf, sizeof(int64_t) * (1 + 2 * (size_t)n), s) != cudaSuccess)
    return BFP_ERR_NOMEM;
  int rc = BFP_OK;
  if (n > 0 && (cudaMemcpyAsync(buf + 1, z, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s) !=
                    cudaSuccess ||
                cudaMemcpyAsync(buf + 1 + n, k, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s) !=
                    cudaSuccess))
    rc = BFP_ERR_CUDA;
  if (!rc) rc = bfp::quantize_exact_impl(out, bfp::SrcZK{buf + 1, buf + 1 + n}, w, buf, s);
  cudaFreeAsync(buf, s);
  return rc;
}

int bfp_from_doubles(const double* v, int64_t n, int64_t w, bfp_vec_t out, void* stream) {
  if (!out || n != out->nlog || (n > 0 && !v) || w < 1 || w > out->ebytes * 8) return BFP_ERR_ARG;
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return BFP_ERR_ARG;
  cudaStream_t s = S(stream);
  char* buf = nullptr;
  if (cudaMallocAsync((void**)&buf, sizeof(int64_t) + sizeof(double) * (size_t)n, s) !=
      cudaSuccess)
    return BFP_ERR_NOMEM;
  double* d = reinterpret_cast<double*>(buf + sizeof(int64_t));
  int rc = BFP_OK;
  if (n > 0 &&
      cudaMemcpyAsync(d, v, sizeof(double) * n, cudaMemcpyHostToDevice, s) != cudaSuccess)
    rc = BFP_ERR_CUDA;
  if (!rc) rc = bfp::quantize_exact_impl(out, bfp::SrcDbl{d}, w, (int64_t*)buf, s);
  cudaFreeAsync(buf, s);
  return rc;
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
  WinParams p = win_params(mode == 1 ? MODE_NNQ : MODE_QCOMP, w_out, w_tmp, 0);
  return bfp::window_finalize(out, p, stage, d_part, S(stream));
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
