// op_dot.cu -- exact BFP dot product <x, y> = sum_i m_x,i m_y,i * 2^(e_x + e_y).
//
// No reference function exists; the paper discusses the exact dot of two BFP blocks
// and config 5 asks for 128-bit exact accumulation and a dot-product
// all-reduce.  Products of int64 mantissas are ~126 bits and a 1023^3 sum adds 30 more,
// so the accumulation is wider than 128 bits:
//
//   * each thread adds its sign-extended 128-bit products into a 192-bit two's
//     complement accumulator (add.cc / addc.cc / addc: exact, branch free);
//   * the 192 bits are split into four 48-bit limbs (three unsigned, the top one signed)
//     and the block sums each limb in 64 bits (256 x 2^48 < 2^56);
//   * one thread per block adds the block's limbs into the caller's device accumulator
//     with 64-bit atomics (<= 148 x 8 blocks: < 2^59 per limb; integer addition is
//     associative, so the order of the atomics cannot change the value).
//
// The device result is 5 int64: the limb sums L0..L3 (value = sum_k L_k 2^(48k)) and
// the exponent e_x + e_y.  A multi-rank dot all-reduces the four limbs with an int64 SUM
// (NCCL has no 128-bit type; eight ranks stay below 2^62), and bfp_dot_value turns limbs
// into the exact 192-bit two's complement value, flagging results beyond 128 bits.
// Everything is stream-ordered (a memset + one kernel): no allocation, no host
// synchronisation, graph-capturable.
#include "bfp_kernels.cuh"

namespace {

__device__ __forceinline__ void add192(uint64_t& w0, uint64_t& w1, uint64_t& w2, i128 p) {
  const u128 up = (u128)p;
  const uint64_t lo = (uint64_t)up, hi = (uint64_t)(up >> 64);
  const uint64_t sx = (uint64_t)((int64_t)hi >> 63);
  asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
      : "+l"(w0), "+l"(w1), "+l"(w2)
      : "l"(lo), "l"(hi), "l"(sx));
}

__device__ __forceinline__ int64_t warp_sum(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename M>
__global__ void __launch_bounds__(kThreads) dot_limb_kernel(Vec x, Vec y,
                                                            unsigned long long* acc) {
  const int64_t sx = x.hdr->shift, sy = y.hdr->shift;
  uint64_t w0 = 0, w1 = 0, w2 = 0;
  const int64_t ng = x.n >> 2, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += stride) {
    int64_t a[4], b[4];
    V4<M>::load(x, g * 4, sx, a);
    V4<M>::load(y, g * 4, sy, b);
#pragma unroll
    for (int j = 0; j < 4; ++j) add192(w0, w1, w2, (i128)a[j] * (i128)b[j]);
  }
  constexpr uint64_t M48 = (1ull << 48) - 1;
  int64_t l[4] = {(int64_t)(w0 & M48), (int64_t)(((w0 >> 48) | (w1 << 16)) & M48),
                  (int64_t)(((w1 >> 32) | (w2 << 32)) & M48), (int64_t)w2 >> 16};
  __shared__ int64_t s_l[4][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    l[k] = warp_sum(l[k]);
    if (lane == 0) s_l[k][wid] = l[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t[4];
    for (int k = 0; k < 4; ++k) {
      t[k] = 0;
      for (int w = 0; w < nw; ++w) t[k] += s_l[k][w];
    }
    // carry-normalise the block sums (limbs 0..2 back below 2^48) before the cross-block
    // atomics: <= 148 x 8 blocks then keep every limb below 2^59
    for (int k = 0; k < 3; ++k) {
      t[k + 1] += t[k] >> 48;
      t[k] &= (int64_t)M48;
    }
    for (int k = 0; k < 4; ++k) atomicAdd(acc + k, (unsigned long long)t[k]);
    if (blockIdx.x == 0) acc[4] = (unsigned long long)(x.hdr->e + y.hdr->e);
  }
}

// carry-normalise a device accumulator (limbs 0..2 in [0, 2^48)) before a multi-rank SUM
__global__ void limb_norm_kernel(int64_t* acc) {
  if (threadIdx.x == 0) {
    for (int k = 0; k < 3; ++k) {
      acc[k + 1] += acc[k] >> 48;
      acc[k] &= (int64_t)((1ull << 48) - 1);
    }
  }
}

// LocalComm: sum the limbs of the in-process ranks' accumulators (every rank gets the sum)
__global__ void limb_sum_kernel(bfp::LimbPtrs acc, int P) {
  const int k = threadIdx.x;
  if (k >= 4) return;
  int64_t t = 0;
  for (int r = 0; r < P; ++r) t += acc.p[r][k];
  for (int r = 0; r < P; ++r) acc.p[r][k] = t;
}

}  // namespace

namespace bfp {

int dot_limbs(bfp_vec_s* x, bfp_vec_s* y, int64_t* d_acc, cudaStream_t s, bool normalise) {
  if (!x || !y || !d_acc || x->span != y->span || x->ebytes != y->ebytes || x->dim != y->dim ||
      x->nz != y->nz)
    return BFP_ERR_ARG;
  if (cudaMemsetAsync(d_acc, 0, 4 * sizeof(int64_t), s) != cudaSuccess) return BFP_ERR_CUDA;
  const int nb = blocks_for(x->span / 4);
  if (x->ebytes == 4)
    dot_limb_kernel<int32_t><<<nb, kThreads, 0, s>>>(view(x), view(y), (unsigned long long*)d_acc);
  else
    dot_limb_kernel<int64_t><<<nb, kThreads, 0, s>>>(view(x), view(y), (unsigned long long*)d_acc);
  count_launch();
  if (normalise) {
    limb_norm_kernel<<<1, 32, 0, s>>>(d_acc);
    count_launch();
  }
  return last_launch();
}

int limb_sum_local(int64_t* const* d_ptrs, int P, cudaStream_t s) {
  if (P < 1 || P > kMaxLimbRanks) return BFP_ERR_ARG;
  LimbPtrs a;
  for (int r = 0; r < P; ++r) a.p[r] = d_ptrs[r];
  limb_sum_kernel<<<1, 32, 0, s>>>(a, P);
  count_launch();
  return last_launch();
}

}  // namespace bfp

using namespace bfp;

extern "C" {

int bfp_dot_exact_async(bfp_vec_t x, bfp_vec_t y, int64_t* d_acc, void* stream) {
  return dot_limbs(x, y, d_acc, reinterpret_cast<cudaStream_t>(stream), false);
}

int bfp_dot_value(const int64_t* acc, uint64_t* words, int64_t* hi, uint64_t* lo) {
  if (!acc) return BFP_ERR_ARG;
  // sum_k L_k 2^(48k) mod 2^192; |value| < 2^191 by construction, so this is exact
  uint64_t w[3] = {0, 0, 0};
  for (int k = 0; k < 4; ++k) {
    const int sh = 48 * k;
    const int64_t L = acc[k];
    const uint64_t sx = (uint64_t)(L >> 63);
    uint64_t t[3] = {0, 0, 0};  // L * 2^sh as 192-bit two's complement
    const int q = sh / 64, r = sh % 64;
    uint64_t ext[4] = {(uint64_t)L, sx, sx, sx};
    for (int i = 0; i < 3; ++i) {
      const int j = i - q;
      if (j < 0) continue;
      t[i] = r ? (ext[j] << r) | (j > 0 ? ext[j - 1] >> (64 - r) : 0) : ext[j];
    }
    unsigned __int128 c = 0;
    for (int i = 0; i < 3; ++i) {
      c += (unsigned __int128)w[i] + t[i];
      w[i] = (uint64_t)c;
      c >>= 64;
    }
  }
  if (words) memcpy(words, w, sizeof(w));
  if (hi) *hi = (int64_t)w[1];
  if (lo) *lo = w[0];
  // fits 128 bits iff the top word is the sign extension of bit 127
  const bool fits = w[2] == (uint64_t)((int64_t)w[1] >> 63);
  return fits ? BFP_OK : BFP_ERR_WIDTH;
}

int bfp_dot_exact(bfp_vec_t x, bfp_vec_t y, int64_t* hi, uint64_t* lo, int64_t* e, void* stream) {
  if (!x || !y) return BFP_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!x->dot_acc && cudaMalloc(&x->dot_acc, 8 * sizeof(int64_t)) != cudaSuccess)
    return BFP_ERR_NOMEM;  // once per vector, reused by every later call
  int rc = dot_limbs(x, y, x->dot_acc, s, false);
  if (rc) return rc;
  int64_t acc[5];
  if (cudaMemcpyAsync(acc, x->dot_acc, sizeof(acc), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return BFP_ERR_CUDA;
  if (e) *e = acc[4];
  return bfp_dot_value(acc, nullptr, hi, lo);
}

int bfp_dot_exact192(bfp_vec_t x, bfp_vec_t y, uint64_t* words, int64_t* e, void* stream) {
  if (!x || !y || !words) return BFP_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!x->dot_acc && cudaMalloc(&x->dot_acc, 8 * sizeof(int64_t)) != cudaSuccess)
    return BFP_ERR_NOMEM;
  int rc = dot_limbs(x, y, x->dot_acc, s, false);
  if (rc) return rc;
  int64_t acc[5];
  if (cudaMemcpyAsync(acc, x->dot_acc, sizeof(acc), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return BFP_ERR_CUDA;
  if (e) *e = acc[4];
  bfp_dot_value(acc, words, nullptr, nullptr);  // 192 bits always hold the exact value
  return BFP_OK;
}

}  // extern "C"
