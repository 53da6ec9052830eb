// write_tiles.cu -- write-only ceiling of the tiled plane march: every CTA owns a W x H tile
// of an N x N plane and marches planes along z, each warp storing int4 per lane (the store
// pattern of the prolongation / stencil marches), against a flat coalesced fill.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o write_tiles write_tiles.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int H>
__global__ void __launch_bounds__(W / 4 * H) tile_march(int* out, int l, int R, int v) {
  const int N = 1 << l;
  const size_t N2 = (size_t)N * N;
  const int tx = N / W, ty = N / H, chunks = (N + R - 1) / R;
  const int lane4 = threadIdx.x % (W / 4), row = threadIdx.x / (W / 4);
  for (int item = blockIdx.x; item < tx * ty * chunks; item += gridDim.x) {
    const int tile = item % (tx * ty), ch = item / (tx * ty);
    const int x0 = (tile % tx) * W, y0 = (tile / tx) * H;
    int* p = out + (size_t)ch * R * N2 + (size_t)(y0 + row) * N + x0 + 4 * lane4;
    const int n = min(R, N - ch * R);
    for (int k = 0; k < n; ++k) {
      *reinterpret_cast<int4*>(p) = make_int4(v, v + k, v, v);
      p += N2;
    }
  }
}
__global__ void flat_fill(int4* out, size_t n4, int v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    out[i] = make_int4(v, v, v, v);
}

template <typename F> float best(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float t = 1e9f;
  for (int i = 0; i < 8; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    t = ms < t ? ms : t;
  }
  return t;
}

int main() {
  const int l = 9;
  const size_t n = (size_t)1 << (3 * l);
  int* d[2];
  for (auto& p : d) cudaMalloc(&p, n * 4);
  int flip = 0;
  auto rep = [&](const char* name, float ms) {
    printf("%-28s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, n * 4 / (ms * 1e-3) / 1e9);
  };
  rep("flat fill (148x8 CTAs)", best([&] { flat_fill<<<148 * 8, 256>>>((int4*)d[flip ^= 1], n / 4, 3); }));
  for (int ctas : {2, 4, 8}) {
    for (int R : {64, 128, 222, 512}) {
      char nm[64];
      snprintf(nm, sizeof nm, "128x8  %d/SM R=%d", ctas, R);
      rep(nm, best([&] { tile_march<128, 8><<<148 * ctas, 256>>>(d[flip ^= 1], l, R, 3); }));
      snprintf(nm, sizeof nm, "256x4  %d/SM R=%d", ctas, R);
      rep(nm, best([&] { tile_march<256, 4><<<148 * ctas, 256>>>(d[flip ^= 1], l, R, 3); }));
      snprintf(nm, sizeof nm, "512x2  %d/SM R=%d", ctas, R);
      rep(nm, best([&] { tile_march<512, 2><<<148 * ctas, 256>>>(d[flip ^= 1], l, R, 3); }));
      snprintf(nm, sizeof nm, "512x4(512thr) %d/SM R=%d", ctas, R);
      rep(nm, best([&] { tile_march<512, 4><<<148 * ctas, 512>>>(d[flip ^= 1], l, R, 3); }));
    }
  }
  return 0;
}
