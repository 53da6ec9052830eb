// Latency floor of dependent kernel chains on B200 (graph replay, PDL on/off):
// empty kernels, one dependent header read/write per kernel, multi-block last-block
// reductions, a serial chain of dependent loads in thread 0.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void gd_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void gd_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct H { long long v[16]; unsigned int done; };

__global__ void k_empty(H* h) { gd_wait(); gd_launch(); }
__global__ void k_rw(H* h, int chain) {  // thread 0: `chain` dependent loads, one store
  gd_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    volatile long long* p = h->v;
    long long a = p[0];
    for (int i = 1; i < chain; ++i) a = p[(a & 7) + 1] + a;  // dependent
    h->v[0] = a & 7;
  }
  gd_launch();
}
__global__ void k_lastblock(H* h) {  // every block: atomic + fence + counter; last block finalizes
  gd_wait();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    atomicMax((unsigned long long*)&h->v[2], (unsigned long long)blockIdx.x);
    __threadfence();
    unsigned d = atomicAdd(&h->done, 1u);
    last = d == gridDim.x - 1;
  }
  __syncthreads();
  gd_launch();
  if (last && threadIdx.x == 0) {
    __threadfence();
    volatile H* vh = h;
    long long m = vh->v[2];
    h->v[3] = m;
    h->v[2] = 0;
    h->done = 0;
  }
}
// persistent: n ops separated by a software grid barrier (sense-reversing counter)
__device__ __forceinline__ void grid_barrier(unsigned int* cnt, volatile unsigned int* gen, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g = *gen;
    __threadfence();
    if (atomicAdd(cnt, 1u) == nb - 1) {
      *cnt = 0;
      __threadfence();
      atomicAdd((unsigned int*)gen, 1u);
    } else {
      while (*gen == g) { }
    }
    __threadfence();
  }
  __syncthreads();
}
__global__ void k_persist(H* h, unsigned int* bar, int n) {
  gd_wait();
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x == 0) atomicMax((unsigned long long*)&h->v[4 + (i & 3)], (unsigned long long)(blockIdx.x + i));
    grid_barrier(bar, bar + 32, gridDim.x);
  }
}

template <typename F>
float time_graph(cudaStream_t s, int n, F launch) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) launch();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return best * 1e3f / n;
}

template <typename... KArgs, typename... Args>
void lpdl(bool pdl, void (*k)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

int main() {
  H* h;
  unsigned int* bar;
  cudaMalloc(&h, sizeof(H));
  cudaMemset(h, 0, sizeof(H));
  cudaMalloc(&bar, 256);
  cudaMemset(bar, 0, 256);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int n = 400;
  for (int pdl = 0; pdl <= 1; ++pdl) {
    for (int grid : {1, 16, 148, 592})
      printf("pdl=%d empty grid=%4d: %6.2f us/kernel\n", pdl, grid,
             time_graph(s, n, [&] { lpdl(pdl, k_empty, grid, 256, s, h); }));
    for (int chain : {1, 2, 4, 8})
      printf("pdl=%d rw chain=%d: %6.2f us/kernel\n", pdl, chain,
             time_graph(s, n, [&] { lpdl(pdl, k_rw, 1, 256, s, h, chain); }));
    for (int grid : {2, 16, 148, 592})
      printf("pdl=%d lastblock grid=%4d: %6.2f us/kernel\n", pdl, grid,
             time_graph(s, n, [&] { lpdl(pdl, k_lastblock, grid, 256, s, h); }));
  }
  for (int grid : {16, 74, 148}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_persist<<<grid, 256, 0, s>>>(h, bar, 100);
    cudaEventRecord(a, s);
    k_persist<<<grid, 256, 0, s>>>(h, bar, 1000);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("persistent grid barrier grid=%d: %6.2f us/barrier (%s)\n", grid, ms * 1e3f / 1000,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
