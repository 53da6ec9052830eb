// Cycle cost of the one-thread window setup / finalize of a grid op (the serial part of
// every single-block coarse-level launch): GemvOp::setup, win_setup (config gamma rule with
// two norm terms), win_finalize.  Headers in global memory (L2-resident), clock64 per phase.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o setup_cost setup_cost.cu
#include <cstdio>
#include <cstring>
#include "../../paper_2307_00124_b200/csrc/bfp_ops.cuh"
using namespace bfpdev;

__global__ void k(Vec x, Vec y, Vec out, WinParams p, long long* t) {
  if (threadIdx.x) return;
  long long t0 = clock64();
  GemvOp op;
  memset(&op, 0, sizeof(op));
  op.x = x; op.y = y; op.al = Scal{-1, 1, 0}; op.be = Scal{1, 2, 0};
  op.dim = 2; op.l = 3; op.z0 = 0; op.ea = 6; op.gs = 0; op.st9 = 0;
  int64_t e_star = 0, need = 0;
  op.setup(e_star, need);
  long long t1 = clock64();
  WinCtx c;
  win_setup(p, out.hdr, e_star, 32, c);
  long long t2 = clock64();
  win_finalize(p, c, out.hdr, 20, 12345, -4321, 0);
  long long t3 = clock64();
  G15 a = gterm_eval(p.gamma.t[0]);
  long long t4 = clock64();
  G15 b = gterm_eval(p.gamma.t[1]);
  long long t5 = clock64();
  G15 s = g15_add(G15{0, 0}, a);
  s = g15_add(s, b);
  long long t6 = clock64();
  uint64_t ma = max_abs(x.hdr);
  long long t7 = clock64();
  G15 f = g15_from(ma, 3);
  long long t8 = clock64();
  volatile int sink = (int)need + (int)c.lam + (op.narrow ? 1 : 0) + (int)s.m + (int)f.m;
  (void)sink;
  t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2;
  t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5; t[6] = t7 - t6; t[7] = t8 - t7;
}

int main() {
  Hdr h[3];
  memset(h, 0, sizeof(h));
  for (int i = 0; i < 3; ++i) {
    h[i].q = 20; h[i].e = -19 - i; h[i].max_m = 500000 + i; h[i].min_m = -400000; h[i].shift = 0;
  }
  Hdr* dh;
  cudaMalloc(&dh, sizeof(h));
  cudaMemcpy(dh, h, sizeof(h), cudaMemcpyHostToDevice);
  Vec x{}, y{}, o{};
  x.hdr = dh; y.hdr = dh + 1; o.hdr = dh + 2;
  x.dim = y.dim = o.dim = 2; x.l = y.l = o.l = 3;
  WinParams p;
  memset(&p, 0, sizeof(p));
  p.w_out = 20; p.w_tmp = 25; p.mode = MODE_QCOMP; p.trace_slot = -1; p.hist_slot = -1;
  p.gamma.nterms = 2;
  p.gamma.t[0].v = dh; p.gamma.t[0].cm = 0;
  p.gamma.t[1].v = dh + 1; p.gamma.t[1].cm = 3; p.gamma.t[1].ce = 2;
  long long* dt;
  cudaMalloc(&dt, 64);
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 32>>>(x, y, o, p, dt);
    long long t[8];
    cudaMemcpy(t, dt, sizeof(t), cudaMemcpyDeviceToHost);
    printf("op.setup %lld  win_setup(gamma) %lld  win_finalize %lld | term0 %lld term1 %lld add2 %lld max_abs %lld g15_from %lld cyc (%s)\n",
           t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
