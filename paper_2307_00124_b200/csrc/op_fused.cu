// op_fused.cu -- fused single-CTA op lists (shared-memory arena) for coarse levels.
#include "bfp_lean.cuh"

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
      f->u.gemv.ea = 2 * a->l; f->u.gemv.gs = 0;
      break;
    case FK_JACOBI:
      f->u.jac.x = view(a); f->u.jac.b = view(b); f->u.jac.c = s1;
      f->u.jac.dim = a->dim; f->u.jac.l = a->l; f->u.jac.z0 = a->z0;
      break;
    case FK_SCAL: f->u.scal.r = view(a); f->u.scal.c = s1; break;
    case FK_AXPBY:
      f->u.axpby.x = view(a); f->u.axpby.y = view(b); f->u.axpby.al = s1; f->u.axpby.be = s2;
      break;
    case FK_RESTRICT:
      f->u.rst.r = view(a); f->u.rst.dim = a->dim; f->u.rst.l = a->l; f->u.rst.zc = 0;
      f->u.rst.er = -2 * a->dim; f->u.rst.gs = 0;
      break;
    case FK_PROLONG:
      f->u.pro.xc = view(a); f->u.pro.dim = out->dim; f->u.pro.l = out->l;
      f->u.pro.zf = f->u.pro.zp = 0;
      f->u.pro.ep = -out->dim; f->u.pro.gs = 0;
      break;
    case FK_PCORR:
      f->u.pc.ec = view(a); f->u.pc.y = view(b); f->u.pc.dim = out->dim; f->u.pc.l = out->l;
      f->u.pc.zf = f->u.pc.zp = 0;
      f->u.pc.ep = -out->dim; f->u.pc.gs = 0;
      f->u.pc.al = Scal{1, 2, 0}; f->u.pc.be = Scal{1, 2, 0};
      break;
    case FK_ZERO: break;
    default: return BFP_ERR_ARG;
  }
  return BFP_OK;
}

int fused_launch(const FusedOp* d_ops, int n, const ArenaEntry* d_ar, int nar, int arena_bytes,
                 int zoff, int64_t* zglobal, int loff, int ebytes, cudaStream_t s) {
  static std::atomic<int> attr[kMaxDev];  // function attributes are per device
  per_device(attr, [] {
    cudaFuncSetAttribute(lean_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kArenaMaxBytes);
    cudaFuncSetAttribute(coarse_kernel<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kArenaMaxBytes);
    return 1;
  });
  // int32 storage: the lean engine (generic path inside); int64 storage: the generic engine
  if (ebytes == 4)
    launch_pdl(lean_kernel, 1, kFusedThreads, (size_t)arena_bytes, s, d_ops, n, d_ar, nar, zoff,
               zglobal, loff);
  else
    launch_pdl(coarse_kernel<int64_t>, 1, kFusedThreads, (size_t)arena_bytes, s, d_ops, n, d_ar,
               nar);
  count_launch();
  count_family(FAM_FUSED);
  return last_launch();
}

}  // namespace bfp

#ifdef BFP_COARSE_TIMING
// measurement builds: per-phase clock totals of coarse_kernel (read and reset)
extern "C" int bfp_dbg_coarse(long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_coarse_prof, sizeof(long long) * 16);
  long long z[16] = {};
  cudaMemcpyToSymbol(g_coarse_prof, z, sizeof(z));
  return 16;
}
extern "C" int bfp_dbg_coarse_ops(int* out, int n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_coarse_ops, sizeof(int) * 4 * (size_t)n);
  return n;
}
#endif
