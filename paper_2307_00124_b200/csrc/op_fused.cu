// op_fused.cu -- fused single-CTA op lists (shared-memory arena) for coarse levels.
#include "bfp_lean.cuh"

namespace bfp {

// The lean engine's digest of the record (bfp_internal.h: LeanRec): the static fields, and
// `ok` = every static condition of the fast path holds (the dynamic ones -- operand widths
// and exponents -- are checked per op on the device, bfp_lean.cuh: lean_post).  Vector ids
// and data pointers are filled in when the arena is laid out (bfp_solver.cu).
static void lean_digest(FusedOp* f) {
  LeanRec& r = f->lr;
  memset(&r, 0, sizeof(r));
  r.vout = r.va = r.vb = 0xff;
  r.gv[0] = r.gv[1] = r.gv[2] = 0xff;
  const WinParams& p = f->p;
  auto small_e = [](int64_t e) { return e > -(1 << 20) && e < (1 << 20); };
  auto fits = [](int64_t m) { return m == (int64_t)(int32_t)m; };
  r.n4 = (int32_t)(f->out.n >> 2);
  r.w_out = (int16_t)p.w_out;
  r.nnq = p.mode == MODE_NNQ;
  bool ok = f->out.ebytes == 4;
  if (f->kind != FK_ZERO) {
    ok = ok && !p.part && !p.force && p.w_tmp <= 32 && p.w_out >= 1 && p.w_out <= 32 &&
         (p.mode == MODE_QCOMP || p.mode == MODE_NNQ);
    const GammaRule& g = p.gamma;
    ok = ok && !g.literal && !g.exact && g.nterms <= 3;
    for (int i = 0; ok && i < g.nterms; ++i)
      ok = g.t[i].cm >= 0 && g.t[i].cm <= 0xffffffffll && small_e(g.t[i].ce);
    r.ng = (uint8_t)(g.literal ? 0 : g.nterms);
  }
  auto coef = [&](const Scal& a, const Scal& b) {
    ok = ok && fits(a.m) && fits(b.m) && small_e(a.e) && small_e(b.e);
    r.am = (int32_t)a.m, r.ae = (int32_t)a.e, r.bm = (int32_t)b.m, r.be = (int32_t)b.e;
  };
  switch (f->kind) {
    case FK_GEMV: {
      const GemvOp& g = f->u.gemv;
      ok = ok && !g.st9 && !g.gs && g.l >= 2 && !g.z0;
      coef(g.al, g.be);
      r.dim = (int8_t)g.dim, r.l = (int8_t)g.l, r.ea = g.ea;
      break;
    }
    case FK_JACOBI: {
      const JacobiOp& j = f->u.jac;
      ok = ok && j.l >= 2 && !j.z0 && j.c.m >= 0 && j.c.m <= 0x7fffffff;
      coef(j.c, Scal{0, 0, 0});
      r.dim = (int8_t)j.dim, r.l = (int8_t)j.l, r.ea = 2 * j.l;
      break;
    }
    case FK_SCAL: coef(f->u.scal.c, Scal{0, 0, 0}); break;
    case FK_AXPBY: coef(f->u.axpby.al, f->u.axpby.be); break;
    case FK_RESTRICT: {
      const RestrictOp& q = f->u.rst;
      ok = ok && !q.gs && !q.zc && q.l >= 3;
      r.dim = (int8_t)q.dim, r.l = (int8_t)q.l, r.ea = q.er;
      break;
    }
    case FK_PROLONG: {
      const ProlongOp& q = f->u.pro;
      ok = ok && !q.gs && !q.zf && !q.zp && q.l >= 3;
      r.dim = (int8_t)q.dim, r.l = (int8_t)q.l, r.ea = q.ep;
      break;
    }
    case FK_PCORR: {
      const ProlongCorrectOp& q = f->u.pc;
      ok = ok && !q.gs && !q.zf && !q.zp && q.l >= 3 && q.al.m == 1 && q.be.m == 1;
      coef(q.al, q.be);
      r.dim = (int8_t)q.dim, r.l = (int8_t)q.l, r.ea = q.ep;
      break;
    }
    default: break;
  }
  r.ok = ok;
}

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
    case FK_ZERO: memset(&f->p, 0, sizeof(f->p)); break;  // no window, no gamma rule
    default: return BFP_ERR_ARG;
  }
  lean_digest(f);
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
