// op_transfer.cu -- pointwise and grid-transfer ops (scal, axpby, restriction,
// prolongation, prolong + correct).
#include "bfp_kernels.cuh"

namespace bfp {

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

// slabs (multi-rank, dim >= 2): a fine slab [2 zc, 2 zc + 2 nzc) restricts to the coarse
// slab [zc, zc + nzc) (one fine halo plane above); a fine slab prolongs from the aligned
// coarse slab (one coarse halo plane below) or from a full (replicated) coarse grid
static bool aligned(const bfp_vec_s* fine, const bfp_vec_s* coarse) {
  return fine->dim >= 2 && fine->z0 == 2 * coarse->z0 && fine->nz == 2 * coarse->nz;
}

int op_restrict(bfp_vec_s* r, const WinParams& p, bfp_vec_s* out, cudaStream_t s, int er,
                int gs) {
  if (r->dim < 1 || out->dim != r->dim || out->l != r->l - 1 || out->ebytes != r->ebytes)
    return BFP_ERR_ARG;
  if (!(full_grid(r) && full_grid(out)) && !aligned(r, out)) return BFP_ERR_ARG;
  RestrictOp op;
  op.r = view(r);
  op.dim = r->dim;
  op.l = r->l;
  op.zc = out->z0;
  op.er = er == kDefaultRep ? -2 * r->dim : er;
  op.gs = gs;
  if (gs) return launch_grid(op, out, p, s);
  static const int r3 = min_level("BFP_RST3_MIN_L", 7), r2 = min_level("BFP_RST2_MIN_L", 9);
  if (g_use_bulk && out->dim == 3 && out->l >= r3)
    return out->ebytes == 4 ? launch_rst3<int32_t>(op, out, p, s) : launch_rst3<int64_t>(op, out, p, s);
  if (g_use_bulk && out->dim == 2 && out->ebytes == 4 && out->l >= r2) return launch_rst2(op, out, p, s);
  return launch_grid(op, out, p, s);
}

static bool prolong_ok(const bfp_vec_s* xc, const bfp_vec_s* fine) {
  if (xc->dim < 1 || fine->dim != xc->dim || fine->l != xc->l + 1 || fine->ebytes != xc->ebytes)
    return false;
  return full_grid(xc) || aligned(fine, xc);
}

int op_prolong(bfp_vec_s* xc, const WinParams& p, bfp_vec_s* out, cudaStream_t s, int ep,
               int gs) {
  if (!prolong_ok(xc, out)) return BFP_ERR_ARG;
  ProlongOp op;
  op.xc = view(xc);
  op.dim = out->dim;
  op.l = out->l;
  op.zf = out->z0;
  op.zp = out->z0 - 2 * xc->z0;
  op.ep = ep == kDefaultRep ? -out->dim : ep;
  op.gs = gs;
  if (gs) return launch_grid(op, out, p, s);
  static const int p3 = min_level("BFP_PRO3_MIN_L", 7), p2 = min_level("BFP_PRO2_MIN_L", 10);
  if (g_use_bulk && out->dim == 3 && out->l >= p3)
    return out->ebytes == 4 ? launch_pro3<int32_t>(op, out, p, s) : launch_pro3<int64_t>(op, out, p, s);
  if (g_use_bulk && out->dim == 2 && out->ebytes == 4 && out->l >= p2) return launch_pro2(op, out, p, s);
  return launch_grid(op, out, p, s);
}

int op_prolong_correct(bfp_vec_s* ec, bfp_vec_s* y, const WinParams& p, bfp_vec_s* out,
                       cudaStream_t s, int ep, int gs, Scal al, Scal be) {
  if (!prolong_ok(ec, y) || !same_grid(y, out)) return BFP_ERR_ARG;
  if (out == y) return BFP_ERR_ALIAS;
  ProlongCorrectOp op;
  op.ec = view(ec);
  op.y = view(y);
  op.dim = y->dim;
  op.l = y->l;
  op.zf = y->z0;
  op.zp = y->z0 - 2 * ec->z0;
  op.ep = ep == kDefaultRep ? -y->dim : ep;
  op.gs = gs;
  op.al = al;
  op.be = be;
  if (gs || al.m != 1 || be.m != 1) return launch_grid(op, out, p, s);
  static const int p3 = min_level("BFP_PRO3_MIN_L", 7), p2 = min_level("BFP_PRO2_MIN_L", 10);
  if (g_use_bulk && out->dim == 3 && out->l >= p3)
    return out->ebytes == 4 ? launch_pro3<int32_t>(op, out, p, s) : launch_pro3<int64_t>(op, out, p, s);
  if (g_use_bulk && out->dim == 2 && out->ebytes == 4 && out->l >= p2) return launch_pro2(op, out, p, s);
  return launch_grid(op, out, p, s);
}

}  // namespace bfp

#ifdef BFP_P3_TIMING
// measurement builds: per-phase clocks of block 0 / thread 0 of the pro3 marches (read + reset)
extern "C" int bfp_dbg_p3(long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_p3_prof, sizeof(long long) * 8);
  long long z[8] = {};
  cudaMemcpyToSymbol(g_p3_prof, z, sizeof(z));
  return 8;
}
#endif
