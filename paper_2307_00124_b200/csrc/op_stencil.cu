// op_stencil.cu -- stencil ops (residual / gemv, fused Jacobi): instantiates the
// bulk-async, register-march and generic grid kernels for GemvOp / JacobiOp.
#include "bfp_kernels.cuh"

namespace bfp {

int op_gemv(bfp_vec_s* x, bfp_vec_s* y, Scal al, Scal be, const WinParams& p, bfp_vec_s* out,
            cudaStream_t s, int ea, int gs, int st9) {
  if (x->dim < 1 || !same_grid(x, y) || !same_grid(x, out)) return BFP_ERR_ARG;
  if (st9 && x->dim != 2) return BFP_ERR_ARG;
  if (out == x || out == y) return BFP_ERR_ALIAS;
  GemvOp op;
  op.x = view(x);
  op.y = view(y);
  op.al = al;
  op.be = be;
  op.dim = x->dim;
  op.l = x->l;
  op.z0 = x->z0;
  op.ea = ea == kDefaultRep ? 2 * x->l : ea;
  op.gs = gs;
  op.st9 = st9;
  if (gs || st9) return launch_grid(op, out, p, s);  // scaled mantissas / 9-point: generic path
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


}  // namespace bfp
