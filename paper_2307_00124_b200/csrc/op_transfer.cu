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

}  // namespace bfp
