/*
 * bfp_oracle.h -- CPU restatement of the reference BFP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product (paper_2307_00124_b200/) never links or calls it.
 *
 * It restates, with int64 mantissa storage and __int128 exact rows (the
 * reference uses GMP mpz; GMP headers/libgmpxx are absent here so the
 * reference itself is unbuildable):
 *   msb / shift_floor / truncate_to_width / clamp   P/src/wideint.cpp:15-25,74-79,94-107
 *   normalize / quantize / inf_norm_upper           P/src/bfp.cpp:97-148
 *   quantize_exact                                  P/src/bfp.cpp:163-187
 *   EaxpbyKernel / EspmvKernel / EgemvKernel        P/src/blas.cpp:41-142
 *   qcomp / nnqcomp                                 P/src/blas.cpp:144-212
 * plus the frozen config-driver ops and drivers of DESIGN.md section 3
 * (stencil gemv, fused weighted Jacobi, full-weighting restriction, linear
 * prolongation, IR / V-cycle / FMG), composed from those primitives exactly
 * as P/src/multigrid.cpp:399-518 composes its ExactKernels.
 *
 * Parity pin: the known answers of P/tests/test_{wideint,bfp,blas}.cpp and
 * a Python big-int restatement (oracle/pyref.py) -- see tests/.
 * Any result that would need more than 127 bits returns OB_ERR_WIDTH.
 */
#ifndef BFP_ORACLE_H
#define BFP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef __int128 ob_i128;

enum { OB_OK = 0, OB_ERR_ARG = 1, OB_ERR_WIDTH = 2, OB_ERR_GAMMA = 3, OB_ERR_DIM = 4 };

/* ---- scalar primitives (P/src/wideint.cpp) ---- */
int64_t ob_msb64(int64_t v);
int64_t ob_shift_floor64(int64_t x, int64_t s, int* ovf);
int64_t ob_wrap64(int64_t x, int64_t w);
/* 128-bit variants used internally; exported for tests via hi/lo pairs */
int64_t ob_msb128(int64_t hi, uint64_t lo);

/* ---- BFP block (P/include/bfpmg/bfp.hpp:18-56) : n int64 mantissas ---- */
typedef struct {
  int64_t n, q, e;
  int64_t* m;
} ob_block;

/* normalize / quantize in place-to-out (out->m may alias x->m) */
int ob_normalize(const ob_block* x, ob_block* out);
int ob_quantize(const ob_block* x, int64_t w, ob_block* out);
/* inf_norm_upper: returns scalar (m,q,e) */
int ob_inf_norm_upper(const ob_block* x, int64_t q_gamma, int64_t* m, int64_t* q, int64_t* e);

/* ---- exact kernels (P/include/bfpmg/blas.hpp:25-96) ---- */
typedef struct ob_kernel {
  int64_t q, e; /* ExactTemplate */
  int64_t n;
  int (*row)(const struct ob_kernel* k, int64_t i, ob_i128* out);
  const void* a; /* kernel specific state */
  int64_t p[24];
  const int64_t* ptr[8];
  int64_t zd; /* e - e_ref >= 0: rows are the reference rows / 2^zd (axpby_setup_z) */
} ob_kernel;

typedef struct {
  int overflow, underflow, recomputed;
} ob_flags;

/* qcomp / nnqcomp (P/src/blas.cpp:144-212).  gamma = (gm, ge), gm > 0. */
int ob_qcomp(const ob_kernel* k, int64_t w_out, int64_t w_tmp, int64_t gm, int64_t ge,
             int force_recompute, ob_block* out, ob_flags* flags);
int ob_nnqcomp(const ob_kernel* k, int64_t w_out, int64_t gm, int64_t ge, ob_block* out);

/* kernel builders over flat blocks.  Scalars are (m, q, e). */
int ob_make_axpby(ob_kernel* k, const ob_block* x, const ob_block* y, int64_t am, int64_t aq,
                  int64_t ae, int64_t bm, int64_t bq, int64_t be);
/* CSR (int64 rowptr/col/mantissas, q_A, e_A), m_a = declared row bound (0 = exact) */
typedef struct {
  int64_t rows, cols, q, e, max_row_nnz;
  const int64_t *rowptr, *col, *m;
} ob_csr;
int ob_make_spmv(ob_kernel* k, const ob_csr* a, const ob_block* x, int64_t m_a);
int ob_make_gemv(ob_kernel* k, const ob_csr* a, const ob_block* x, const ob_block* y, int64_t am,
                 int64_t aq, int64_t ae, int64_t bm, int64_t bq, int64_t be, int64_t m_a);
/* explicit exact rows (the test FixedKernel, P/tests/test_blas.cpp:14-26), rows as hi/lo */
int ob_make_rows(ob_kernel* k, int64_t n, const int64_t* hi, const uint64_t* lo, int64_t q,
                 int64_t e);
/* evaluate one row of any kernel (tests) */
int ob_kernel_row(const ob_kernel* k, int64_t i, int64_t* hi, uint64_t* lo);

/* ---- grid operators (frozen config semantics) ----
 * A grid vector of dimension d at level l has n = 2^l - 1 interior points per
 * axis, x fastest, interior only (Dirichlet 0 outside).                      */
typedef struct {
  int d, l;
} ob_grid;
int64_t ob_grid_n(ob_grid g);   /* points per axis */
int64_t ob_grid_size(ob_grid g); /* n^d */

/* stencil A_l = 2^{2l} * S_d (S: centre 2d, neighbours -1), q_A, e_A, m_A */
void ob_stencil_desc(ob_grid g, int64_t* qa, int64_t* ea, int64_t* ma);
/* z = alpha*(A x) + beta*y   (EgemvKernel with A = stencil) */
int ob_make_stencil_gemv(ob_kernel* k, ob_grid g, const ob_block* x, const ob_block* y,
                         int64_t am, int64_t aq, int64_t ae, int64_t bm, int64_t bq, int64_t be);
/* z = x + c*(b - A x)   (fused weighted Jacobi, composed egemv + eaxpby) */
int ob_make_jacobi(ob_kernel* k, ob_grid g, const ob_block* x, const ob_block* b, int64_t cm,
                   int64_t cq, int64_t ce);
/* z = c*r  (first sweep from a zero iterate) */
int ob_make_scal(ob_kernel* k, const ob_block* r, int64_t cm, int64_t cq, int64_t ce);
/* coarse z = R r  (full weighting, espmv) ; g = fine grid */
int ob_make_restrict(ob_kernel* k, ob_grid gf, const ob_block* r);
/* fine z = P xc (espmv)  ; gf = fine grid */
int ob_make_prolong(ob_kernel* k, ob_grid gf, const ob_block* xc);
/* fine z = P ec + y  (egemv with alpha = beta = bfp_one) */
int ob_make_prolong_correct(ob_kernel* k, ob_grid gf, const ob_block* ec, const ob_block* y);
/* Jacobi coefficient c = floor_q(omega_d/(2d)) * 2^{-2l} */
void ob_jacobi_coeff(ob_grid g, int64_t qc, int64_t* cm, int64_t* ce);

/* ---- gamma arithmetic: 15-bit round-up values ---- */
typedef struct {
  int64_t m, e; /* m in [2^14, 2^15) or m == 0 */
} ob_g15;
ob_g15 ob_g15_norm(const ob_block* x, int64_t pending_shift_unused);
ob_g15 ob_g15_from(uint64_t mag, int64_t e);
ob_g15 ob_g15_mul(ob_g15 a, ob_g15 b);
ob_g15 ob_g15_add(ob_g15 a, ob_g15 b);
void ob_g15_gamma(ob_g15 g, int64_t* gm, int64_t* ge); /* degenerate 2^-400 if zero */

/* ---- generators ---- */
uint64_t ob_splitmix64(uint64_t x);
/* m_i uniform in T_p at e = -(p-1), then normalize */
int ob_gen_uniform(ob_grid g, int64_t p, uint64_t seed, uint64_t stream, ob_block* out);
/* f = d*pi^2 * prod sin(pi x_a), quantize_exact floor at p bits */
int ob_gen_sine(ob_grid g, int64_t p, ob_block* out);

/* ---- multigrid driver ---- */
enum { OB_STEP_IR_RES = 0, OB_STEP_IR_CORR, OB_STEP_RELAX0, OB_STEP_RELAX, OB_STEP_V_RES,
       OB_STEP_RESTRICT, OB_STEP_V_CORR, OB_STEP_FMG_PROLONG, OB_STEP_FINAL_RES, OB_STEP_COUNT };
typedef struct {
  int32_t step, level, w_out, w_tmp;
  int64_t gm, ge;
  int32_t overflow, underflow, recomputed, normalized;
} ob_trace_rec;

typedef struct {
  int d;            /* 1,2,3 */
  int l_fine;       /* finest level */
  int l_coarse;     /* coarsest level */
  int nu1, nu2;     /* pre/post sweeps */
  int n_coarse;     /* sweeps on the coarsest level */
  int cycles;       /* IR iterations (mode 0) or IR steps per FMG level (mode 1) */
  int fmg;          /* 0: IR-V cycles at fine level, 1: FMG */
  int nonnormalized;/* 1: nnqcomp everywhere except the diagnostic final residual;
                       2: hybrid, qcomp only for the IR residual of iterations <= 2 */
  int x0_random;    /* 1: x0 uniform (seed, stream 1); 0: zero_vec */
  int rhs_kind;     /* 0: uniform (seed, stream 2); 1: sine; 2: zero */
  int qc;           /* width of the Jacobi coefficient */
  uint64_t seed;
  int p[32];        /* w: iterate width per level (index = level) */
  int pd[32];       /* wdot: residual / V-cycle width (0 = p) */
  int pc[32];       /* wcheck: right-hand-side width (0 = p) */
  int w_add_cap;    /* GammaPolicy::w_add_cap: -1 unlimited */
} ob_mg_config;

typedef struct {
  ob_block x;             /* final iterate at the finest level (caller allocates m) */
  double* res_history;    /* capacity >= cycles*levels + 2 */
  int n_history;
  ob_trace_rec* trace;    /* capacity trace_cap */
  int64_t trace_cap, n_trace;
  int err;
} ob_mg_result;

int ob_mg_run(const ob_mg_config* cfg, ob_mg_result* res);

/* ---- CPU baseline: the fine-level residual r = b - A x in qcomp mode, OpenMP ---- */
int ob_residual_qcomp_omp(ob_grid g, const ob_block* x, const ob_block* b, int64_t w_out,
                          int64_t w_tmp, int64_t gm, int64_t ge, ob_block* out, ob_flags* fl,
                          int threads);

#ifdef __cplusplus
}
#endif
#endif
