/*
 * bfpmg_b200.h -- C-ABI of the B200-native BFP multigrid hot path.
 *
 * Plain pointers, sizes and status codes; no torch or CUDA types in the
 * signatures (streams are passed as void* = cudaStream_t, 0 = default).
 * Every call is stream-ordered and asynchronous unless it says otherwise;
 * results that need the host (headers, flags, mantissas) come back through
 * the explicit *_download / *_header calls, which synchronise the stream.
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/proj):
 *   bfp_vec_*            BfpBlock / BfpBlock::vec / zero_vec / dump+parse    include/bfpmg/bfp.hpp:18-56, src/bfp.cpp:26-55,230-272
 *   bfp_normalize        normalize                                           src/bfp.cpp:97-108
 *   bfp_quantize         quantize                                            src/bfp.cpp:110-122
 *   bfp_inf_norm_upper   inf_norm_upper                                      src/bfp.cpp:124-148
 *   bfp_qaxpby / nnq     qaxpby / nnqaxpby (EaxpbyKernel + qcomp|nnqcomp)     src/blas.cpp:41-72,214-218,236-240
 *   bfp_qspmv_csr / nnq  qspmv / nnqspmv (EspmvKernel)                        src/blas.cpp:74-94,225-228,247-250
 *   bfp_qgemv_csr / nnq  qgemv / nnqgemv (EgemvKernel)                        src/blas.cpp:96-142,230-234,252-256
 *   bfp_qcomp_rows       qcomp/nnqcomp over a fixed exact-row ExactKernel    src/blas.cpp:144-212 (tests/test_blas.cpp:14-26)
 *   bfp_stencil_*        EgemvKernel/EspmvKernel with the FD stencil, R, P    src/blas.cpp:96-142
 *   bfp_mg_*             run_step / vcycle / ir / fmg                         src/multigrid.cpp:399-518
 */
#ifndef BFPMG_B200_H
#define BFPMG_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (the C++ facade maps them to the reference exceptions) ---- */
enum {
  BFP_OK = 0,
  BFP_ERR_ARG = 1,       /* std::invalid_argument: bad window, gamma <= 0, layout/dim mismatch */
  BFP_ERR_WIDTH = 2,     /* an exact row needs more than 127 bits (documented limit) */
  BFP_ERR_DOMAIN = 3,    /* std::domain_error: mantissa does not fit T_q */
  BFP_ERR_CUDA = 4,      /* CUDA runtime failure */
  BFP_ERR_ALIAS = 5,     /* output aliases an input */
  BFP_ERR_NOMEM = 6,
  BFP_ERR_STORAGE = 7    /* value does not fit the vector's mantissa storage (int32) */
};

/* ---- qcomp flags (QcompFlags, include/bfpmg/blas.hpp:98-102) ---- */
enum {
  BFP_FLAG_OVERFLOW = 1,
  BFP_FLAG_UNDERFLOW = 2,
  BFP_FLAG_RECOMPUTED = 4,
  BFP_FLAG_NORMALIZED = 8 /* produced by qcomp (1) or nnqcomp (0) */
};

typedef struct bfp_vec_s* bfp_vec_t;

/* host-visible header of a device block */
typedef struct {
  int64_t q;     /* mantissa width */
  int64_t e;     /* shared exponent: values are 2^e * m_i */
  int64_t n;     /* logical entries */
  int64_t max_abs;/* max |m_i| */
  int32_t flags; /* BFP_FLAG_* of the op that produced it */
  int32_t err;   /* sticky BFP_ERR_* raised on the device */
} bfp_header_t;

/* ---- device blocks ---- */
/* flat vector of n entries; mant_bytes 4 (int32) or 8 (int64) */
int bfp_vec_create(int64_t n, int mant_bytes, bfp_vec_t* out);
/* grid vector: dim 1..3, level l (n = (2^l - 1)^dim interior points, x fastest) */
int bfp_vec_create_grid(int dim, int level, int mant_bytes, bfp_vec_t* out);
int bfp_vec_destroy(bfp_vec_t v);
int64_t bfp_vec_size(bfp_vec_t v);
/* host mantissas (int64, logical order) -> device; sets q, e; checks fit T_q */
int bfp_vec_upload(bfp_vec_t v, const int64_t* m, int64_t q, int64_t e, void* stream);
/* same with int32 host mantissas (e2e path: no host-side widening) */
int bfp_vec_upload_i32(bfp_vec_t v, const int32_t* m, int64_t q, int64_t e, void* stream);
/* device -> host mantissas (pending shifts applied); synchronises the stream */
int bfp_vec_download(bfp_vec_t v, int64_t* m, bfp_header_t* hdr, void* stream);
int bfp_vec_download_i32(bfp_vec_t v, int32_t* m, bfp_header_t* hdr, void* stream);
/* stream-ordered download (gather + D2H into a pinned buffer), no synchronisation;
   read q/e afterwards with bfp_vec_header */
int bfp_vec_download_async_i32(bfp_vec_t v, int32_t* m, void* stream);
int bfp_vec_header(bfp_vec_t v, bfp_header_t* hdr, void* stream);
/* zero_vec(n, q): all zero, e = 0 (src/bfp.cpp:53-55) */
int bfp_vec_zero(bfp_vec_t v, int64_t q, void* stream);
/* dump_block text (src/bfp.cpp:230-241): writes at most cap bytes, returns needed size */
int64_t bfp_vec_dump(bfp_vec_t v, char* buf, int64_t cap, void* stream);
/* parse_block text into a flat int64 vector (src/bfp.cpp:243-272) */
int bfp_vec_parse(const char* text, bfp_vec_t* out, void* stream);

/* ---- BFP block operations ---- */
int bfp_normalize(bfp_vec_t x, bfp_vec_t out, void* stream);
int bfp_quantize(bfp_vec_t x, int64_t w, bfp_vec_t out, void* stream);
/* synchronous: scalar (m, q, e) >= max|x| rounded up to q_gamma bits */
int bfp_inf_norm_upper(bfp_vec_t x, int64_t q_gamma, int64_t* m, int64_t* q, int64_t* e,
                       void* stream);
/* ---- exact dot product <x, y> = sum_i m_x,i m_y,i 2^(e_x + e_y) (no
 * reference function).  Accumulated exactly in 192 bits on the device; the device result
 * is int64 acc[5] = {L0, L1, L2, L3, e} with value sum_k L_k 2^(48 k) (limb sums, not
 * carried), e = e_x + e_y.
 *   bfp_dot_exact_async  stream-ordered into a caller device buffer (memset + one kernel:
 *                        no allocation, no synchronisation, graph-capturable)
 *   bfp_dot_value        host: limbs -> the exact 192-bit two's complement words[3]
 *                        (little endian) and its low 128 bits; BFP_ERR_WIDTH when the value
 *                        does not fit 128 bits (sticky overflow detection)
 *   bfp_dot_exact        synchronous, 128-bit (hi, lo); BFP_ERR_WIDTH beyond 128 bits
 *   bfp_dot_exact192     synchronous, the full 192-bit value
 * The synchronous calls reuse an accumulator owned by x (calls sharing x must not
 * overlap on different streams). */
int bfp_dot_exact_async(bfp_vec_t x, bfp_vec_t y, int64_t* d_acc, void* stream);
int bfp_dot_value(const int64_t* acc, uint64_t* words, int64_t* hi, uint64_t* lo);
int bfp_dot_exact(bfp_vec_t x, bfp_vec_t y, int64_t* hi, uint64_t* lo, int64_t* e, void* stream);
int bfp_dot_exact192(bfp_vec_t x, bfp_vec_t y, uint64_t* words, int64_t* e, void* stream);

/* ---- windowed BLAS (qcomp: w_tmp >= w_out; nnqcomp: w_tmp ignored) ----
 * Scalars are BFP scalars (m, q, e); gamma = (gm, gq, ge) with gm > 0.
 * mode: 0 = qcomp, 1 = nnqcomp.  force_recompute: QcompOptions test hook. */
typedef struct {
  int64_t m, q, e;
} bfp_scalar_t;

/* a positive extended-precision constant: (hi 2^64 + lo) 2^e, plus a nonzero tail below
   lo when sticky != 0 (the top 128 bits of an ExtFloat) */
typedef struct {
  uint64_t hi, lo;
  int64_t e;
  int32_t sticky, pad;
} bfp_xf_t;

int bfp_axpby(bfp_vec_t x, bfp_vec_t y, bfp_scalar_t alpha, bfp_scalar_t beta, int mode,
              int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma, int force_recompute,
              bfp_vec_t out, void* stream);

/* CSR matrix (int64 rowptr/col/mantissas, host pointers copied to the device) */
typedef struct bfp_csr_s* bfp_csr_t;
int bfp_csr_create(int64_t rows, int64_t cols, const int64_t* rowptr, const int64_t* col,
                   const int64_t* m, int64_t q, int64_t e, bfp_csr_t* out);
int bfp_csr_destroy(bfp_csr_t a);
int bfp_spmv_csr(bfp_csr_t a, bfp_vec_t x, int64_t m_a, int mode, int64_t w_out, int64_t w_tmp,
                 bfp_scalar_t gamma, int force_recompute, bfp_vec_t out, void* stream);
int bfp_gemv_csr(bfp_csr_t a, bfp_vec_t x, bfp_vec_t y, bfp_scalar_t alpha, bfp_scalar_t beta,
                 int64_t m_a, int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                 int force_recompute, bfp_vec_t out, void* stream);
/* exact rows given as 128-bit (hi, lo) at template (q, e): the FixedKernel hook */
int bfp_qcomp_rows(int64_t n, const int64_t* hi, const uint64_t* lo, int64_t q, int64_t e,
                   int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                   int force_recompute, bfp_vec_t out, void* stream);

/* ---- stencil family on grid vectors ---- */
/* z = alpha*(A_l x) + beta*y ; A_l = 2^{2l} S_d (residual: alpha=-1, beta=+1) */
int bfp_stencil_gemv(bfp_vec_t x, bfp_vec_t y, bfp_scalar_t alpha, bfp_scalar_t beta, int mode,
                     int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma, int force_recompute,
                     bfp_vec_t out, void* stream);
/* z = x + c*(b - A_l x)   (fused weighted-Jacobi sweep) */
int bfp_stencil_jacobi(bfp_vec_t x, bfp_vec_t b, bfp_scalar_t c, int mode, int64_t w_out,
                       int64_t w_tmp, bfp_scalar_t gamma, bfp_vec_t out, void* stream);
/* z = c*r */
int bfp_scal(bfp_vec_t r, bfp_scalar_t c, int mode, int64_t w_out, int64_t w_tmp,
             bfp_scalar_t gamma, bfp_vec_t out, void* stream);
/* coarse z = R r (full weighting) ; fine z = P xc ; fine z = P ec + y */
int bfp_restrict_fw(bfp_vec_t r, int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                    bfp_vec_t out, void* stream);
int bfp_prolong(bfp_vec_t xc, int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                bfp_vec_t out, void* stream);
int bfp_prolong_correct(bfp_vec_t ec, bfp_vec_t y, int mode, int64_t w_out, int64_t w_tmp,
                        bfp_scalar_t gamma, bfp_vec_t out, void* stream);
/* ---- multi-rank z-slab decomposition ----
 * A slab holds planes [z_lo, z_hi) of the padded global grid along the slowest axis
 * (2-D rows, 3-D planes) plus one halo plane on each side.  Stencil ops on slabs run
 * in two stages per window: stage 0 (qcomp pass 1 / nnqcomp) and stage 1 (qcomp
 * recompute, a no-op unless the finalized header asks for it).  Each stage writes its
 * partials {mu*, max, -min, err} (int64[4], device) to d_part; after an all-reduce(MAX)
 * of d_part over the ranks, bfp_window_finalize applies them to the header exactly as
 * the single-rank finalizer does. */
int bfp_vec_create_slab(int dim, int level, int z_lo, int z_hi, int mant_bytes, bfp_vec_t* out);
/* device pointers: first / last owned plane and the lower / upper halo planes */
int bfp_vec_planes(bfp_vec_t v, void** first, void** last, void** halo_lo, void** halo_hi,
                   int64_t* plane_bytes);
int bfp_stencil_gemv_part(bfp_vec_t x, bfp_vec_t y, bfp_scalar_t alpha, bfp_scalar_t beta,
                          int mode, int stage, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                          bfp_vec_t out, int64_t* d_part, void* stream);
int bfp_stencil_jacobi_part(bfp_vec_t x, bfp_vec_t b, bfp_scalar_t c, int mode, int stage,
                            int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma, bfp_vec_t out,
                            int64_t* d_part, void* stream);
int bfp_window_finalize(bfp_vec_t out, int mode, int stage, int64_t w_out, int64_t w_tmp,
                        const int64_t* d_part, void* stream);

/* quantize_exact (P/src/bfp.cpp:163-187): entries z_i * 2^k_i (host arrays of the
   vector's logical size) -> m_i = floor(z_i 2^(k_i - e)), e = max(msb z_i + k_i) - w,
   q = w; all-zero input -> e = 0.  bfp_from_doubles is from_extfloat
   (P/src/bfp.cpp:189-194) for IEEE doubles (non-finite -> BFP_ERR_ARG). */
int bfp_quantize_exact(const int64_t* z, const int64_t* k, int64_t n, int64_t w, bfp_vec_t out,
                       void* stream);
int bfp_from_doubles(const double* v, int64_t n, int64_t w, bfp_vec_t out, void* stream);

/* Jacobi coefficient c = floor_qc(omega_d / 2d) * 2^{-2l} as a BFP scalar */
int bfp_jacobi_coeff(int dim, int level, int64_t qc, bfp_scalar_t* c);

/* ---- generators ---- */
int bfp_gen_uniform(bfp_vec_t v, int64_t p, uint64_t seed, uint64_t stream_id, void* stream);
int bfp_gen_sine(bfp_vec_t v, int64_t p, void* stream);

/* ---- multigrid solver ---- */
/* nonnormalized = NormMode (P/src/multigrid.cpp:403-409): 0 normalized (qcomp),
   1 nonnormalized (nnqcomp except the diagnostic final residual), 2 hybrid (qcomp only
   for the IR residual of iterations <= 2, hybrid_qcomp_iters).
   PrecisionSchedule (P/include/bfpmg/multigrid.hpp:16-27) per level: p = w (iterate),
   pd = wdot (residual and V-cycle), pc = wcheck (right-hand side); 0 entries = p.
   w_add_cap: GammaPolicy::w_add_cap (-1 unlimited).
   x0_random (IR runs): 0 zero_vec, 1 seeded uniform, 2 the caller's iterate (written into
   the x handle of bfp_mg_vectors before each solve; single rank). */
typedef struct {
  int d, l_fine, l_coarse, nu1, nu2, n_coarse, cycles, fmg, nonnormalized, x0_random, rhs_kind,
      qc;
  uint64_t seed;
  int p[32];
  int pd[32];
  int pc[32];
  int w_add_cap;
  /* levels whose padded grid has <= fuse_points points run as one fused CTA with their
     vectors staged in shared memory; 0 = off, -1 = library default */
  int fuse_points;
  /* reference-algorithm mode (P/src/multigrid.cpp:430-518), d = 1 or 2:
     Chebyshev V(1,0) cycles, IR (r = A x - b, x - y) and FMG (fresh ir per n_ir, level 1
     = zero_vec) on the reference's p = 1 operators after the D = I scaling
     (P/src/multigrid.cpp:277-306): 1-D A = tridiag(-1/2, 1, -1/2), P = linear
     interpolation, R = 2 P^T; 2-D (P/src/fem.cpp:426-457, 542-543) A = 9-point
     (1, -1/8 x 8), P = P1 (x) P1, R = P^T.  Operators quantize_csr'd at wcheck / wdot / w
     (every width >= 3 in 1-D, >= 5 in 2-D), coarsest level 1, gamma = Table 1
     (gamma_policy_eval, :121-155) evaluated exactly with one final round-up.  The host
     supplies the derived Chebyshev scalars: ref_c1 = c1 rounded to the hierarchy
     precision (ExtFloat), ref_kres = add_up(2 c1, 1) / 4, ref_c1d / ref_c2d[l] = c1 / c2
     floor-quantised at wdot_l (quantize_scalar_floor); rhs_kind 1 = h^2 / 2^d * the
     config's d pi^2 prod sin (the D^-1-scaled load up to a constant); rhs_kind 3 = the
     caller's vectors (bfp_mg_level_rhs), e.g. the FEM load by quadrature. */
  int ref_mode;
  bfp_xf_t ref_c1, ref_kres;
  bfp_scalar_t ref_c1d[32], ref_c2d[32];
} bfp_mg_config_t;

typedef struct {
  int32_t step, level, w_out, w_tmp;
  int64_t gm, ge;
  int32_t overflow, underflow, recomputed, normalized;
} bfp_trace_rec_t;

typedef struct bfp_mg_s* bfp_mg_t;
int bfp_mg_create(const bfp_mg_config_t* cfg, bfp_mg_t* out);
int bfp_mg_destroy(bfp_mg_t mg);
/* full solve on the device; use_graph != 0 replays a captured CUDA graph */
int bfp_mg_solve(bfp_mg_t mg, int use_graph, void* stream);
/* results (synchronise): finest-level iterate, residual history, trace */
int bfp_mg_result(bfp_mg_t mg, int64_t* x, bfp_header_t* xh, double* hist, int hist_cap,
                  int* n_hist, bfp_trace_rec_t* trace, int64_t trace_cap, int64_t* n_trace,
                  void* stream);
/* handles to the solver's finest-level vectors (x, b) for benchmarks */
int bfp_mg_vectors(bfp_mg_t mg, bfp_vec_t* x, bfp_vec_t* b, bfp_vec_t* r);
/* rhs_kind 3 (caller-provided right-hand sides; the reference's hierarchy keeps one D^-1-scaled
   FEM load vector per level, Hierarchy::setup_scaling, P/src/multigrid.cpp:286-289): the
   handle of level `level`'s b (FMG: every level; otherwise the finest) and its mantissa
   bytes.  The solver zero-initialises it at create; the caller writes it (bfp_quantize_exact,
   bfp_vec_upload, ...) before a solve.  Single-rank solvers only. */
int bfp_mg_level_rhs(bfp_mg_t mg, int level, bfp_vec_t* b, int* mant_bytes);
int64_t bfp_mg_kernel_launches(bfp_mg_t mg);

/* ---- sharded solve ----
 * Levels with >= min_planes planes per rank along the slowest axis (d >= 2) are
 * slabs of 2^l / world planes; coarser levels are replicated on every rank.
 * nccl_id = NULL: an in-process group of `world` ranks on the current device
 * (bit-exact stand-in for the transport, tests); otherwise this process is `rank`
 * of an NCCL communicator created from a unique id made by bfp_nccl_unique_id on
 * one rank and broadcast by the caller (the current CUDA device must be set). */
int bfp_nccl_unique_id(void* id, int id_bytes);
int bfp_mg_create_sharded(const bfp_mg_config_t* cfg, int world, int rank, const void* nccl_id,
                          int min_planes, bfp_mg_t* out);
/* per local rank: the final iterate / residual (slabs on sharded levels), global rank and
   the lowest sharded level (64: none) */
/* Transport of the per-op exponent all-reduce of sharded solves created AFTER the call
 * (DESIGN.md section 9): 0 = default (NCCL groups: peer-memory mailboxes over CUDA IPC when
 * they can be mapped, else ncclAllReduce; in-process groups: one reduction kernel),
 * 1 = mailboxes for in-process groups too (the protocol's test path), 2 = never mailboxes.
 * bfp_mg_transport reports what a solver uses: 0 local kernel, 1 mailboxes, 2 ncclAllReduce. */
int bfp_set_transport(int transport);
int bfp_mg_transport(bfp_mg_t mg);
int bfp_mg_rank_result(bfp_mg_t mg, int local_rank, bfp_vec_t* x_final, bfp_vec_t* r_final,
                       int* rank, int* lowest_sharded_level);

/* sharded single stencil ops (a fine-level residual / Jacobi sweep over z-slabs):
 * halo exchange, pass 1 with partial windows, MAX all-reduce of {mu*, max, -min, err},
 * finalize (+ the recompute pass) -- all stream-ordered, no host synchronisation.
 * The vector arguments are arrays of one slab handle per local rank (world for an
 * in-process group, 1 with NCCL). */
typedef struct bfp_dist_s* bfp_dist_t;
int bfp_dist_create(int world, int rank, const void* nccl_id, bfp_dist_t* out);
int bfp_dist_destroy(bfp_dist_t d);
int bfp_dist_stencil_gemv(bfp_dist_t d, bfp_vec_t const* x, bfp_vec_t const* y,
                          bfp_scalar_t alpha, bfp_scalar_t beta, int mode, int64_t w_out,
                          int64_t w_tmp, bfp_scalar_t gamma, bfp_vec_t const* out, void* stream);
int bfp_dist_stencil_jacobi(bfp_dist_t d, bfp_vec_t const* x, bfp_vec_t const* b, bfp_scalar_t c,
                            int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                            bfp_vec_t const* out, void* stream);

/* sharded exact dot over z-slabs: per-rank limb accumulators (device int64[5] each, one
 * per local rank), carried into [0, 2^48) per rank and all-reduced with an int64 SUM
 * (every rank ends with the global limbs; exact for up to 2^14 ranks); stream-ordered */
int bfp_dist_dot_exact(bfp_dist_t d, bfp_vec_t const* x, bfp_vec_t const* y,
                       int64_t* const* d_acc, void* stream);

/* ---- measurement hooks ----
 * When enabled, every windowed pass-1 / nnqcomp kernel launch is bracketed by
 * CUDA events recorded on its own stream; read() synchronises and returns the
 * summed device time and the launch count since the last reset. */
int bfp_profile_enable(int on);
int bfp_profile_read(double* total_ms, int64_t* count, int reset);
/* kernel-path switches (bit-identical results; for A/B measurement and tests):
   bit 0: 2-D stencil via the bulk-async shared-memory pipeline (1, default) or the
          register march (0); bit 1: disable programmatic dependent launch;
   bit 2: skip the qcomp recompute launch (pass-1 timing only; flags must be clear) */
int bfp_set_kernel_path(int bulk);

/* ---- misc ---- */
const char* bfp_status_string(int status);
int bfp_device_sync(void* stream);
/* number of kernels this library launched since load (evidence counter) */
int64_t bfp_launch_count(void);
/* windowed-kernel launches since load per kernel family (evidence of the pipelines a solve
   used; launches recorded while capturing a solve graph count once):
   0 grid, 1 2-D bulk pipeline, 2 3-D tiled-TMA pipeline, 3 register march, 4 3-D
   prolongation march, 5 3-D restriction march, 6 2-D prolongation march, 7 2-D restriction
   march, 8 flat rows, 9 fused single-CTA, 10 persistent coarse-level kernel */
int bfp_kernel_family_counts(int64_t* counts, int n);

#ifdef __cplusplus
}
#endif
#endif
