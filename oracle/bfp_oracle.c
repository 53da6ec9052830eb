/*
 * bfp_oracle.c -- CPU restatement of the reference BFP hot path.
 * TEST INFRASTRUCTURE ONLY (see bfp_oracle.h).  Never linked by the product.
 *
 * Every function cites the reference file:line it restates.  Rows are exact
 * __int128 values computed with overflow-checked arithmetic; a row that would
 * leave 128 bits yields OB_ERR_WIDTH instead of a wrong answer.
 */
#include "bfp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;
typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* scalar primitives                                                         */

static inline int64_t bitlen_u128(u128 u) {
  uint64_t hi = (uint64_t)(u >> 64), lo = (uint64_t)u;
  if (hi) return 128 - __builtin_clzll(hi);
  if (lo) return 64 - __builtin_clzll(lo);
  return 0;
}

/* msb: minimal w >= 1 with v in T_w.  P/src/wideint.cpp:15-25 */
static inline int64_t msb128(i128 v) {
  u128 u = (u128)(v ^ (v >> 127)); /* v for v >= 0, -v-1 for v < 0 */
  return bitlen_u128(u) + 1;
}

int64_t ob_msb64(int64_t v) { return msb128((i128)v); }
int64_t ob_msb128(int64_t hi, uint64_t lo) { return msb128((i128)(((u128)(uint64_t)hi << 64) | lo)); }

/* floor(x / 2^s); s < 0 is an exact left shift.  P/src/wideint.cpp:94-100 */
static inline int shift_floor128(i128 x, int64_t s, i128* out) {
  if (s >= 0) {
    *out = s >= 127 ? (x < 0 ? -1 : 0) : (x >> s);
    return 0;
  }
  int64_t k = -s;
  if (x == 0) {
    *out = 0;
    return 0;
  }
  if (msb128(x) + k > 128) return 1; /* would leave 128 bits */
  *out = (i128)((u128)x << k);
  return 0;
}

/* low w bits reinterpreted as two's complement.  P/src/wideint.cpp:102-107 */
static inline i128 wrap128(i128 x, int64_t w) {
  if (w >= 128) return x;
  return (i128)((u128)x << (128 - w)) >> (128 - w);
}

/* wrap_w(floor(x / 2^s)) without intermediate overflow (the low w bits of
 * x*2^k only depend on x mod 2^(w-k)). */
static inline i128 wrap_shift128(i128 x, int64_t s, int64_t w) {
  if (s >= 0) return wrap128(s >= 127 ? (x < 0 ? -1 : 0) : (x >> s), w);
  int64_t k = -s;
  if (k >= w) return 0;
  return wrap128((i128)((u128)x << k), w);
}

/* clamp to T_w.  P/src/wideint.cpp:74-79, inline form P/src/blas.cpp:196-209 */
static inline i128 clamp_w(i128 x, int64_t w) {
  if (w >= 128) return x;
  i128 hi = (((i128)1) << (w - 1)) - 1, lo = -(((i128)1) << (w - 1));
  return x > hi ? hi : (x < lo ? lo : x);
}

int64_t ob_shift_floor64(int64_t x, int64_t s, int* ovf) {
  i128 r = 0;
  int o = shift_floor128(x, s, &r);
  if (!o && (r > INT64_MAX || r < INT64_MIN)) o = 1;
  if (ovf) *ovf = o;
  return (int64_t)r;
}
int64_t ob_wrap64(int64_t x, int64_t w) { return (int64_t)wrap128(x, w); }

static inline int mul_chk(i128 a, i128 b, i128* r) { return __builtin_mul_overflow(a, b, r); }
static inline int add_chk(i128 a, i128 b, i128* r) { return __builtin_add_overflow(a, b, r); }
static inline int shl_chk(i128 a, int64_t k, i128* r) { /* k >= 0 */
  if (a == 0 || k == 0) {
    *r = a;
    return 0;
  }
  if (msb128(a) + k > 128) return 1;
  *r = (i128)((u128)a << k);
  return 0;
}

static inline int64_t ceil_log2(int64_t m) { /* P/src/blas.cpp:11-19 */
  int64_t r = 0, v = 1;
  while (v < m) {
    v <<= 1;
    ++r;
  }
  return r;
}
static inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
static inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* ------------------------------------------------------------------------ */
/* blocks: P/src/bfp.cpp                                                     */

static int64_t max_msb_block(const ob_block* x) { /* P/src/bfp.cpp:17-22 (0 if all zero) */
  int64_t mu = 0;
  for (int64_t i = 0; i < x->n; ++i)
    if (x->m[i] != 0) mu = max64(mu, msb128(x->m[i]));
  return mu;
}

int ob_normalize(const ob_block* x, ob_block* out) { /* P/src/bfp.cpp:97-108 */
  int64_t mu = max_msb_block(x);
  out->n = x->n;
  out->q = x->q;
  if (mu == 0) {
    if (out->m != x->m) memcpy(out->m, x->m, sizeof(int64_t) * x->n);
    out->e = 0;
    return OB_OK;
  }
  int64_t shift = x->q - mu;
  for (int64_t i = 0; i < x->n; ++i) {
    i128 r = 0;
    if (shift_floor128(x->m[i], -shift, &r) || r > INT64_MAX || r < INT64_MIN) return OB_ERR_WIDTH;
    out->m[i] = (int64_t)r;
  }
  out->e = x->e - shift;
  return OB_OK;
}

int ob_quantize(const ob_block* x, int64_t w, ob_block* out) { /* P/src/bfp.cpp:110-122 */
  if (w < 1) return OB_ERR_ARG;
  int64_t mu = max_msb_block(x);
  out->n = x->n;
  out->q = w;
  if (mu == 0) {
    if (out->m != x->m) memcpy(out->m, x->m, sizeof(int64_t) * x->n);
    out->e = 0;
    return OB_OK;
  }
  int64_t s = mu - w;
  for (int64_t i = 0; i < x->n; ++i) {
    i128 r = 0;
    if (shift_floor128(x->m[i], s, &r) || r > INT64_MAX || r < INT64_MIN) return OB_ERR_WIDTH;
    out->m[i] = (int64_t)r;
  }
  out->e = x->e + s;
  return OB_OK;
}

int ob_inf_norm_upper(const ob_block* x, int64_t q_gamma, int64_t* m, int64_t* q, int64_t* e) {
  /* P/src/bfp.cpp:124-148 */
  if (q_gamma < 2 || q_gamma > 62) return OB_ERR_ARG;
  u128 mx = 0;
  for (int64_t i = 0; i < x->n; ++i) {
    i128 v = x->m[i];
    u128 a = (u128)(v < 0 ? -v : v);
    if (a > mx) mx = a;
  }
  *q = q_gamma;
  if (mx == 0) {
    *m = (int64_t)1 << (q_gamma - 2);
    *e = x->e - (q_gamma - 2);
    return OB_OK;
  }
  int64_t s = msb128((i128)mx) - q_gamma;
  u128 mm;
  if (s <= 0) {
    mm = mx << (-s);
  } else {
    mm = (mx + (((u128)1 << s) - 1)) >> s; /* mpz_cdiv_q_2exp for positive */
    if (msb128((i128)mm) > q_gamma) {
      mm >>= 1;
      ++s;
    }
  }
  *m = (int64_t)mm;
  *e = x->e + s;
  return OB_OK;
}

/* ------------------------------------------------------------------------ */
/* exact kernels: P/src/blas.cpp:41-142                                      */

/* eaxpby setup on (qa, ea) (qb, eb): P/src/blas.cpp:46-58 / 112-119 */
static void axpby_setup(int64_t qa, int64_t ea, int64_t qb, int64_t eb, int64_t* d, int64_t* q,
                        int64_t* e) {
  *d = ea - eb;
  *q = (*d < 0) ? max64(qa, qb - *d) + 1 : max64(qb, qa + *d) + 1;
  *e = min64(ea, eb);
}

/* The same with all-zero terms dropped (za / zb: the term is zero on every row).  When
 * exactly one term is zero its alignment shift goes too: d = 0, e* = the other term's
 * exponent, and *zd grows by e* - min(ea, eb).  Every row is then the reference row
 * / 2^zd exactly, so qcomp/nnqcomp windows are unchanged; only qcomp's all-zero anchor
 * (mu* = 1, P/src/blas.cpp:153) needs zd.  This keeps rows within 127 bits where a zero
 * block at e = 0 meets a far-away operand (b = 0 and a diverging iterate, C5 p = 4);
 * the reference's mpz rows are merely long there.  pyref.py keeps the plain template. */
static void axpby_setup_z(int64_t qa, int64_t ea, int za, int64_t qb, int64_t eb, int zb,
                          int64_t* d, int64_t* q, int64_t* e, int64_t* zd) {
  axpby_setup(qa, ea, qb, eb, d, q, e);
  if (!za != !zb) {
    const int64_t ee = za ? eb : ea;
    *zd += ee - *e;
    *e = ee;
    *d = 0;
    *q = max64(qa, qb) + 1;
  }
}
static int blk_zero(const ob_block* b) {
  for (int64_t i = 0; i < b->n; ++i)
    if (b->m[i]) return 0;
  return 1;
}

/* alpha*a*2^max(d,0) + beta*b*2^max(-d,0) with alpha/beta mantissas.
 * P/src/blas.cpp:60-72 (row) and 133-141 */
static inline int axpby_combine(i128 am, i128 a, i128 bm, i128 b, int64_t d, i128* out) {
  i128 ta, tb;
  if (mul_chk(am, a, &ta) || mul_chk(bm, b, &tb)) return 1;
  if (d < 0) {
    if (shl_chk(tb, -d, &tb)) return 1;
  } else {
    if (shl_chk(ta, d, &ta)) return 1;
  }
  return add_chk(ta, tb, out);
}

/* --- axpby: p[0..5] = am,aq,ae,bm,bq,be ; p[6] = d; ptr[0]=x, ptr[1]=y --- */
static int row_axpby(const ob_kernel* k, int64_t i, i128* out) {
  return axpby_combine(k->p[0], k->ptr[0][i], k->p[3], k->ptr[1][i], k->p[6], out) ? OB_ERR_WIDTH
                                                                                    : OB_OK;
}

int ob_make_axpby(ob_kernel* k, const ob_block* x, const ob_block* y, int64_t am, int64_t aq,
                  int64_t ae, int64_t bm, int64_t bq, int64_t be) {
  /* P/src/blas.cpp:41-58 */
  if (x->n != y->n) return OB_ERR_ARG;
  memset(k, 0, sizeof(*k));
  int64_t qa = aq + x->q, qb = bq + y->q, ea = ae + x->e, eb = be + y->e;
  axpby_setup_z(qa, ea, am == 0 || blk_zero(x), qb, eb, bm == 0 || blk_zero(y), &k->p[6], &k->q,
                &k->e, &k->zd);
  k->p[0] = am; k->p[1] = aq; k->p[2] = ae;
  k->p[3] = bm; k->p[4] = bq; k->p[5] = be;
  k->ptr[0] = x->m;
  k->ptr[1] = y->m;
  k->n = x->n;
  k->row = row_axpby;
  return OB_OK;
}

/* --- CSR spmv / gemv --- */
static int csr_dot(const ob_csr* a, const int64_t* x, int64_t i, i128* g) {
  /* P/src/blas.cpp:84-94 */
  i128 acc = 0;
  for (int64_t kk = a->rowptr[i]; kk < a->rowptr[i + 1]; ++kk) {
    i128 t;
    if (mul_chk(a->m[kk], x[a->col[kk]], &t) || add_chk(acc, t, &acc)) return 1;
  }
  *g = acc;
  return 0;
}
static int row_spmv(const ob_kernel* k, int64_t i, i128* out) {
  return csr_dot((const ob_csr*)k->a, k->ptr[0], i, out) ? OB_ERR_WIDTH : OB_OK;
}
int ob_make_spmv(ob_kernel* k, const ob_csr* a, const ob_block* x, int64_t m_a) {
  /* P/src/blas.cpp:74-82 */
  if (a->cols != x->n) return OB_ERR_DIM;
  if (m_a == 0) m_a = a->max_row_nnz;
  if (m_a < a->max_row_nnz) return OB_ERR_ARG;
  memset(k, 0, sizeof(*k));
  k->q = a->q + x->q + ceil_log2(max64(m_a, 1));
  k->e = a->e + x->e;
  k->a = a;
  k->ptr[0] = x->m;
  k->n = a->rows;
  k->row = row_spmv;
  return OB_OK;
}
static int row_gemv(const ob_kernel* k, int64_t i, i128* out) {
  i128 g;
  if (csr_dot((const ob_csr*)k->a, k->ptr[0], i, &g)) return OB_ERR_WIDTH;
  return axpby_combine(k->p[0], g, k->p[3], k->ptr[1][i], k->p[6], out) ? OB_ERR_WIDTH : OB_OK;
}
int ob_make_gemv(ob_kernel* k, const ob_csr* a, const ob_block* x, const ob_block* y, int64_t am,
                 int64_t aq, int64_t ae, int64_t bm, int64_t bq, int64_t be, int64_t m_a) {
  /* P/src/blas.cpp:96-120 */
  if (a->cols != x->n || a->rows != y->n) return OB_ERR_DIM;
  if (m_a == 0) m_a = a->max_row_nnz;
  if (m_a < a->max_row_nnz) return OB_ERR_ARG;
  memset(k, 0, sizeof(*k));
  int64_t gq = a->q + x->q + ceil_log2(max64(m_a, 1)), ge = a->e + x->e;
  axpby_setup_z(aq + gq, ae + ge, am == 0 || blk_zero(x), bq + y->q, be + y->e,
                bm == 0 || blk_zero(y), &k->p[6], &k->q, &k->e, &k->zd);
  k->p[0] = am; k->p[1] = aq; k->p[2] = ae;
  k->p[3] = bm; k->p[4] = bq; k->p[5] = be;
  k->p[7] = gq; k->p[8] = ge;
  k->a = a;
  k->ptr[0] = x->m;
  k->ptr[1] = y->m;
  k->n = a->rows;
  k->row = row_gemv;
  return OB_OK;
}

/* --- explicit rows (test FixedKernel) --- */
static int row_rows(const ob_kernel* k, int64_t i, i128* out) {
  *out = (i128)(((u128)(uint64_t)k->ptr[0][i] << 64) | (uint64_t)k->ptr[1][i]);
  return OB_OK;
}
int ob_make_rows(ob_kernel* k, int64_t n, const int64_t* hi, const uint64_t* lo, int64_t q,
                 int64_t e) {
  memset(k, 0, sizeof(*k));
  k->q = q;
  k->e = e;
  k->n = n;
  k->ptr[0] = hi;
  k->ptr[1] = (const int64_t*)lo;
  k->row = row_rows;
  return OB_OK;
}

int ob_kernel_row(const ob_kernel* k, int64_t i, int64_t* hi, uint64_t* lo) {
  i128 z;
  int rc = k->row(k, i, &z);
  *hi = (int64_t)(z >> 64);
  *lo = (uint64_t)z;
  return rc;
}

/* ------------------------------------------------------------------------ */
/* window drivers: P/src/blas.cpp:144-212                                    */

int ob_qcomp(const ob_kernel* k, int64_t w_out, int64_t w_tmp, int64_t gm, int64_t ge,
             int force_recompute, ob_block* out, ob_flags* flags) {
  if (w_out < 1 || w_out > w_tmp) return OB_ERR_ARG; /* :146 */
  if (w_out > 64 || w_tmp > 127) return OB_ERR_ARG;  /* storage limits of this restatement */
  if (gm <= 0) return OB_ERR_GAMMA;                   /* :32-36 */
  const int64_t n = k->n;
  const int64_t mu_tmp = msb128(gm) + ge - k->e;      /* :150 */
  const int64_t lam_tmp = mu_tmp - w_tmp;             /* :151 */
  /* the wrapped temporaries live in T_{w_tmp}: 64-bit storage when w_tmp <= 64 (config
     scale: halves the host memory of a 1023^3 solve), 128-bit otherwise */
  const int narrow = w_tmp <= 64;
  void* tmpv = malloc((narrow ? sizeof(int64_t) : sizeof(i128)) * (size_t)(n > 0 ? n : 1));
  i128* tmp = (i128*)tmpv;
  int64_t* tmp64 = (int64_t*)tmpv;
  int64_t mu_star = 1 - k->zd; /* :153 (mu* = 1 in the reference's coordinates) */
  int err = 0;
#pragma omp parallel for reduction(max : mu_star) reduction(| : err) schedule(static)
  for (int64_t i = 0; i < n; ++i) { /* :156-162 */
    i128 z;
    if (k->row(k, i, &z)) {
      err |= 1;
      continue;
    }
    if (z != 0) mu_star = max64(mu_star, msb128(z));
    i128 t = wrap_shift128(z, lam_tmp, w_tmp);
    if (narrow)
      tmp64[i] = (int64_t)t;
    else
      tmp[i] = t;
  }
  if (err) {
    free(tmpv);
    return OB_ERR_WIDTH;
  }
  const int64_t lam_out = mu_star - w_out; /* :164 */
  const int64_t e_out = k->e + lam_out;
  flags->overflow = mu_tmp < mu_star;      /* :167 */
  flags->underflow = lam_out < lam_tmp;    /* :168 */
  flags->recomputed = 0;
  if (flags->overflow || flags->underflow || force_recompute) { /* :171-177 */
    flags->recomputed = 1;
#pragma omp parallel for reduction(| : err) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      i128 z = 0, r = 0;
      if (k->row(k, i, &z) || shift_floor128(z, lam_out, &r)) {
        err |= 1;
        continue;
      }
      out->m[i] = (int64_t)r;
    }
  } else { /* :178-184 */
    const int64_t s = lam_out - lam_tmp;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      i128 r = 0;
      shift_floor128(narrow ? (i128)tmp64[i] : tmp[i], s, &r);
      out->m[i] = (int64_t)wrap128(r, w_out);
    }
  }
  free(tmpv);
  if (err) return OB_ERR_WIDTH;
  out->n = n;
  out->q = w_out;
  out->e = e_out;
  return OB_OK;
}

int ob_nnqcomp(const ob_kernel* k, int64_t w_out, int64_t gm, int64_t ge, ob_block* out) {
  /* P/src/blas.cpp:189-212 */
  if (w_out < 1 || w_out > 64) return OB_ERR_ARG;
  if (gm <= 0) return OB_ERR_GAMMA;
  const int64_t n = k->n;
  const int64_t mu_out = msb128(gm) + ge - k->e;
  const int64_t lam_out = mu_out - w_out;
  int err = 0;
#pragma omp parallel for reduction(| : err) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    i128 z, r;
    if (k->row(k, i, &z)) {
      err |= 1;
      continue;
    }
    if (shift_floor128(z, lam_out, &r)) /* left shift beyond 128 bits: saturates anyway */
      r = z < 0 ? -(((i128)1) << 126) : (((i128)1) << 126);
    out->m[i] = (int64_t)clamp_w(r, w_out);
  }
  if (err) return OB_ERR_WIDTH;
  out->n = n;
  out->q = w_out;
  out->e = k->e + lam_out;
  return OB_OK;
}

/* ------------------------------------------------------------------------ */
/* grid operators                                      */

int64_t ob_grid_n(ob_grid g) { return ((int64_t)1 << g.l) - 1; }
int64_t ob_grid_size(ob_grid g) {
  int64_t n = ob_grid_n(g), s = 1;
  for (int a = 0; a < g.d; ++a) s *= n;
  return s;
}

void ob_stencil_desc(ob_grid g, int64_t* qa, int64_t* ea, int64_t* ma) {
  *qa = msb128(2 * g.d); /* centre mantissa 2d, neighbours -1 */
  *ea = 2 * (int64_t)g.l; /* h^-2 = 2^{2l} */
  *ma = 2 * g.d + 1;
}

/* exact (S_d x)_i in mantissa units; x interior-only, zero outside */
static inline i128 stencil_row(int d, int64_t n, const int64_t* x, int64_t i) {
  int64_t ix = i % n;
  i128 acc = (i128)(2 * d) * x[i];
  if (ix > 0) acc -= x[i - 1];
  if (ix < n - 1) acc -= x[i + 1];
  if (d >= 2) {
    int64_t iy = (i / n) % n;
    if (iy > 0) acc -= x[i - n];
    if (iy < n - 1) acc -= x[i + n];
  }
  if (d >= 3) {
    int64_t n2 = n * n, iz = i / n2;
    if (iz > 0) acc -= x[i - n2];
    if (iz < n - 1) acc -= x[i + n2];
  }
  return acc;
}

/* stencil gemv: p[0..5] alpha/beta, p[6] d, p[10] dim, p[11] n */
static int row_stencil_gemv(const ob_kernel* k, int64_t i, i128* out) {
  i128 g = stencil_row((int)k->p[10], k->p[11], k->ptr[0], i);
  return axpby_combine(k->p[0], g, k->p[3], k->ptr[1][i], k->p[6], out) ? OB_ERR_WIDTH : OB_OK;
}
int ob_make_stencil_gemv(ob_kernel* k, ob_grid g, const ob_block* x, const ob_block* y,
                         int64_t am, int64_t aq, int64_t ae, int64_t bm, int64_t bq, int64_t be) {
  /* EgemvKernel (P/src/blas.cpp:96-120) with A = the level-l stencil */
  int64_t N = ob_grid_size(g);
  if (x->n != N || y->n != N) return OB_ERR_DIM;
  memset(k, 0, sizeof(*k));
  int64_t qa, ea, ma;
  ob_stencil_desc(g, &qa, &ea, &ma);
  int64_t gq = qa + x->q + ceil_log2(ma), ge = ea + x->e;
  axpby_setup_z(aq + gq, ae + ge, am == 0 || blk_zero(x), bq + y->q, be + y->e,
                bm == 0 || blk_zero(y), &k->p[6], &k->q, &k->e, &k->zd);
  k->p[0] = am; k->p[1] = aq; k->p[2] = ae;
  k->p[3] = bm; k->p[4] = bq; k->p[5] = be;
  k->p[7] = gq; k->p[8] = ge;
  k->p[10] = g.d;
  k->p[11] = ob_grid_n(g);
  k->ptr[0] = x->m;
  k->ptr[1] = y->m;
  k->n = N;
  k->row = row_stencil_gemv;
  return OB_OK;
}

/* Jacobi: z = x + c*(b - A x).  p[0]=cm, p[1]=d1, p[2]=d2, p[10]=dim, p[11]=n */
static int row_jacobi(const ob_kernel* k, int64_t i, i128* out) {
  i128 g = stencil_row((int)k->p[10], k->p[11], k->ptr[0], i), r;
  /* r = (-1)*g*2^max(d1,0) + (+1)*b*2^max(-d1,0) */
  if (axpby_combine(-1, g, 1, k->ptr[1][i], k->p[1], &r)) return OB_ERR_WIDTH;
  /* z = (+1)*x*2^max(d2,0) + c*r*2^max(-d2,0) */
  return axpby_combine(1, k->ptr[0][i], k->p[0], r, k->p[2], out) ? OB_ERR_WIDTH : OB_OK;
}
int ob_make_jacobi(ob_kernel* k, ob_grid g, const ob_block* x, const ob_block* b, int64_t cm,
                   int64_t cq, int64_t ce) {
  int64_t N = ob_grid_size(g);
  if (x->n != N || b->n != N) return OB_ERR_DIM;
  memset(k, 0, sizeof(*k));
  int64_t qa, ea, ma, d1, qr, er, d2;
  ob_stencil_desc(g, &qa, &ea, &ma);
  int64_t gq = qa + x->q + ceil_log2(ma), ge = ea + x->e;
  const int zx = blk_zero(x), zb = blk_zero(b);
  int64_t zr = 0, e_ref = min64(x->e, ce + min64(ge, b->e)); /* the reference chain's e* */
  /* r = egemv(A, x, b, bfp_minus_one, bfp_one): alpha q=1 e=0, beta q=2 e=0 */
  axpby_setup_z(1 + gq, ge, zx, 2 + b->q, b->e, zb, &d1, &qr, &er, &zr);
  /* z = eaxpby(x, r, bfp_one, c) */
  axpby_setup_z(2 + x->q, x->e, zx, cq + qr, ce + er, cm == 0 || (zx && zb), &d2, &k->q, &k->e,
                &zr);
  k->zd = k->e - e_ref;
  k->p[0] = cm;
  k->p[1] = d1;
  k->p[2] = d2;
  k->p[3] = qr;
  k->p[4] = er;
  k->p[10] = g.d;
  k->p[11] = ob_grid_n(g);
  k->ptr[0] = x->m;
  k->ptr[1] = b->m;
  k->n = N;
  k->row = row_jacobi;
  return OB_OK;
}

static int row_scal(const ob_kernel* k, int64_t i, i128* out) {
  return mul_chk(k->p[0], k->ptr[0][i], out) ? OB_ERR_WIDTH : OB_OK;
}
int ob_make_scal(ob_kernel* k, const ob_block* r, int64_t cm, int64_t cq, int64_t ce) {
  memset(k, 0, sizeof(*k));
  k->q = cq + r->q;
  k->e = ce + r->e;
  k->p[0] = cm;
  k->ptr[0] = r->m;
  k->n = r->n;
  k->row = row_scal;
  return OB_OK;
}

/* full weighting: coarse (I,J,K) <- fine (2I+1+a, ...), weights prod (2-|a|) */
static int row_restrict(const ob_kernel* k, int64_t ic, i128* out) {
  const int d = (int)k->p[10];
  const int64_t nf = k->p[11], nc = k->p[12];
  const int64_t* r = k->ptr[0];
  int64_t c[3] = {0, 0, 0}, t = ic;
  for (int a = 0; a < d; ++a) {
    c[a] = t % nc;
    t /= nc;
  }
  i128 acc = 0;
  int lim1 = d >= 2 ? 1 : 0, lim2 = d >= 3 ? 1 : 0;
  for (int dz = -lim2; dz <= lim2; ++dz)
    for (int dy = -lim1; dy <= lim1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int64_t fx = 2 * c[0] + 1 + dx, fy = 2 * c[1] + 1 + dy, fz = 2 * c[2] + 1 + dz;
        int64_t w = (2 - (dx < 0 ? -dx : dx));
        if (d >= 2) w *= (2 - (dy < 0 ? -dy : dy));
        if (d >= 3) w *= (2 - (dz < 0 ? -dz : dz));
        int64_t fi = fx + (d >= 2 ? nf * fy : 0) + (d >= 3 ? nf * nf * fz : 0);
        acc += (i128)w * r[fi];
      }
  *out = acc;
  return OB_OK;
}
int ob_make_restrict(ob_kernel* k, ob_grid gf, const ob_block* r) {
  /* EspmvKernel (P/src/blas.cpp:74-82) with R = full weighting P^T/2^d:
     mantissas (1,2,1)^{(x)d}, e_R = -2d, q_R = d+2, m_R = 3^d */
  if (gf.l < 2 || r->n != ob_grid_size(gf)) return OB_ERR_DIM;
  memset(k, 0, sizeof(*k));
  ob_grid gc = {gf.d, gf.l - 1};
  int64_t m_r = 1;
  for (int a = 0; a < gf.d; ++a) m_r *= 3;
  k->q = (gf.d + 2) + r->q + ceil_log2(m_r);
  k->e = -2 * (int64_t)gf.d + r->e;
  k->p[10] = gf.d;
  k->p[11] = ob_grid_n(gf);
  k->p[12] = ob_grid_n(gc);
  k->ptr[0] = r->m;
  k->n = ob_grid_size(gc);
  k->row = row_restrict;
  return OB_OK;
}

/* linear interpolation P: fine (i) from coarse; 1-D weights: odd i -> coarse
   (i-1)/2 mantissa 2; even i -> coarse i/2-1 and i/2 mantissa 1 each.      */
static inline i128 prolong_row(int d, int64_t nf, int64_t nc, const int64_t* xc, int64_t i) {
  int64_t f[3] = {0, 0, 0}, t = i;
  for (int a = 0; a < d; ++a) {
    f[a] = t % nf;
    t /= nf;
  }
  int64_t ci[3][2], cw[3][2];
  int cnt[3] = {1, 1, 1};
  for (int a = 0; a < 3; ++a) {
    ci[a][0] = 0;
    cw[a][0] = 1;
    if (a >= d) continue;
    if (f[a] & 1) {
      ci[a][0] = (f[a] - 1) / 2;
      cw[a][0] = 2;
      cnt[a] = 1;
    } else {
      cnt[a] = 0;
      int64_t lo = f[a] / 2 - 1, hi = f[a] / 2;
      if (lo >= 0) {
        ci[a][cnt[a]] = lo;
        cw[a][cnt[a]++] = 1;
      }
      if (hi < nc) {
        ci[a][cnt[a]] = hi;
        cw[a][cnt[a]++] = 1;
      }
    }
  }
  i128 acc = 0;
  for (int z = 0; z < cnt[2]; ++z)
    for (int y = 0; y < cnt[1]; ++y)
      for (int x = 0; x < cnt[0]; ++x) {
        int64_t idx = ci[0][x] + (d >= 2 ? nc * ci[1][y] : 0) + (d >= 3 ? nc * nc * ci[2][z] : 0);
        acc += (i128)(cw[0][x] * cw[1][y] * cw[2][z]) * xc[idx];
      }
  return acc;
}
static int row_prolong(const ob_kernel* k, int64_t i, i128* out) {
  *out = prolong_row((int)k->p[10], k->p[11], k->p[12], k->ptr[0], i);
  return OB_OK;
}
int ob_make_prolong(ob_kernel* k, ob_grid gf, const ob_block* xc) {
  /* EspmvKernel with P: mantissas prod of {2 | 1,1}, e_P = -d, q_P = d+2, m_P = 2^d */
  ob_grid gc = {gf.d, gf.l - 1};
  if (gf.l < 2 || xc->n != ob_grid_size(gc)) return OB_ERR_DIM;
  memset(k, 0, sizeof(*k));
  k->q = (gf.d + 2) + xc->q + gf.d; /* + ceil_log2(2^d) */
  k->e = -(int64_t)gf.d + xc->e;
  k->p[10] = gf.d;
  k->p[11] = ob_grid_n(gf);
  k->p[12] = ob_grid_n(gc);
  k->ptr[0] = xc->m;
  k->n = ob_grid_size(gf);
  k->row = row_prolong;
  return OB_OK;
}
static int row_prolong_correct(const ob_kernel* k, int64_t i, i128* out) {
  i128 g = prolong_row((int)k->p[10], k->p[11], k->p[12], k->ptr[0], i);
  return axpby_combine(1, g, 1, k->ptr[1][i], k->p[6], out) ? OB_ERR_WIDTH : OB_OK;
}
int ob_make_prolong_correct(ob_kernel* k, ob_grid gf, const ob_block* ec, const ob_block* y) {
  /* EgemvKernel(P, ec, y, bfp_one, bfp_one) */
  ob_grid gc = {gf.d, gf.l - 1};
  if (gf.l < 2 || ec->n != ob_grid_size(gc) || y->n != ob_grid_size(gf)) return OB_ERR_DIM;
  memset(k, 0, sizeof(*k));
  int64_t gq = (gf.d + 2) + ec->q + gf.d, ge = -(int64_t)gf.d + ec->e;
  axpby_setup_z(2 + gq, ge, blk_zero(ec), 2 + y->q, y->e, blk_zero(y), &k->p[6], &k->q, &k->e,
                &k->zd);
  k->p[10] = gf.d;
  k->p[11] = ob_grid_n(gf);
  k->p[12] = ob_grid_n(gc);
  k->ptr[0] = ec->m;
  k->ptr[1] = y->m;
  k->n = ob_grid_size(gf);
  k->row = row_prolong_correct;
  return OB_OK;
}

void ob_jacobi_coeff(ob_grid g, int64_t qc, int64_t* cm, int64_t* ce) {
  /* omega_d/(2d) = {1/3, 1/5, 1/7} (omega = 2/3, 4/5, 6/7), floor-quantised
     at qc bits like quantize_scalar_floor (P/src/multigrid.cpp:233-241) */
  int64_t num = 1, den = g.d == 1 ? 3 : (g.d == 2 ? 5 : 7);
  /* top = floor(log2 v) + 2 */
  int64_t fl = 0;
  while ((num << (-fl)) < den) --fl; /* v < 1: largest fl<=0 with 2^fl <= v */
  int64_t top = fl + 2;
  int64_t sh = qc - top; /* m = floor(num * 2^sh / den), sh > 0 here */
  *cm = (int64_t)(((i128)num << sh) / den);
  *ce = top - qc - 2 * (int64_t)g.l;
}

/* ------------------------------------------------------------------------ */
/* gamma arithmetic                                    */

ob_g15 ob_g15_from(uint64_t mag, int64_t e) {
  ob_g15 r = {0, 0};
  if (mag == 0) return r;
  int64_t b = bitlen_u128(mag);
  if (b <= 15) {
    r.m = (int64_t)(mag << (15 - b));
    r.e = e - (15 - b);
  } else {
    int64_t s = b - 15;
    uint64_t m = (mag >> s) + ((mag & ((1ull << s) - 1)) != 0);
    if (m == (1ull << 15)) {
      m >>= 1;
      ++s;
    }
    r.m = (int64_t)m;
    r.e = e + s;
  }
  return r;
}
static ob_g15 g15_from128(u128 mag, int64_t e) {
  int64_t b = bitlen_u128(mag);
  if (b <= 64) return ob_g15_from((uint64_t)mag, e);
  int64_t s = b - 64;
  /* fold the sticky bits: ceil is preserved by OR-ing them into bit 0 */
  uint64_t top = (uint64_t)(mag >> s) | ((mag & ((((u128)1) << s) - 1)) != 0);
  return ob_g15_from(top, e + s);
}
ob_g15 ob_g15_norm(const ob_block* x, int64_t unused) {
  (void)unused;
  uint64_t mx = 0;
  for (int64_t i = 0; i < x->n; ++i) {
    int64_t v = x->m[i];
    uint64_t a = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
    if (a > mx) mx = a;
  }
  return ob_g15_from(mx, x->e);
}
ob_g15 ob_g15_mul(ob_g15 a, ob_g15 b) {
  ob_g15 z = {0, 0};
  if (a.m == 0 || b.m == 0) return z;
  return ob_g15_from((uint64_t)a.m * (uint64_t)b.m, a.e + b.e);
}
ob_g15 ob_g15_add(ob_g15 a, ob_g15 b) {
  if (a.m == 0) return b;
  if (b.m == 0) return a;
  if (a.e < b.e) {
    ob_g15 t = a;
    a = b;
    b = t;
  } /* a has the larger exponent */
  int64_t gap = a.e - b.e;
  if (gap <= 100) {
    u128 s = ((u128)a.m << gap) + (u128)b.m;
    return g15_from128(s, b.e);
  }
  ob_g15 r = a;
  r.m += 1;
  if (r.m == (1 << 15)) {
    r.m = 1 << 14;
    r.e += 1;
  }
  return r;
}
void ob_g15_gamma(ob_g15 g, int64_t* gm, int64_t* ge) {
  if (g.m == 0) { /* degenerate gamma, P/src/multigrid.cpp:84-89 */
    *gm = 1 << 14;
    *ge = -400 - 14;
  } else {
    *gm = g.m;
    *ge = g.e;
  }
}

/* ------------------------------------------------------------------------ */
/* generators                                          */

uint64_t ob_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int ob_gen_uniform(ob_grid g, int64_t p, uint64_t seed, uint64_t stream, ob_block* out) {
  if (p < 2 || p > 62) return OB_ERR_ARG;
  int64_t N = ob_grid_size(g);
  uint64_t key = ob_splitmix64(ob_splitmix64(seed) ^ stream);
  for (int64_t i = 0; i < N; ++i) {
    uint64_t r = ob_splitmix64(key + (uint64_t)i);
    out->m[i] = (int64_t)(r >> (64 - p)) - ((int64_t)1 << (p - 1));
  }
  out->n = N;
  out->q = p;
  out->e = -(p - 1);
  return ob_normalize(out, out);
}

int ob_gen_sine(ob_grid g, int64_t p, ob_block* out) {
  /* f = d*pi^2 prod_a sin(pi x_a), x_a = (i_a+1) h, double products without
     contraction, then quantize_exact at p bits (P/src/bfp.cpp:163-187) */
  if (p < 2 || p > 62) return OB_ERR_ARG;
  int64_t n = ob_grid_n(g), N = ob_grid_size(g);
  double h = ldexp(1.0, -g.l);
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) s[i] = sin(M_PI * ((double)(i + 1) * h));
  const double C = (double)g.d * (M_PI * M_PI);
  int64_t top = INT64_MIN;
  int64_t* zk = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  for (int64_t i = 0; i < N; ++i) {
    int64_t ix = i % n, iy = (i / n) % n, iz = i / (n * n);
    double v = C * s[ix];
    if (g.d >= 2) v = v * s[iy];
    if (g.d >= 3) v = v * s[iz];
    int ex;
    double fr = frexp(v, &ex);
    int64_t z = (int64_t)ldexp(fr, 53);
    int64_t k = (int64_t)ex - 53;
    out->m[i] = z;
    zk[i] = k;
    if (z != 0) top = max64(top, msb128(z) + k);
  }
  int64_t e_out = 0;
  if (top != INT64_MIN) {
    e_out = top - p;
    for (int64_t i = 0; i < N; ++i) {
      i128 r = 0;
      shift_floor128(out->m[i], e_out - zk[i], &r);
      out->m[i] = (int64_t)r;
    }
  }
  free(s);
  free(zk);
  out->n = N;
  out->q = p;
  out->e = e_out;
  return OB_OK;
}

/* ------------------------------------------------------------------------ */
/* multigrid driver (structure of P/src/multigrid.cpp:399-518) */

typedef struct {
  const ob_mg_config* cfg;
  ob_mg_result* res;
  int err;
  int have_prev_res[33];
  ob_g15 prev_res[33];
  int ir_iter; /* 1-based IR iteration of the current ir() loop (hybrid mode) */
} mg_ctx;

static ob_block blk_alloc(int64_t n) {
  ob_block b;
  b.n = n;
  b.q = 1;
  b.e = 0;
  b.m = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  return b;
}
static void blk_free(ob_block* b) {
  free(b->m);
  b->m = NULL;
}
static ob_g15 nrm(const ob_block* b) { return ob_g15_norm(b, 0); }
static double norm_double(const ob_block* b) {
  uint64_t mx = 0;
  for (int64_t i = 0; i < b->n; ++i) {
    int64_t v = b->m[i];
    uint64_t a = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
    if (a > mx) mx = a;
  }
  return ldexp((double)mx, (int)b->e);
}

/* run_step: P/src/multigrid.cpp:399-426 */
static void run_step(mg_ctx* c, int step, int level, const ob_kernel* k, int64_t w_out,
                     ob_g15 gamma, int w_add, ob_block* out) {
  if (c->err) return;
  /* NormMode (P/src/multigrid.cpp:403-409): 0 normalized, 1 nonnormalized,
     2 hybrid = qcomp only for the IR residual of iterations <= hybrid_qcomp_iters (2) */
  int normalized = c->cfg->nonnormalized == 0 || step == OB_STEP_FINAL_RES ||
                   (c->cfg->nonnormalized == 2 && step == OB_STEP_IR_RES && c->ir_iter <= 2);
  int64_t gm, ge;
  ob_g15_gamma(gamma, &gm, &ge);
  ob_flags fl = {0, 0, 0};
  int rc;
  /* GammaPolicy::w_tmp_for (P/src/multigrid.cpp:81-85): w_out + min(w_add, cap) */
  if (c->cfg->w_add_cap >= 0 && w_add > c->cfg->w_add_cap) w_add = c->cfg->w_add_cap;
  int64_t w_tmp = w_out + w_add;
  if (normalized)
    rc = ob_qcomp(k, w_out, w_tmp, gm, ge, 0, out, &fl);
  else
    rc = ob_nnqcomp(k, w_out, gm, ge, out);
  if (rc) {
    c->err = rc;
    return;
  }
  ob_mg_result* r = c->res;
  if (r->trace && r->n_trace < r->trace_cap) {
    ob_trace_rec* t = &r->trace[r->n_trace];
    t->step = step;
    t->level = level;
    t->w_out = (int32_t)w_out;
    t->w_tmp = (int32_t)(normalized ? w_tmp : w_out);
    t->gm = gm;
    t->ge = ge;
    t->overflow = fl.overflow;
    t->underflow = fl.underflow;
    t->recomputed = fl.recomputed;
    t->normalized = normalized;
  }
  r->n_trace++;
}

/* PrecisionSchedule (P/src/multigrid.cpp:13-44): w = iterate, wdot = residual and
   V-cycle, wcheck = right-hand side; 0 entries default to w */
static int64_t wl(const mg_ctx* c, int l) { return c->cfg->p[l]; }
static int64_t wd(const mg_ctx* c, int l) { return c->cfg->pd[l] ? c->cfg->pd[l] : c->cfg->p[l]; }
static int64_t wc(const ob_mg_config* cfg, int l) { return cfg->pc[l] ? cfg->pc[l] : cfg->p[l]; }

/* V-cycle correction scheme on A e = r, e0 = 0 */
static void vcycle(mg_ctx* c, int l, const ob_block* r, ob_block* e_out) {
  const ob_mg_config* cfg = c->cfg;
  ob_grid g = {cfg->d, l};
  int64_t N = ob_grid_size(g), cm, ce;
  ob_jacobi_coeff(g, cfg->qc, &cm, &ce);
  ob_g15 c15 = ob_g15_from((uint64_t)cm, ce);
  ob_kernel k;
  ob_block e = *e_out, t = blk_alloc(N); /* e starts in the caller's buffer */
  e.n = N;
  ob_make_scal(&k, r, cm, cfg->qc, ce);
  run_step(c, OB_STEP_RELAX0, l, &k, wd(c, l), ob_g15_mul(c15, nrm(r)), 2, &e);
  int sweeps = (l == cfg->l_coarse) ? cfg->n_coarse : cfg->nu1;
  for (int s = 1; s < sweeps && !c->err; ++s) {
    ob_make_jacobi(&k, g, &e, r, cm, cfg->qc, ce);
    run_step(c, OB_STEP_RELAX, l, &k, wd(c, l), ob_g15_add(nrm(&e), ob_g15_mul(c15, nrm(r))), 3,
             &t);
    ob_block sw = e;
    e = t;
    t = sw;
  }
  if (l > cfg->l_coarse && !c->err) {
    ob_grid gc = {cfg->d, l - 1};
    int64_t Nc = ob_grid_size(gc);
    ob_block rv = blk_alloc(N), rc = blk_alloc(Nc), ec = blk_alloc(Nc);
    ob_make_stencil_gemv(&k, g, &e, r, -1, 1, 0, 1, 2, 0);
    run_step(c, OB_STEP_V_RES, l, &k, wd(c, l), nrm(r), 4, &rv);
    ob_make_restrict(&k, g, &rv);
    run_step(c, OB_STEP_RESTRICT, l, &k, wd(c, l), nrm(&rv), 6, &rc);
    if (!c->err) vcycle(c, l - 1, &rc, &ec);
    ob_make_prolong_correct(&k, g, &ec, &e);
    run_step(c, OB_STEP_V_CORR, l, &k, wd(c, l), ob_g15_add(nrm(&e), nrm(&ec)), 2, &t);
    ob_block sw = e;
    e = t;
    t = sw;
    for (int s = 0; s < cfg->nu2 && !c->err; ++s) {
      ob_make_jacobi(&k, g, &e, r, cm, cfg->qc, ce);
      run_step(c, OB_STEP_RELAX, l, &k, wd(c, l),
               ob_g15_add(nrm(&e), ob_g15_mul(c15, nrm(r))), 3, &t);
      sw = e;
      e = t;
      t = sw;
    }
    blk_free(&rv);
    blk_free(&rc);
    blk_free(&ec);
  }
  if (e.m != e_out->m) { /* the result ended in the scratch buffer */
    memcpy(e_out->m, e.m, sizeof(int64_t) * (size_t)N);
    blk_free(&e);
  } else {
    blk_free(&t);
  }
  e_out->n = N;
  e_out->q = e.q;
  e_out->e = e.e;
}

static void push_hist(mg_ctx* c, double v) {
  ob_mg_result* r = c->res;
  if (r->res_history) r->res_history[r->n_history] = v;
  r->n_history++;
}

/* IR with V-cycle inner solver (P/src/multigrid.cpp:458-500), x updated in place */
static void ir(mg_ctx* c, int l, ob_block* x, const ob_block* b, int iters) {
  const ob_mg_config* cfg = c->cfg;
  ob_grid g = {cfg->d, l};
  int64_t N = ob_grid_size(g);
  ob_kernel k;
  ob_block r = blk_alloc(N), e = blk_alloc(N);
  c->have_prev_res[l] = 0;
  for (int i = 1; i <= iters && !c->err; ++i) {
    int first = !c->have_prev_res[l];
    ob_g15 gam = c->prev_res[l];
    if (first) { /* ||b|| + ||A|| ulp(x) */
      ob_g15 ulp = nrm(x).m ? ob_g15_from(1, x->e) : (ob_g15){0, 0};
      gam = ob_g15_add(nrm(b), ob_g15_mul(ob_g15_from((uint64_t)(4 * cfg->d), 2 * (int64_t)l), ulp));
    }
    ob_make_stencil_gemv(&k, g, x, b, -1, 1, 0, 1, 2, 0);
    c->ir_iter = i;
    run_step(c, OB_STEP_IR_RES, l, &k, wd(c, l), gam, first ? 5 : 4, &r);
    if (c->err) break;
    c->prev_res[l] = nrm(&r);
    c->have_prev_res[l] = 1;
    push_hist(c, norm_double(&r));
    vcycle(c, l, &r, &e);
    /* r is dead after the V-cycle: it receives the corrected iterate */
    ob_make_axpby(&k, x, &e, 1, 2, 0, 1, 2, 0);
    run_step(c, OB_STEP_IR_CORR, l, &k, wl(c, l), ob_g15_add(nrm(x), nrm(&e)), 1, &r);
    memcpy(x->m, r.m, sizeof(int64_t) * (size_t)N);
    x->q = r.q;
    x->e = r.e;
  }
  blk_free(&r);
  blk_free(&e);
}

static int gen_rhs(const ob_mg_config* cfg, ob_grid g, ob_block* b) {
  int64_t p = wc(cfg, g.l);
  if (cfg->rhs_kind == 1) return ob_gen_sine(g, p, b);
  if (cfg->rhs_kind == 0) return ob_gen_uniform(g, p, cfg->seed, 2, b);
  b->n = ob_grid_size(g);
  b->q = p;
  b->e = 0;
  memset(b->m, 0, sizeof(int64_t) * (size_t)b->n);
  return OB_OK;
}

static void fmg(mg_ctx* c, int l, ob_block* x_out) {
  const ob_mg_config* cfg = c->cfg;
  ob_grid g = {cfg->d, l};
  int64_t N = ob_grid_size(g);
  ob_block b = blk_alloc(N);
  int rc = gen_rhs(cfg, g, &b);
  if (rc) c->err = rc;
  if (l == cfg->l_coarse) { /* zero_vec (P/src/bfp.cpp:53-55) */
    memset(x_out->m, 0, sizeof(int64_t) * (size_t)N);
    x_out->n = N;
    x_out->q = wl(c, l);
    x_out->e = 0;
  } else {
    ob_grid gc = {cfg->d, l - 1};
    ob_block xc = blk_alloc(ob_grid_size(gc));
    fmg(c, l - 1, &xc);
    ob_kernel k;
    ob_make_prolong(&k, g, &xc);
    run_step(c, OB_STEP_FMG_PROLONG, l, &k, wl(c, l), nrm(&xc), 1, x_out);
    blk_free(&xc);
  }
  if (!c->err) ir(c, l, x_out, &b, cfg->cycles);
  if (l == cfg->l_fine && !c->err) {
    ob_block r = blk_alloc(N);
    ob_kernel k;
    ob_make_stencil_gemv(&k, g, x_out, &b, -1, 1, 0, 1, 2, 0);
    run_step(c, OB_STEP_FINAL_RES, l, &k, wd(c, l), c->prev_res[l], 4, &r);
    push_hist(c, norm_double(&r));
    blk_free(&r);
  }
  blk_free(&b);
}

int ob_mg_run(const ob_mg_config* cfg, ob_mg_result* res) {
  if (cfg->d < 1 || cfg->d > 3 || cfg->l_coarse < 2 || cfg->l_fine < cfg->l_coarse ||
      cfg->l_fine > 30 || cfg->nu1 < 1 || cfg->n_coarse < 1)
    return OB_ERR_ARG;
  mg_ctx c;
  memset(&c, 0, sizeof(c));
  c.cfg = cfg;
  c.res = res;
  res->n_history = 0;
  res->n_trace = 0;
  ob_grid g = {cfg->d, cfg->l_fine};
  int64_t N = ob_grid_size(g);
  if (cfg->fmg) {
    fmg(&c, cfg->l_fine, &res->x);
  } else {
    ob_block b = blk_alloc(N);
    int rc = gen_rhs(cfg, g, &b);
    if (rc) c.err = rc;
    ob_block* x = &res->x;
    if (cfg->x0_random)
      rc = ob_gen_uniform(g, cfg->p[cfg->l_fine], cfg->seed, 1, x);
    else {
      memset(x->m, 0, sizeof(int64_t) * (size_t)N);
      x->n = N;
      x->q = cfg->p[cfg->l_fine];
      x->e = 0;
    }
    if (rc) c.err = rc;
    if (!c.err) ir(&c, cfg->l_fine, x, &b, cfg->cycles);
    if (!c.err) {
      ob_block r = blk_alloc(N);
      ob_kernel k;
      ob_make_stencil_gemv(&k, g, x, &b, -1, 1, 0, 1, 2, 0);
      run_step(&c, OB_STEP_FINAL_RES, cfg->l_fine, &k, wd(&c, cfg->l_fine),
               c.prev_res[cfg->l_fine], 4, &r);
      push_hist(&c, norm_double(&r));
      blk_free(&r);
    }
    blk_free(&b);
  }
  res->err = c.err;
  return c.err;
}

/* ------------------------------------------------------------------------ */
/* CPU baseline: fine residual r = b - A x, qcomp, OpenMP (reference loops
   P/src/blas.cpp:156-185 with the row of P/src/blas.cpp:122-142)            */

int ob_residual_qcomp_omp(ob_grid g, const ob_block* x, const ob_block* b, int64_t w_out,
                          int64_t w_tmp, int64_t gm, int64_t ge, ob_block* out, ob_flags* fl,
                          int threads) {
#ifdef _OPENMP
  int saved = omp_get_max_threads();
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  ob_kernel k;
  int rc = ob_make_stencil_gemv(&k, g, x, b, -1, 1, 0, 1, 2, 0);
  if (!rc) rc = ob_qcomp(&k, w_out, w_tmp, gm, ge, 0, out, fl);
#ifdef _OPENMP
  omp_set_num_threads(saved);
#endif
  return rc;
}
