// bfpmg_b200.hpp -- C++ facade over the C-ABI (include/bfpmg_b200.h) that restores the
// reference's BLAS-level API: the names, argument order, result types and exception types
// of P/include/bfpmg/blas.hpp:98-146 and P/include/bfpmg/bfp.hpp (paths relative to
// /root/reference/proj), with int64 mantissas where the reference holds mpz_class.
//
//   reference                                  facade (namespace bfpmg_b200)
//   BfpBlock::vec / zero_vec / mant(i)         BfpBlock::vec / zero_vec / mant(i)
//   BfpScalar (a one-element block)            BfpScalar{m, q, e}
//   BfpCsr                                     BfpCsr(rows, cols, rowptr, col, m, q, e)
//   normalize / quantize / inf_norm_upper      same names (P/src/bfp.cpp:97-148)
//   qaxpby qsub qspmv qgemv                    same names (P/src/blas.cpp:214-234)
//   nnqaxpby nnqsub nnqspmv nnqgemv            same names (P/src/blas.cpp:236-256)
//   QcompResult{z, flags}, QcompFlags          same
//   bfp_one / bfp_minus_one                    same (q = 2 resp. 1, e = 0)
//   dump_block / parse_block                   same (P/src/bfp.cpp:230-272)
//   std::invalid_argument / std::domain_error  thrown from the status codes;
//   (mpz rows are unbounded)                   std::overflow_error beyond 127-bit rows
//
// Header-only: compile with -I<repo>/include and link -lbfpmg_b200.  Every call uploads its
// operands, runs the sm_100a kernels and downloads the result (one round trip per op, like
// the reference's value semantics); whole solves should use bfp_mg_* and stay on the device.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bfpmg_b200.h"

namespace bfpmg_b200 {

inline void check(int st, const char* what) {
  switch (st) {
    case BFP_OK: return;
    case BFP_ERR_DOMAIN:
    case BFP_ERR_STORAGE: throw std::domain_error(std::string(what) + ": " + bfp_status_string(st));
    case BFP_ERR_WIDTH: throw std::overflow_error(std::string(what) + ": " + bfp_status_string(st));
    case BFP_ERR_ARG:
    case BFP_ERR_ALIAS: throw std::invalid_argument(std::string(what) + ": " + bfp_status_string(st));
    default: throw std::runtime_error(std::string(what) + ": " + bfp_status_string(st));
  }
}

struct BfpScalar {
  std::int64_t m, q, e;
  bfp_scalar_t c() const { return bfp_scalar_t{m, q, e}; }
};
inline BfpScalar bfp_one() { return {1, 2, 0}; }
inline BfpScalar bfp_minus_one() { return {-1, 1, 0}; }

/// A BFP vector block on the host: mantissas in T_q with one shared exponent.
class BfpBlock {
 public:
  BfpBlock() = default;
  /// check_fits (P/src/bfp.cpp:33-40): a mantissa outside T_q throws std::domain_error.
  static BfpBlock vec(std::vector<std::int64_t> m, std::int64_t q, std::int64_t e) {
    if (q < 1 || q > 64) throw std::invalid_argument("BfpBlock::vec: width");
    for (std::int64_t v : m) {
      const std::int64_t lo = q >= 64 ? INT64_MIN : -(std::int64_t(1) << (q - 1));
      const std::int64_t hi = q >= 64 ? INT64_MAX : (std::int64_t(1) << (q - 1)) - 1;
      if (v < lo || v > hi) throw std::domain_error("BfpBlock::vec: mantissa does not fit T_q");
    }
    BfpBlock b;
    b.m_ = std::move(m);
    b.q_ = q;
    b.e_ = e;
    return b;
  }
  static BfpBlock zero_vec(std::int64_t n, std::int64_t q) {
    return vec(std::vector<std::int64_t>((std::size_t)n, 0), q, 0);
  }
  std::int64_t q() const { return q_; }
  std::int64_t e() const { return e_; }
  std::size_t size() const { return m_.size(); }
  std::int64_t rows() const { return (std::int64_t)m_.size(); }
  std::int64_t mant(std::size_t i) const { return m_.at(i); }
  const std::vector<std::int64_t>& mantissas() const { return m_; }
  bool operator==(const BfpBlock& o) const { return q_ == o.q_ && e_ == o.e_ && m_ == o.m_; }

 private:
  std::vector<std::int64_t> m_;
  std::int64_t q_ = 1, e_ = 0;
};

struct QcompFlags {
  bool overflow = false;
  bool underflow = false;
  bool recomputed = false;
};
struct QcompResult {
  BfpBlock z;
  QcompFlags flags;
};
struct QcompOptions {
  bool force_recompute = false;
};

namespace detail {
// RAII device block
struct Dev {
  bfp_vec_t v = nullptr;
  Dev() = default;
  explicit Dev(const BfpBlock& b) {
    check(bfp_vec_create((std::int64_t)b.size(), 8, &v), "bfp_vec_create");
    const int st = bfp_vec_upload(v, b.mantissas().data(), b.q(), b.e(), nullptr);
    if (st) {
      bfp_vec_destroy(v);
      check(st, "bfp_vec_upload");
    }
  }
  explicit Dev(std::int64_t n) { check(bfp_vec_create(n, 8, &v), "bfp_vec_create"); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  ~Dev() {
    if (v) bfp_vec_destroy(v);
  }
  QcompResult get() const {
    std::vector<std::int64_t> m((std::size_t)bfp_vec_size(v));
    bfp_header_t h;
    check(bfp_vec_download(v, m.data(), &h, nullptr), "bfp_vec_download");
    if (h.err) check(h.err, "device");
    QcompResult r;
    r.z = BfpBlock::vec(std::move(m), h.q, h.e);
    r.flags = {bool(h.flags & BFP_FLAG_OVERFLOW), bool(h.flags & BFP_FLAG_UNDERFLOW),
               bool(h.flags & BFP_FLAG_RECOMPUTED)};
    return r;
  }
};
}  // namespace detail

/// CSR matrix with BFP values (P/include/bfpmg/bfp.hpp: BfpCsr), resident on the device.
class BfpCsr {
 public:
  BfpCsr(std::int64_t rows, std::int64_t cols, const std::vector<std::int64_t>& rowptr,
         const std::vector<std::int64_t>& col, const std::vector<std::int64_t>& m, std::int64_t q,
         std::int64_t e)
      : rows_(rows), cols_(cols) {
    if ((std::int64_t)rowptr.size() != rows + 1 || col.size() != m.size())
      throw std::invalid_argument("BfpCsr: layout");
    check(bfp_csr_create(rows, cols, rowptr.data(), col.data(), m.data(), q, e, &a_), "bfp_csr_create");
  }
  BfpCsr(const BfpCsr&) = delete;
  BfpCsr& operator=(const BfpCsr&) = delete;
  ~BfpCsr() {
    if (a_) bfp_csr_destroy(a_);
  }
  std::int64_t rows() const { return rows_; }
  std::int64_t cols() const { return cols_; }
  bfp_csr_t handle() const { return a_; }

 private:
  bfp_csr_t a_ = nullptr;
  std::int64_t rows_, cols_;
};

// ---- block operations (P/src/bfp.cpp:97-148) -----------------------------------------
inline BfpBlock normalize(const BfpBlock& x) {
  detail::Dev dx(x), out((std::int64_t)x.size());
  check(bfp_normalize(dx.v, out.v, nullptr), "normalize");
  return out.get().z;
}
inline BfpBlock quantize(const BfpBlock& x, std::int64_t w) {
  detail::Dev dx(x), out((std::int64_t)x.size());
  check(bfp_quantize(dx.v, w, out.v, nullptr), "quantize");
  return out.get().z;
}
inline BfpScalar inf_norm_upper(const BfpBlock& x, std::int64_t q_gamma = 16) {
  detail::Dev dx(x);
  BfpScalar s{0, 0, 0};
  check(bfp_inf_norm_upper(dx.v, q_gamma, &s.m, &s.q, &s.e, nullptr), "inf_norm_upper");
  return s;
}
inline std::string dump_block(const BfpBlock& x) {
  detail::Dev dx(x);
  const std::int64_t n = bfp_vec_dump(dx.v, nullptr, 0, nullptr);  // text size + NUL
  if (n < 0) check((int)-n, "dump_block");
  std::vector<char> buf((std::size_t)n);
  bfp_vec_dump(dx.v, buf.data(), n, nullptr);
  return std::string(buf.data(), (std::size_t)n - 1);
}
inline BfpBlock parse_block(const std::string& text) {
  detail::Dev d;
  check(bfp_vec_parse(text.c_str(), &d.v, nullptr), "parse_block");
  return d.get().z;
}

// ---- windowed BLAS (P/src/blas.cpp:214-256) ------------------------------------------
namespace detail {
inline QcompResult axpby(const BfpBlock& x, const BfpBlock& y, const BfpScalar& a,
                         const BfpScalar& b, int mode, std::int64_t w_out, std::int64_t w_tmp,
                         const BfpScalar& g, bool force) {
  if (x.size() != y.size()) throw std::invalid_argument("eaxpby: size mismatch");
  Dev dx(x), dy(y), out((std::int64_t)x.size());
  check(bfp_axpby(dx.v, dy.v, a.c(), b.c(), mode, w_out, w_tmp, g.c(), force, out.v, nullptr),
        "qaxpby");
  return out.get();
}
inline QcompResult spmv(const BfpCsr& A, const BfpBlock& x, int mode, std::int64_t w_out,
                        std::int64_t w_tmp, const BfpScalar& g, std::int64_t m_a, bool force) {
  Dev dx(x), out(A.rows());
  check(bfp_spmv_csr(A.handle(), dx.v, m_a, mode, w_out, w_tmp, g.c(), force, out.v, nullptr),
        "qspmv");
  return out.get();
}
inline QcompResult gemv(const BfpCsr& A, const BfpBlock& x, const BfpBlock& y, const BfpScalar& a,
                        const BfpScalar& b, int mode, std::int64_t w_out, std::int64_t w_tmp,
                        const BfpScalar& g, std::int64_t m_a, bool force) {
  Dev dx(x), dy(y), out(A.rows());
  check(bfp_gemv_csr(A.handle(), dx.v, dy.v, a.c(), b.c(), m_a, mode, w_out, w_tmp, g.c(), force,
                     out.v, nullptr),
        "qgemv");
  return out.get();
}
}  // namespace detail

inline QcompResult qaxpby(const BfpBlock& x, const BfpBlock& y, const BfpScalar& alpha,
                          const BfpScalar& beta, std::int64_t w_out, std::int64_t w_tmp,
                          const BfpScalar& gamma, const QcompOptions& opt = {}) {
  return detail::axpby(x, y, alpha, beta, 0, w_out, w_tmp, gamma, opt.force_recompute);
}
inline QcompResult qsub(const BfpBlock& x, const BfpBlock& y, std::int64_t w_out,
                        std::int64_t w_tmp, const BfpScalar& gamma) {
  return qaxpby(x, y, bfp_one(), bfp_minus_one(), w_out, w_tmp, gamma);
}
inline QcompResult qspmv(const BfpCsr& a, const BfpBlock& x, std::int64_t w_out,
                         std::int64_t w_tmp, const BfpScalar& gamma, std::int64_t m_a = 0,
                         const QcompOptions& opt = {}) {
  return detail::spmv(a, x, 0, w_out, w_tmp, gamma, m_a, opt.force_recompute);
}
inline QcompResult qgemv(const BfpCsr& a, const BfpBlock& x, const BfpBlock& y,
                         const BfpScalar& alpha, const BfpScalar& beta, std::int64_t w_out,
                         std::int64_t w_tmp, const BfpScalar& gamma, std::int64_t m_a = 0,
                         const QcompOptions& opt = {}) {
  return detail::gemv(a, x, y, alpha, beta, 0, w_out, w_tmp, gamma, m_a, opt.force_recompute);
}
inline QcompResult nnqaxpby(const BfpBlock& x, const BfpBlock& y, const BfpScalar& alpha,
                            const BfpScalar& beta, std::int64_t w_out, const BfpScalar& gamma) {
  return detail::axpby(x, y, alpha, beta, 1, w_out, w_out, gamma, false);
}
inline QcompResult nnqsub(const BfpBlock& x, const BfpBlock& y, std::int64_t w_out,
                          const BfpScalar& gamma) {
  return nnqaxpby(x, y, bfp_one(), bfp_minus_one(), w_out, gamma);
}
inline QcompResult nnqspmv(const BfpCsr& a, const BfpBlock& x, std::int64_t w_out,
                           const BfpScalar& gamma, std::int64_t m_a = 0) {
  return detail::spmv(a, x, 1, w_out, w_out, gamma, m_a, false);
}
inline QcompResult nnqgemv(const BfpCsr& a, const BfpBlock& x, const BfpBlock& y,
                           const BfpScalar& alpha, const BfpScalar& beta, std::int64_t w_out,
                           const BfpScalar& gamma, std::int64_t m_a = 0) {
  return detail::gemv(a, x, y, alpha, beta, 1, w_out, w_out, gamma, m_a, false);
}

/// The solver drivers (vcycle / ir / fmg, P/src/multigrid.cpp:430-518) stay on the device.
class Multigrid {
 public:
  explicit Multigrid(const bfp_mg_config_t& cfg) : cfg_(cfg) {
    check(bfp_mg_create(&cfg_, &mg_), "bfp_mg_create");
  }
  Multigrid(const Multigrid&) = delete;
  Multigrid& operator=(const Multigrid&) = delete;
  ~Multigrid() {
    if (mg_) bfp_mg_destroy(mg_);
  }
  void solve(bool use_graph = true, void* stream = nullptr) {
    check(bfp_mg_solve(mg_, use_graph, stream), "bfp_mg_solve");
  }
  /// final iterate and the residual-norm history
  std::pair<BfpBlock, std::vector<double>> result(void* stream = nullptr) {
    std::int64_t n = 1;
    for (int a = 0; a < cfg_.d; ++a) n *= (std::int64_t(1) << cfg_.l_fine) - 1;
    std::vector<std::int64_t> x((std::size_t)n);
    std::vector<double> hist(4096);
    bfp_header_t h;
    int nh = 0;
    std::int64_t nt = 0;
    check(bfp_mg_result(mg_, x.data(), &h, hist.data(), 4096, &nh, nullptr, 0, &nt, stream),
          "bfp_mg_result");
    hist.resize((std::size_t)nh);
    return {BfpBlock::vec(std::move(x), h.q, h.e), hist};
  }
  /// rhs_kind 3: write level `level`'s right-hand side as entries z_i 2^k_i, floor-quantised
  /// at w (the reference's quantize_vec of the D^-1-scaled load, P/src/multigrid.cpp:231)
  void set_level_rhs(int level, const std::vector<std::int64_t>& z,
                     const std::vector<std::int64_t>& k, std::int64_t w, void* stream = nullptr) {
    bfp_vec_t b = nullptr;
    check(bfp_mg_level_rhs(mg_, level, &b, nullptr), "bfp_mg_level_rhs");
    if (z.size() != k.size()) check(BFP_ERR_ARG, "set_level_rhs: size mismatch");
    check(bfp_quantize_exact(z.data(), k.data(), (std::int64_t)z.size(), w, b, stream),
          "bfp_quantize_exact");
  }

 private:
  bfp_mg_config_t cfg_;
  bfp_mg_t mg_ = nullptr;
};

}  // namespace bfpmg_b200
