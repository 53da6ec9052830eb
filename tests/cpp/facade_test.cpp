// facade_test.cpp -- exercises include/bfpmg_b200.hpp (the reference-named C++ facade) on the
// GPU and prints the results as JSON lines; tests/test_gpu_facade.py compares them with the
// oracle.  Cases follow the reference's own tests (P/tests/test_blas.cpp: hand-derived
// eaxpby rows, qsub(x, x) = 0, qspmv(I, x) = normalize(x), exception types).
#include <cstdio>
#include <string>

#include "bfpmg_b200.hpp"

using namespace bfpmg_b200;

static void print_block(const char* name, const QcompResult& r) {
  std::printf("{\"name\": \"%s\", \"q\": %lld, \"e\": %lld, \"m\": [", name, (long long)r.z.q(),
              (long long)r.z.e());
  for (std::size_t i = 0; i < r.z.size(); ++i)
    std::printf("%s%lld", i ? ", " : "", (long long)r.z.mant(i));
  std::printf("], \"flags\": [%d, %d, %d]}\n", (int)r.flags.overflow, (int)r.flags.underflow,
              (int)r.flags.recomputed);
}

int main() {
  const BfpBlock x = BfpBlock::vec({5, -3, 7, 0, 2, -8, 1, 6}, 5, -2);
  const BfpBlock y = BfpBlock::vec({1, 4, -2, 3, -7, 0, 5, -1}, 4, 1);
  const BfpScalar a{3, 3, 0}, b{-2, 3, -1}, g{1 << 14, 16, -6};
  print_block("qaxpby", qaxpby(x, y, a, b, 8, 12, g));
  print_block("qaxpby_forced", qaxpby(x, y, a, b, 8, 12, g, QcompOptions{true}));
  print_block("qaxpby_overflow", qaxpby(x, y, a, b, 8, 12, BfpScalar{1 << 14, 16, -20}));
  print_block("nnqaxpby", nnqaxpby(x, y, a, b, 6, BfpScalar{1 << 14, 16, -9}));
  print_block("qsub_xx", qsub(x, x, 8, 12, g));
  // identity matrix: qspmv(I, x) = normalize(x) at width 5
  std::vector<std::int64_t> rp(9), col(8), one(8, 1);
  for (int i = 0; i < 8; ++i) rp[i] = col[i] = i;
  rp[8] = 8;
  const BfpCsr I(8, 8, rp, col, one, 2, 0);
  print_block("qspmv_I", qspmv(I, x, 5, 9, BfpScalar{1 << 14, 16, -11}));
  QcompResult n;
  n.z = normalize(x);
  print_block("normalize", n);
  n.z = quantize(x, 3);
  print_block("quantize3", n);
  // tridiagonal (-1, 2, -1): qgemv(A, x, y, -1, +1) = y - A x
  std::vector<std::int64_t> trp{0}, tcol, tm;
  for (int i = 0; i < 8; ++i) {
    if (i > 0) tcol.push_back(i - 1), tm.push_back(-1);
    tcol.push_back(i), tm.push_back(2);
    if (i < 7) tcol.push_back(i + 1), tm.push_back(-1);
    trp.push_back((std::int64_t)tcol.size());
  }
  const BfpCsr A(8, 8, trp, tcol, tm, 3, 2);
  print_block("qgemv", qgemv(A, x, y, bfp_minus_one(), bfp_one(), 10, 14, BfpScalar{1 << 14, 16, -7}));
  print_block("nnqgemv", nnqgemv(A, x, y, bfp_minus_one(), bfp_one(), 7, BfpScalar{1 << 14, 16, -7}));
  const BfpScalar nu = inf_norm_upper(x);
  std::printf("{\"name\": \"inf_norm_upper\", \"m\": %lld, \"q\": %lld, \"e\": %lld}\n",
              (long long)nu.m, (long long)nu.q, (long long)nu.e);
  const std::string text = dump_block(x);
  std::printf("{\"name\": \"dump_roundtrip\", \"ok\": %d}\n", (int)(parse_block(text) == x));
  // exception types (P/tests/test_bfp.cpp, test_blas.cpp): domain_error for a mantissa outside
  // T_q, invalid_argument for a bad window / mismatched sizes
  int domain = 0, invalid = 0, invalid2 = 0;
  try {
    BfpBlock::vec({16}, 5, 0);
  } catch (const std::domain_error&) {
    domain = 1;
  }
  try {
    qaxpby(x, y, a, b, 12, 8, g);  // w_tmp < w_out
  } catch (const std::invalid_argument&) {
    invalid = 1;
  }
  try {
    qsub(x, BfpBlock::vec({1, 2}, 3, 0), 8, 12, g);
  } catch (const std::invalid_argument&) {
    invalid2 = 1;
  }
  std::printf("{\"name\": \"exceptions\", \"domain\": %d, \"invalid\": %d, \"invalid2\": %d}\n", domain,
              invalid, invalid2);
  return 0;
}
