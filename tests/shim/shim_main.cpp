// Drop-in check of the C++ shim (hpeel_shim.hpp): reference-style user code --
// a LinearOperator subclass wrapped in a column-counting decorator, the way
// proj/src/operators.cpp:320-342 counts -- compressed on the GPU through the
// callback boundary. Prints one JSON line. Built by tests/test_shim.py with
//   g++ -std=c++17 -O2 -I include tests/shim/shim_main.cpp -L<pkg> -lhpeel_b200
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "hpeel_shim.hpp"

using hpeel_shim::Index;
using hpeel_shim::Matrix;

// DenseOperator (proj/include/hpeel/operators.hpp:56-69): explicit matrix
class DenseOperator final : public hpeel_shim::LinearOperator {
 public:
  explicit DenseOperator(Matrix a) : a_(std::move(a)) {}
  Index rows() const override { return a_.rows(); }
  Index cols() const override { return a_.cols(); }
  Matrix apply(const Matrix& x) const override { return mul(x, false); }
  Matrix apply_adjoint(const Matrix& x) const override { return mul(x, true); }

 private:
  Matrix mul(const Matrix& x, bool trans) const {
    const Index n = a_.rows();
    Matrix y(n, x.cols());
    for (Index c = 0; c < x.cols(); ++c)
      for (Index j = 0; j < n; ++j) {
        const double xv = x(j, c);
        if (xv == 0.0) continue;  // test matrices are block-sparse
        if (!trans)
          for (Index i = 0; i < n; ++i) y(i, c) += a_(i, j) * xv;
        else
          for (Index i = 0; i < n; ++i) y(i, c) += a_(j, i) * xv;
      }
    return y;
  }
  Matrix a_;
};

// CountingOperator (proj/include/hpeel/operators.hpp:124-149)
class CountingOperator final : public hpeel_shim::LinearOperator {
 public:
  explicit CountingOperator(const LinearOperator& inner) : inner_(inner) {}
  Index rows() const override { return inner_.rows(); }
  Index cols() const override { return inner_.cols(); }
  Matrix apply(const Matrix& x) const override {
    std::lock_guard<std::mutex> lock(mu_);
    fwd_ += x.cols();
    ++calls_;
    return inner_.apply(x);
  }
  Matrix apply_adjoint(const Matrix& x) const override {
    std::lock_guard<std::mutex> lock(mu_);
    adj_ += x.cols();
    ++calls_;
    return inner_.apply_adjoint(x);
  }
  Index fwd() const { return fwd_; }
  Index adj() const { return adj_; }
  Index calls() const { return calls_; }

 private:
  const LinearOperator& inner_;
  mutable std::mutex mu_;
  mutable Index fwd_ = 0, adj_ = 0, calls_ = 0;
};

int main(int argc, char** argv) {
  const Index n = argc > 1 ? std::atol(argv[1]) : 1024;
  Matrix pts(n, 1);
  for (Index i = 0; i < n; ++i) pts(i, 0) = (double(i) + 0.5) / double(n);
  // A_ij = log|x_i - x_j|, A_ii = 0 (BASELINE config 1 kernel)
  Matrix a(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) a(i, j) = i == j ? 0.0 : std::log(std::fabs(pts(i, 0) - pts(j, 0)));
  DenseOperator dense(a);
  CountingOperator counted(dense);
  auto tree = hpeel_shim::BoxTree::build(pts, 64);
  hpeel_shim::PeelConfig cfg;
  cfg.trunc = hpeel_shim::TruncationSpec::fixed_rank(20, 10);
  cfg.seed = 7;
  const auto res = hpeel_shim::compress(counted, tree, cfg);
  // relative error of the representation on a few random vectors
  Matrix x(n, 3);
  std::uint64_t z = 12345;
  for (Index i = 0; i < n * 3; ++i) {
    z = z * 6364136223846793005ULL + 1442695040888963407ULL;
    x.data()[i] = double(z >> 11) * 0x1.0p-53 - 0.5;
  }
  const Matrix ya = dense.apply(x), yr = res.rep->apply(x);
  double num = 0, den = 0;
  for (Index i = 0; i < n * 3; ++i) {
    num += (ya.data()[i] - yr.data()[i]) * (ya.data()[i] - yr.data()[i]);
    den += ya.data()[i] * ya.data()[i];
  }
  // the reference's exception types across the boundary
  bool threw_invalid = false;
  try {
    DenseOperator small(Matrix(n - 1, n - 1));
    hpeel_shim::compress(small, tree, cfg);
  } catch (const std::invalid_argument&) {
    threw_invalid = true;
  }
  std::printf(
      "{\"n\": %ld, \"depth\": %d, \"report_forward_cols\": %ld, \"report_adjoint_cols\": %ld, "
      "\"counted_forward_cols\": %ld, \"counted_adjoint_cols\": %ld, \"calls\": %ld, \"rel_error\": %.3e, "
      "\"csv_lines\": %d, \"threw_invalid_argument\": %s}\n",
      long(n), tree->depth(), long(res.report.forward_cols), long(res.report.adjoint_cols), long(counted.fwd()),
      long(counted.adj()), long(counted.calls()), std::sqrt(num / den),
      int(std::count(res.report.csv.begin(), res.report.csv.end(), '\n')), threw_invalid ? "true" : "false");
  return 0;
}
