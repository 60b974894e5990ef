// Column-major FP64 host matrix. Stands in for Eigen::MatrixXd, which the
// reference uses throughout (proj/include/hpeel/rng.hpp:9): same rows()/cols()
// semantics, element (i, j) at data[i + j * rows].
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

namespace hpeel {

using Index = std::int64_t;

class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : rows_(rows), cols_(cols), data_(size_t(rows * cols), 0.0) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("negative shape");
  }
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  static Matrix Identity(Index rows, Index cols) {
    Matrix m(rows, cols);
    for (Index i = 0; i < std::min(rows, cols); ++i) m(i, i) = 1.0;
    return m;
  }

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  double& operator()(Index i, Index j) { return data_[size_t(i + j * rows_)]; }
  double operator()(Index i, Index j) const { return data_[size_t(i + j * rows_)]; }

 private:
  Index rows_ = 0;
  Index cols_ = 0;
  std::vector<double> data_;
};

}  // namespace hpeel
