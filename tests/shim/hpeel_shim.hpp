// C++ drop-in shim over the hpeel_b200 C ABI with the reference's API surface
// for the H1 hot path (proj/include/hpeel/linear_operator.hpp:12-24,
// proj/include/hpeel/box_tree.hpp:61-85, proj/include/hpeel/peeling.hpp:27-77):
// a user-derived LinearOperator is handed to the GPU driver through
// hp_op_callback, compress() returns PeelResult{H1Rep, RunReport}, and C ABI
// status codes come back as the reference's exception types. Eigen is not
// available here, so Matrix is a small column-major stand-in with the same
// (rows, cols, operator()(i, j)) surface.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hpeel_b200.h"

namespace hpeel_shim {

using Index = std::int64_t;

class Matrix {
 public:
  Matrix() = default;
  Matrix(Index r, Index c) : rows_(r), cols_(c), data_(size_t(r * c), 0.0) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  double& operator()(Index i, Index j) { return data_[size_t(i + j * rows_)]; }
  double operator()(Index i, Index j) const { return data_[size_t(i + j * rows_)]; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

inline void check(int rc) {
  if (rc == HP_OK) return;
  const std::string msg = hp_last_error();
  if (rc == HP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == HP_ERR_LOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

/// proj/include/hpeel/linear_operator.hpp:12-24
class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  virtual Matrix apply(const Matrix& x) const = 0;
  virtual Matrix apply_adjoint(const Matrix& x) const = 0;
  virtual bool reentrant() const { return true; }
};

/// proj/include/hpeel/linalg.hpp TruncationSpec (fixed rank only on this path)
struct TruncationSpec {
  int rank = 8;
  int oversample = 10;
  static TruncationSpec fixed_rank(int k, int p) { return TruncationSpec{k, p}; }
};

enum class PeelFormat { kH1 = HP_FORMAT_H1, kUnifH1 = HP_FORMAT_UNIF_H1, kH1PlusUnif = HP_FORMAT_H1_PLUS_UNIF,
                        kH2 = HP_FORMAT_H2 };
enum class ColoringStrategy { kGraph = HP_STRATEGY_GRAPH, kFallbackPattern = HP_STRATEGY_FALLBACK_PATTERN };

/// proj/include/hpeel/peeling.hpp:27-34
struct PeelConfig {
  TruncationSpec trunc;
  std::uint64_t seed = 0;
  PeelFormat format = PeelFormat::kH1;
  ColoringStrategy strategy = ColoringStrategy::kGraph;
};

/// BoxTree::build + adjacency (proj/include/hpeel/box_tree.hpp:61-85); raw
/// points n x d column-major.
class BoxTree {
 public:
  static std::shared_ptr<const BoxTree> build(const Matrix& raw, int leaf_capacity) {
    hp_tree* t = nullptr;
    check(hp_tree_build(raw.data(), raw.rows(), int(raw.cols()), leaf_capacity, &t));
    return std::shared_ptr<const BoxTree>(new BoxTree(t));
  }
  ~BoxTree() { hp_tree_free(h_); }
  BoxTree(const BoxTree&) = delete;
  BoxTree& operator=(const BoxTree&) = delete;
  Index num_points() const { return info(0); }
  int depth() const { return int(info(2)); }
  std::vector<std::pair<int, int>> admissible_pairs(int level) const { return pairs(level); }
  std::vector<std::pair<int, int>> dense_pairs() const { return pairs(-1); }
  hp_tree* handle() const { return h_; }

 private:
  explicit BoxTree(hp_tree* h) : h_(h) {}
  Index info(int i) const {
    std::int64_t v[8];
    check(hp_tree_info(h_, v));
    return v[i];
  }
  std::vector<std::pair<int, int>> pairs(int level) const {
    std::int64_t n = 0;
    check(hp_tree_pairs(h_, level, &n, nullptr));
    std::vector<int> flat(size_t(2 * n) + 2);
    check(hp_tree_pairs(h_, level, &n, flat.data()));
    std::vector<std::pair<int, int>> out;
    for (std::int64_t i = 0; i < n; ++i) out.emplace_back(flat[size_t(2 * i)], flat[size_t(2 * i + 1)]);
    return out;
  }
  hp_tree* h_;
};

struct LowRankBlock {
  Matrix u, b, v;
};

/// proj/include/hpeel/hmatrix.hpp:52-70, factors resident on the device.
class H1Rep {
 public:
  explicit H1Rep(hp_rep* h) : h_(h) {}
  ~H1Rep() { hp_rep_free(h_); }
  H1Rep(const H1Rep&) = delete;
  H1Rep& operator=(const H1Rep&) = delete;
  LowRankBlock block(int level, std::int64_t pair, Index rows_a, Index rows_b) const {
    int ku = 0, kv = 0;
    check(hp_rep_block(h_, level, pair, &ku, &kv, nullptr, nullptr, nullptr));
    LowRankBlock blk{Matrix(rows_a, ku), Matrix(ku, kv), Matrix(rows_b, kv)};
    check(hp_rep_block(h_, level, pair, &ku, &kv, blk.u.data(), blk.b.data(), blk.v.data()));
    return blk;
  }
  Matrix apply(const Matrix& x) const {
    Matrix y(x.rows(), x.cols());
    check(hp_rep_apply(h_, 0, x.data(), x.cols(), y.data()));
    return y;
  }
  hp_rep* handle() const { return h_; }

 private:
  hp_rep* h_;
};

/// proj/include/hpeel/peeling.hpp:36-57 (totals and the CSV of to_csv)
struct RunReport {
  std::int64_t forward_cols = 0, adjoint_cols = 0;
  int max_sampling_colors = 0;
  double wall_s_total = 0.0, wall_s_net = 0.0;
  std::string csv;
};

struct PeelResult {
  std::shared_ptr<H1Rep> rep;
  RunReport report;
};

namespace detail {
// hp_apply_fn trampoline: the reference's call pattern (host matrices in and out)
inline int apply_host(void* ctx, int adjoint, const double* x, std::int64_t w, double* y, void*) {
  try {
    const auto* op = static_cast<const LinearOperator*>(ctx);
    Matrix xm(op->rows(), w);
    std::copy(x, x + op->rows() * w, xm.data());
    const Matrix ym = adjoint ? op->apply_adjoint(xm) : op->apply(xm);
    if (ym.rows() != op->rows() || ym.cols() != w) return 2;
    std::copy(ym.data(), ym.data() + ym.rows() * ym.cols(), y);
    return 0;
  } catch (...) {
    return 1;
  }
}
}  // namespace detail

/// proj/include/hpeel/peeling.hpp:66-68 on device `device`
inline PeelResult compress(const LinearOperator& op, std::shared_ptr<const BoxTree> tree, const PeelConfig& cfg,
                           int device = 0) {
  if (!tree) throw std::invalid_argument("null tree");
  if (op.rows() != op.cols() || op.rows() != tree->num_points())
    throw std::invalid_argument("operator and tree dimensions differ");
  hp_op* h = nullptr;
  check(hp_op_callback(op.rows(), 0, 0, &detail::apply_host, const_cast<LinearOperator*>(&op), device, &h));
  std::unique_ptr<hp_op, void (*)(hp_op*)> guard(h, hp_op_free);
  hp_rep* rep = nullptr;
  check(hp_compress(h, tree->handle(), cfg.trunc.rank, cfg.trunc.oversample, cfg.seed, int(cfg.format),
                    int(cfg.strategy), 0, &rep));
  PeelResult out;
  out.rep = std::make_shared<H1Rep>(rep);
  double totals[9] = {0};
  std::int64_t nph = 0;
  check(hp_rep_report(rep, totals, &nph));
  out.report.forward_cols = std::int64_t(totals[0]);
  out.report.adjoint_cols = std::int64_t(totals[1]);
  out.report.max_sampling_colors = int(totals[2]);
  out.report.wall_s_total = totals[3];
  out.report.wall_s_net = totals[4];
  std::int64_t len = 0;
  check(hp_rep_csv(rep, nullptr, 0, &len));
  std::string csv(size_t(len) + 1, '\0');
  check(hp_rep_csv(rep, &csv[0], len + 1, &len));
  csv.resize(size_t(len));
  out.report.csv = csv;
  return out;
}

}  // namespace hpeel_shim
