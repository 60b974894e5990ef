// H1 peeling driver and device-resident H1 representation.
//
// API surface of proj/include/hpeel/peeling.hpp:15-77 and
// proj/include/hpeel/hmatrix.hpp:38-70 for the H1 hot path: PeelConfig,
// RunReport/PhaseReport, compress() -> PeelResult{H1Rep, RunReport}. The
// representation's factors stay in HBM (one arena per rep); host copies are
// produced on request (`export_*`).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "box_tree.hpp"
#include "coloring.hpp"
#include "matrix.hpp"

namespace hpeel {

inline constexpr double kQrRankDropTol = 1e-14;  // proj/include/hpeel/linalg.hpp:33
inline constexpr double kPinvCutoff = 1e-12;     // proj/include/hpeel/linalg.hpp:35

enum class PeelFormat : std::uint8_t { kH1 = 0, kUnifH1 = 1, kH1PlusUnif = 2, kH2 = 3 };
enum class ColoringStrategy : std::uint8_t { kGraph = 0, kFallbackPattern = 1 };

class Comm;  // shard.hpp

struct PeelConfig {
  int rank = 8;          // TruncationSpec::fixed_rank(k, p) (proj/src/linalg.cpp:24-31)
  int oversample = 10;
  int leaf_capacity = 64;
  std::uint64_t seed = 0;
  PeelFormat format = PeelFormat::kH1;
  ColoringStrategy strategy = ColoringStrategy::kGraph;
  bool capture_samples = false;  // keep post-peel sample blocks on the host (tests)
  Comm* comm = nullptr;          // multi-GPU: this process's rank in the NCCL group
  int emulate_shards = 0;        // tests: split K2/K6 launches as `n` ranks would
  // Streamed export: when set, every level's factor slice and the dense leaf
  // blocks are copied to these host arrays (export_sizes() doubles each, the
  // H1Rep::export_all layout) on a second stream as soon as they are final,
  // overlapping the later levels' device work (pinned memory; pageable
  // arrays are filled after the device loop).
  double* export_factors = nullptr;
  double* export_dense = nullptr;
  int sample_width() const { return rank + oversample; }
  void validate() const;
};

struct PhaseReport {
  std::string phase;
  int level = 0;
  int colors = 0;
  std::int64_t forward_cols = 0;
  std::int64_t adjoint_cols = 0;
  double wall_ms_total = 0.0;
  double wall_ms_net = 0.0;
  std::int64_t net_flops = 0;
  // device-side additions (not in the reference report)
  double apply_ms = 0.0;         // black-box (K2) device time
  double peel_ms = 0.0;          // K3
  double qr_ms = 0.0;            // K4
  double bsolve_ms = 0.0;        // K5 (incl. gram reductions)
  double apply_flops = 0.0;      // FMAs*2 executed by K2 on needed rows
  double peel_flops = 0.0;       // FMAs*2 executed by K3 (coefficients + subtraction)
  double qr_flops = 0.0;         // K4: 2 m r^2 per U and per V block (flops.hpp:18-20)
  double kernel_evals = 0.0;
  double host_wait_ms = 0.0;      // driver thread blocked on this phase's host plan
  double start_ms = 0.0;          // device time from the first device work of compress to this phase
  int apply_path = 0;             // K2 arithmetic: 0 FP64 DMMA, 1 int8 tensor-core emulation
};

struct RunReport {
  std::vector<PhaseReport> phases;
  std::int64_t forward_cols = 0;
  std::int64_t adjoint_cols = 0;
  int max_sampling_colors = 0;
  double wall_s_total = 0.0;
  double wall_s_net = 0.0;
  std::int64_t net_flops = 0;
  double setup_ms = 0.0;  // adjacency, layout, device operator staging, plan launch
  std::string to_csv() const;  // proj/src/peeling.cpp:478-488 columns
};

/// A black box behind the reference's LinearOperator plugin boundary
/// (proj/include/hpeel/linear_operator.hpp:12-24), resident on the device.
class DeviceOperator {
 public:
  static std::shared_ptr<DeviceOperator> dense(const Matrix& a, int device);
  static std::shared_ptr<DeviceOperator> kernel(int kind, const Matrix& raw_points, double param,
                                                int device);
  ~DeviceOperator();
  Index rows() const { return n_; }
  Index cols() const { return n_; }
  int kind() const { return kind_; }
  int dim() const { return dim_; }
  double param() const { return param_; }
  bool symmetric() const { return symmetric_; }
  const double* device_points() const { return d_x_; }  // dim x n, input order
  const double* device_matrix() const { return d_a_; }  // n x n col-major, input order
  /// Y = A X (or A^T X), host col-major n x w in and out.
  Matrix apply(const Matrix& x, bool adjoint) const;
  int device() const { return device_; }

 private:
  DeviceOperator() = default;
  int kind_ = 0;
  int dim_ = 1;
  Index n_ = 0;
  double param_ = 1.0;
  bool symmetric_ = true;
  int device_ = 0;
  double* d_x_ = nullptr;
  double* d_a_ = nullptr;
};

struct LowRankBlockHost {
  Matrix u, b, v;
};

/// Device-resident H1 representation (proj/include/hpeel/hmatrix.hpp:52-70).
class H1Rep {
 public:
  struct LevelData {
    std::vector<std::pair<int, int>> pairs;  // admissible_pairs order
    std::vector<std::int64_t> uoff, voff, boff;
    std::vector<int> ku, kv;                 // retained ranks
  };
  struct DenseData {
    std::vector<std::pair<int, int>> pairs;  // dense_pairs order
    std::vector<std::int64_t> off;           // leading |I_lam| x |I_mu| of each block
  };

  std::shared_ptr<const BoxTree> tree;
  std::shared_ptr<const AdjacencyInfo> adj;
  std::shared_ptr<const TreeLayout> layout;
  int rank = 0;
  int built_level = 1;
  bool dense_ready = false;
  std::vector<LevelData> levels;  // indexed by level
  DenseData dense;
  int device = 0;
  double* d_factors = nullptr;  // U, V, B blocks of all levels
  double* d_dense = nullptr;
  std::int64_t factor_doubles = 0;
  std::int64_t dense_doubles = 0;
  // captured post-peel samples (capture_samples): level -> pair -> [Y | Z]
  std::map<int, std::vector<Matrix>> captured;
  std::vector<Matrix> captured_leaf;

  H1Rep() = default;
  H1Rep(const H1Rep&) = delete;
  H1Rep& operator=(const H1Rep&) = delete;
  ~H1Rep();

  /// proj/src/hmatrix.cpp:118-130 on the device; host in/out, input order.
  Matrix apply(const Matrix& x, bool adjoint) const;
  /// Device version: x, y tree order row-major n x w.
  void apply_device(const double* x_tree, int w, bool adjoint, double* y_tree,
                    cudaStream_t s) const;
  /// Host copy of one admissible block, rows in box.points order.
  LowRankBlockHost block(int level, int pair_index) const;
  Matrix dense_block(int pair_index) const;
  /// Stored scalars (proj/src/hmatrix.cpp:132-150): U, V, B and dense totals.
  std::int64_t storage_total() const;
  /// Copy every factor and dense block to pinned host memory (e2e export).
  std::int64_t export_all(double* host_factors, double* host_dense) const;
};

struct PeelResult {
  std::shared_ptr<H1Rep> rep;
  RunReport report;
};

/// proj/src/peeling.cpp:576-639 for format h1 (others: std::invalid_argument).
PeelResult compress(const DeviceOperator& op, std::shared_ptr<const BoxTree> tree,
                    const PeelConfig& config);

/// Doubles of the factor arena and of the dense leaf blocks compress() will
/// produce for this tree and rank (the export_all / export_* layout sizes).
void export_sizes(const BoxTree& tree, int rank, std::int64_t* factor_doubles,
                  std::int64_t* dense_doubles);

/// proj/src/linalg.cpp:206-218 with both operators applied on the device.
double rel_error_power_method(const H1Rep& rep, const DeviceOperator& op, int iters,
                              std::uint64_t seed);

}  // namespace hpeel
