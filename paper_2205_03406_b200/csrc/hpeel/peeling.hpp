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
  Comm* comm = nullptr;          // multi-GPU: this rank's communicator (NCCL, or an emulated group)
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
  double bsolve_flops = 0.0;     // K5: reference B-solve formulas (peeling.cpp:262-264, linalg.cpp:116-117)
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
  double peak_device_bytes = 0.0;  // high-water of the buffers compress() allocated (this rank)
  double exchange_bytes = 0.0;     // bytes this rank sent in sharded exchanges / broadcasts
  std::string to_csv() const;  // proj/src/peeling.cpp:478-488 columns
};

/// Caller-supplied black box (the reference's virtual LinearOperator::apply /
/// apply_adjoint, proj/include/hpeel/linear_operator.hpp:19-20): Y = A X or
/// A^T X for an n x w column-major X in the caller's point order. Host
/// variant: x / y are host arrays and stream is null; device variant: x / y
/// are device pointers on the operator's device and the work must be ordered
/// on `stream` (a cudaStream_t). Nonzero return = failure.
using ApplyFn = int (*)(void* ctx, int adjoint, const double* x, std::int64_t w, double* y, void* stream);

/// A black box behind the reference's LinearOperator plugin boundary
/// (proj/include/hpeel/linear_operator.hpp:12-24), resident on the device.
class DeviceOperator {
 public:
  static std::shared_ptr<DeviceOperator> dense(const Matrix& a, int device);
  static std::shared_ptr<DeviceOperator> kernel(int kind, const Matrix& raw_points, double param,
                                                int device);
  static std::shared_ptr<DeviceOperator> callback(Index n, bool symmetric, bool device_pointers, ApplyFn fn,
                                                  void* ctx, int device);
  bool is_callback() const { return fn_ != nullptr; }
  /// Callback black box on device buffers (input order, n x w col-major),
  /// ordered on s; the host variant stages through pinned host memory.
  void call(bool adjoint, const double* d_x, std::int64_t w, double* d_y, cudaStream_t s) const;
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
  ApplyFn fn_ = nullptr;
  void* ctx_ = nullptr;
  bool device_pointers_ = false;
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
  // owner-computes sharding (shard.hpp): this rank holds the factors of the
  // pairs with uoff >= 0 and the dense blocks with off >= 0
  int world = 1;
  int shard_rank = 0;
  std::vector<int> box_owner;   // per box (-1 above the cut); empty = unsharded
  double* d_factors = nullptr;  // U, V, B blocks of all levels
  double* d_dense = nullptr;
  std::int64_t factor_doubles = 0;
  std::int64_t dense_doubles = 0;
  // captured post-peel samples (capture_samples): level -> pair -> [Y | Z]
  std::map<int, std::vector<Matrix>> captured;
  std::map<int, std::vector<Matrix>> captured_raw;  // the same blocks before peeling (= A Omega rows)
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
  bool sharded() const { return world > 1; }
  bool holds(int level, int pair) const { return levels.at(size_t(level)).uoff.at(size_t(pair)) >= 0; }
  bool holds_dense(int pair) const { return dense.off.at(size_t(pair)) >= 0; }
  /// the rank that computed U and B of the pair (its row box's owner) counts it
  bool counts_pair(int level, int pair) const {
    const auto& ld = levels[size_t(level)];
    if (ld.uoff[size_t(pair)] < 0) return false;
    if (box_owner.empty()) return true;
    const int o = box_owner[size_t(ld.pairs[size_t(pair)].first)];
    return o < 0 ? shard_rank == 0 : o == shard_rank;
  }
};

struct PeelResult {
  std::shared_ptr<H1Rep> rep;
  RunReport report;
};

/// proj/src/peeling.cpp:576-639 for format h1 (others: std::invalid_argument).
PeelResult compress(const DeviceOperator& op, std::shared_ptr<const BoxTree> tree,
                    const PeelConfig& config);

/// Doubles of the factor arena and of the dense leaf blocks compress() will
/// produce for this tree and rank (the export_all / export_* layout sizes);
/// with world > 1, of shard `shard` (owner-computes layout, shard.hpp).
void export_sizes(const BoxTree& tree, int rank, std::int64_t* factor_doubles,
                  std::int64_t* dense_doubles, int world = 1, int shard = 0);

/// compress() on `world` ranks emulated by threads of this process on the
/// operator's device (LocalComm): one representation per rank.
std::vector<PeelResult> compress_group(const DeviceOperator& op, std::shared_ptr<const BoxTree> tree,
                                       const PeelConfig& config, int world);

/// Per-rank device memory plan of an owner-computes compress (bytes):
/// out[g * 4 + 0..3] = factors held, dense blocks, largest level's samples
/// plus its apply buffers, total estimate.
void shard_memory_plan(const BoxTree& tree, int rank, int oversample, int world, double* out);

/// Doubles shard `shard` sends to / receives from each rank in the level's
/// crossing-pair exchange `phase` (1: V to the row owner, 2: U and B to the
/// column owner); zero on replicated levels.
void shard_exchange_counts(const BoxTree& tree, int rank, int world, int shard, int level, int phase,
                           std::int64_t* send, std::int64_t* recv);

/// proj/src/linalg.cpp:206-218 with both operators applied on the device.
double rel_error_power_method(const H1Rep& rep, const DeviceOperator& op, int iters,
                              std::uint64_t seed);

}  // namespace hpeel
