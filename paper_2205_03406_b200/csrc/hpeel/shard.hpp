// Multi-GPU sharding of the peeling hot path.
//
// One process per GPU, owner-computes. The points are cut into `world`
// contiguous tree-order ranges at a frontier of boxes (every box at the cut
// level plus the leaves above it), balanced by point count. A box at or below
// the frontier belongs to exactly one rank; the boxes above it span ranks.
//
//  * H1 levels at or below the cut ("owned" levels): rank g computes the
//    samples, U and B of the pairs (a, b) whose row box a it owns, and V of
//    the pairs whose column box it owns. It keeps the factors of every pair
//    touching its boxes; a pair whose two boxes live on different ranks
//    ("cut-crossing") is held by both, which is all the peeling of later
//    levels needs. Two point-to-point exchanges per level: V of crossing
//    pairs to the row owner (for the B solve), then U and B back to the
//    column owner (for its adjoint peeling).
//  * Levels above the cut ("replicated" levels, few pairs): the black-box
//    apply and the per-pair QR / B solves are split by work-balanced pair
//    ranges and their rows / factors broadcast, so every rank holds them.
//  * Leaf phase: the dense blocks of leaf lambda live on lambda's owner.
//
// Communication goes through `Comm`: NcclComm (NCCL over NVLink, loaded at
// run time) for one process per GPU, LocalComm for a group of ranks emulated
// by threads of one process (tests; stream-ordered device copies between the
// ranks' buffers, host barriers only -- no kernel ever waits on another).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace hpeel {

class BoxTree;
struct TreeLayout;

/// Contiguous ranges [b[r], b[r+1]) of items 0..n-1 for `world` ranks,
/// balancing the prefix sums of `work` (deterministic on every rank).
std::vector<std::int64_t> partition_ranges(const std::vector<double>& work, int world);

/// Box ownership for `world` ranks (see the header comment).
struct Ownership {
  int world = 1;
  int rank = 0;
  int cut = 0;                 // levels < cut are replicated (world > 1 only)
  std::vector<int> owner;      // per box: owning rank, -1 above the frontier
  std::vector<std::int64_t> point_bounds;  // rank g owns tree positions [b[g], b[g+1])
  bool replicated(int level) const { return world > 1 && level < cut; }
  int of(int box) const { return owner[size_t(box)]; }
  bool mine(int box) const { return owner[size_t(box)] == rank; }
};
Ownership make_ownership(const BoxTree& tree, const TreeLayout& lay, int world, int rank);

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  virtual int device() const = 0;
  /// In place: rank r's segment [off[r], off[r+1]) of `buf` reaches every rank.
  virtual void broadcast_segments(double* buf, const std::vector<std::int64_t>& off, cudaStream_t s) = 0;
  virtual void broadcast_segments_i32(int* buf, const std::vector<std::int64_t>& off, cudaStream_t s) = 0;
  /// All-to-all-v: send[soff[j], soff[j+1]) goes to rank j, and
  /// recv[roff[i], roff[i+1]) arrives from rank i (i, j != rank; element
  /// counts must agree pairwise). Stream-ordered on s.
  virtual void exchange(const double* send, const std::vector<std::int64_t>& soff, double* recv,
                        const std::vector<std::int64_t>& roff, cudaStream_t s) = 0;
  virtual void exchange_i32(const int* send, const std::vector<std::int64_t>& soff, int* recv,
                            const std::vector<std::int64_t>& roff, cudaStream_t s) = 0;
};

/// NCCL communicator (one process per GPU).
class NcclComm final : public Comm {
 public:
  /// NCCL unique id (128 bytes) for rank 0 to distribute.
  static void unique_id(unsigned char out[128]);
  NcclComm(const unsigned char id[128], int rank, int world, int device);
  ~NcclComm() override;
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  int device() const override { return device_; }
  void broadcast_segments(double* buf, const std::vector<std::int64_t>& off, cudaStream_t s) override;
  void broadcast_segments_i32(int* buf, const std::vector<std::int64_t>& off, cudaStream_t s) override;
  void exchange(const double* send, const std::vector<std::int64_t>& soff, double* recv,
                const std::vector<std::int64_t>& roff, cudaStream_t s) override;
  void exchange_i32(const int* send, const std::vector<std::int64_t>& soff, int* recv,
                    const std::vector<std::int64_t>& roff, cudaStream_t s) override;

 private:
  void bcast(void* buf, const std::vector<std::int64_t>& off, int type, size_t elem, cudaStream_t s);
  void a2av(const void* send, const std::vector<std::int64_t>& soff, void* recv,
            const std::vector<std::int64_t>& roff, int type, size_t elem, cudaStream_t s);
  int rank_ = 0, world_ = 1, device_ = 0;
  void* comm_ = nullptr;  // ncclComm_t
};

/// Shared state of `world` ranks emulated by threads of one process on one
/// device. Any rank that fails aborts the group: peers blocked in a
/// collective then throw instead of waiting forever.
class LocalGroup {
 public:
  explicit LocalGroup(int world);
  int world() const { return world_; }
  void abort();
  // collective rendezvous: every rank publishes (ptr, offsets, event)
  struct Slot {
    const void* ptr = nullptr;
    std::vector<std::int64_t> off;
    cudaEvent_t ready = nullptr;  // the source is complete on its owner's stream
    cudaEvent_t done = nullptr;   // the owner's copies out of its peers are issued/complete
  };
  void barrier();
  Slot& slot(int r) { return slots_[size_t(r)]; }

 private:
  int world_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  std::uint64_t generation_ = 0;
  bool aborted_ = false;
  std::vector<Slot> slots_;
};

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> group, int rank, int device);
  ~LocalComm() override;
  int rank() const override { return rank_; }
  int world() const override { return group_->world(); }
  int device() const override { return device_; }
  void broadcast_segments(double* buf, const std::vector<std::int64_t>& off, cudaStream_t s) override;
  void broadcast_segments_i32(int* buf, const std::vector<std::int64_t>& off, cudaStream_t s) override;
  void exchange(const double* send, const std::vector<std::int64_t>& soff, double* recv,
                const std::vector<std::int64_t>& roff, cudaStream_t s) override;
  void exchange_i32(const int* send, const std::vector<std::int64_t>& soff, int* recv,
                    const std::vector<std::int64_t>& roff, cudaStream_t s) override;
  LocalGroup& group() { return *group_; }

 private:
  void bcast(void* buf, const std::vector<std::int64_t>& off, size_t elem, cudaStream_t s);
  void a2av(const void* send, const std::vector<std::int64_t>& soff, void* recv,
            const std::vector<std::int64_t>& roff, size_t elem, cudaStream_t s);
  // publish, rendezvous, copy from the peers, then keep every peer's source
  // alive (its stream waits for our copies) before the slots are reused
  std::shared_ptr<LocalGroup> group_;
  int rank_, device_;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
};

}  // namespace hpeel
