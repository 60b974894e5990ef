// Multi-GPU sharding of the peeling hot path.
//
// One process per GPU. Every rank builds the same (deterministic) host plan;
// the black-box apply (K2) and the leaf probes (K6) -- the dominant work --
// are split into contiguous, work-balanced ranges of pairs, and each rank's
// freshly computed sample rows are broadcast to the others with NCCL over
// NVLink before the (replicated, deterministic) peeling; the per-pair QR and
// B solves (K4/K5) are split by pair ranges as well and their factor and
// rank segments broadcast.
// NCCL is loaded at run time (libnccl.so.2; the torch-bundled copy when torch
// already loaded it), so single-GPU use has no NCCL dependency.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace hpeel {

/// Contiguous ranges [b[r], b[r+1]) of items 0..n-1 for `world` ranks,
/// balancing the prefix sums of `work` (deterministic on every rank).
std::vector<std::int64_t> partition_ranges(const std::vector<double>& work, int world);

class Comm {
 public:
  /// NCCL unique id (128 bytes) for rank 0 to distribute.
  static void unique_id(unsigned char out[128]);
  Comm(const unsigned char id[128], int rank, int world, int device);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  int rank() const { return rank_; }
  int world() const { return world_; }
  int device() const { return device_; }
  /// In place: rank r's segment [off[r], off[r+1]) of `buf` reaches every rank.
  void broadcast_segments(double* buf, const std::vector<std::int64_t>& off, cudaStream_t s);
  void broadcast_segments_i32(int* buf, const std::vector<std::int64_t>& off, cudaStream_t s);
  void all_reduce_max(double* dev_value, cudaStream_t s);

 private:
  int rank_ = 0, world_ = 1, device_ = 0;
  void* comm_ = nullptr;  // ncclComm_t
};

}  // namespace hpeel
