// Device-side plumbing shared by the driver (driver.cu) and the
// representation/verifier code (rep.cu): stream-ordered buffers, event
// timers, the per-tree Engine (tree-order coordinates, box ranges, ancestor
// table) and the batched QR / Gram / peeling task builders.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "kernels.hpp"
#include "peeling.hpp"

namespace hpeel::detail {

/// Pinned staging for host->device uploads (DevBuf::upload) inside a
/// StagingScope: a pageable cudaMemcpyAsync waits for the stream to drain,
/// which would tie the driver thread to the device and serialize host
/// planning with device work. Chunks come from a process-wide pool and go
/// back to it when the scope ends (after synchronizing its stream).
class PinnedStaging {
 public:
  static PinnedStaging*& current();
  void* take(size_t bytes);
  void release_to_pool();

 private:
  struct Chunk {
    char* p;
    size_t size;
    size_t used;
  };
  std::vector<Chunk> chunks_;
};

/// Grow-only pinned host buffer `slot` (< 4) of the calling thread.
void* persistent_pinned(size_t bytes, int slot);

class StagingScope {
 public:
  explicit StagingScope(cudaStream_t s) : s_(s), prev_(PinnedStaging::current()) {
    PinnedStaging::current() = &staging_;
  }
  ~StagingScope() {
    cudaStreamSynchronize(s_);
    PinnedStaging::current() = prev_;
    staging_.release_to_pool();
  }
  StagingScope(const StagingScope&) = delete;
  StagingScope& operator=(const StagingScope&) = delete;

 private:
  cudaStream_t s_;
  PinnedStaging* prev_;
  PinnedStaging staging_;
};

/// Device bytes held by the buffers of the calling thread's compress()
/// (peak reported as RunReport::peak_device_bytes).
struct MemTracker {
  std::int64_t cur = 0, peak = 0;
  static MemTracker*& current() {
    thread_local MemTracker* t = nullptr;
    return t;
  }
  static void add(std::int64_t b) {
    if (MemTracker* t = current()) {
      t->cur += b;
      if (t->cur > t->peak) t->peak = t->cur;
    }
  }
};

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
  ~DevBuf() { release(); }
  void alloc(size_t n, cudaStream_t s) {
    release();
    n_ = n;
    s_ = s;
    if (n) {
      HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
      MemTracker::add(std::int64_t(n * sizeof(T)));
    }
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(v.size(), s);
    if (v.empty()) return;
    const size_t bytes = v.size() * sizeof(T);
    if (PinnedStaging* st = PinnedStaging::current()) {
      void* h = st->take(bytes);
      std::memcpy(h, v.data(), bytes);
      HP_CUDA(cudaMemcpyAsync(p_, h, bytes, cudaMemcpyHostToDevice, s));
    } else {
      HP_CUDA(cudaMemcpyAsync(p_, v.data(), bytes, cudaMemcpyHostToDevice, s));
    }
  }
  void release() {
    if (p_) {
      cudaFreeAsync(p_, s_);
      MemTracker::add(-std::int64_t(n_ * sizeof(T)));
    }
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
};

struct Events {
  cudaEvent_t a = nullptr, b = nullptr;
  Events() {
    HP_CUDA(cudaEventCreate(&a));
    HP_CUDA(cudaEventCreate(&b));
  }
  Events(const Events&) = delete;
  ~Events() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  float ms() const {
    float t = 0.f;
    HP_CUDA(cudaEventElapsedTime(&t, a, b));
    return t;
  }
};

/// Keep the device's default stream-ordered pool across synchronizations
/// (release threshold = max), so repeated compress() calls reuse its memory
/// instead of remapping it every time. Once per device.
void retain_default_pool(int dev);

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    HP_CUDA(cudaGetDevice(&prev_));
    if (prev_ != dev) HP_CUDA(cudaSetDevice(dev));
    retain_default_pool(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev_); }

 private:
  int prev_ = 0;
};

constexpr int kTile = 64;  // rows per K2 / K3 CTA

// Tree-order copy of the black box and the box tables, for one tree.
struct Engine {
  const BoxTree& tree;
  const AdjacencyInfo& adj;
  const TreeLayout& lay;
  const DeviceOperator& op;
  cudaStream_t s;
  int r = 0, k = 0;
  Index n = 0;
  DevBuf<double> xt;  // tree-order coordinates (dim x n SoA)
  DevBuf<double> at;  // tree-order dense matrix
  DevOp dop;
  DevBuf<std::int64_t> d_box_start, d_box_count;
  DevBuf<int> d_perm, d_inv;  // tree position -> input index and back
  bool has_dups = false;  // kernel kinds: two distinct points share coordinates
  DevBuf<double> d_box_bbox;  // int8 K2: raw-coordinate bounding box per box (built on first use)
  std::vector<std::vector<int>> anc;  // anc[l][box] = ancestor at level l (or -1)

  Engine(const BoxTree& t, const AdjacencyInfo& a, const TreeLayout& l, const DeviceOperator& o,
         cudaStream_t st);
  std::int64_t start(int b) const { return lay.start[size_t(b)]; }
  int count(int b) const { return int(lay.count[size_t(b)]); }
  void ensure_box_bbox();
  /// y = A x (or A^T x) on tree-order col-major n x w device buffers, through
  /// the black box: on-the-fly / dense kernels or the caller's callback.
  void op_apply(bool adjoint, const double* x_tree, int w, double* y_tree) const;
};

int pair_index(const std::vector<std::pair<int, int>>& pairs, int a, int b);
std::pair<int, int> first_range(const std::vector<std::pair<int, int>>& pairs, int a);

// ---------------------------------------------------------------- K4 plan
struct QrRequest {
  std::int64_t a;
  std::int64_t out;
  int rows;
  int ldo;
  int rank_slot;
};
struct QrPlan {
  std::vector<QrBlock> direct, tops;
  std::vector<std::vector<QrBlock>> chunk_rounds, back_rounds;
  std::int64_t wsize = 0, tausize = 0;
  bool reg = false;  // register-resident kernels (k_qr2.cu)
  // Gram-based range finder (k_gqr.cu) for gblocks; the lists above then hold only the short
  // narrow blocks left to the Householder kernels (plan_qr)
  bool gram = false;
  std::vector<GqrBlock> gblocks;
  std::vector<GqrTask> gtasks;
  std::vector<GqrBlock> hblocks;  // the Householder-routed blocks, for the range rescale
  std::vector<GqrTask> htasks;
};
QrPlan plan_qr(const std::vector<QrRequest>& reqs, int r, int kmax);
void run_qr(const QrPlan& plan, double* data, double* out, int* d_ranks, int r, int kmax,
            cudaStream_t s);

// ---------------------------------------------------------------- K5 grams
struct GramReq {
  std::int64_t x, y;
  int rows, lx, ly, x_rowmajor, y_rowmajor;
};
struct GramPlan {
  std::vector<GramTask> tasks;
  std::vector<std::int64_t> off;
  int nx = 0, ny = 0;
};
GramPlan plan_gram(const std::vector<GramReq>& reqs, int nx, int ny);
void run_gram(const GramPlan& plan, const double* xb, const double* yb, double* out,
              cudaStream_t s);

// ---------------------------------------------------------------- K3 plan
struct PeelPlan {
  std::vector<CoeffTask> coeff_fwd, coeff_adj;
  std::vector<std::int64_t> seg_start, seg_count;
  std::vector<PeelTask> tasks_fwd, tasks_adj;
  std::vector<PeelRef> refs_fwd, refs_adj;
  std::vector<PeelTerm> terms_fwd, terms_adj;
  double coeff_flops = 0, apply_flops = 0;
};
struct SampleBlock {
  int box;
  int color;
  std::int64_t off;  // sample block offset (col-major, ld = |I_box|)
  int cols = 1 << 30;  // columns kept (compact dense blocks: |I_mu|)
};
PeelPlan plan_peel(const Engine& e, const H1Rep& rep, const std::vector<SampleBlock>& blocks,
                   const std::vector<std::vector<int>>& payload_boxes, int top_level, int w,
                   bool with_adjoint);
/// plan_peel with the colors split over `threads` host threads (same tasks,
/// coefficients and term order per output tile; used for the leaf phase).
PeelPlan plan_peel_parallel(const Engine& e, const H1Rep& rep, const std::vector<SampleBlock>& blocks,
                            const std::vector<std::vector<int>>& payload_boxes, int top_level, int w,
                            bool with_adjoint, int threads);
void run_peel(const PeelPlan& pp, const Engine& e, const H1Rep& rep, const double* g, int gld,
              int w, bool identity, double* samples, int adj_col, cudaStream_t s);

}  // namespace hpeel::detail
