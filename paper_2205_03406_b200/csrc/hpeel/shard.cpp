// Ownership plan, the run-time-loaded NCCL communicator and the in-process
// group communicator (shard.hpp).
#include "shard.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "box_tree.hpp"

namespace hpeel {

std::vector<std::int64_t> partition_ranges(const std::vector<double>& work, int world) {
  if (world < 1) throw std::invalid_argument("world size must be >= 1");
  const std::int64_t n = std::int64_t(work.size());
  std::vector<double> prefix(size_t(n) + 1, 0.0);
  for (std::int64_t i = 0; i < n; ++i) prefix[size_t(i) + 1] = prefix[size_t(i)] + work[size_t(i)];
  const double total = prefix[size_t(n)];
  std::vector<std::int64_t> b(size_t(world) + 1, 0);
  b[size_t(world)] = n;
  for (int r = 1; r < world; ++r) {
    const double target = total * double(r) / double(world);
    // boundary whose prefix sum is nearest the target
    const auto it = std::lower_bound(prefix.begin(), prefix.end(), target);
    std::int64_t cut = std::int64_t(it - prefix.begin());
    if (cut > 0 && cut <= n && target - prefix[size_t(cut) - 1] < prefix[size_t(cut)] - target) --cut;
    cut = std::min(std::max(cut, b[size_t(r) - 1]), n);
    b[size_t(r)] = cut;
  }
  return b;
}

Ownership make_ownership(const BoxTree& tree, const TreeLayout& lay, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank / world size");
  Ownership o;
  o.world = world;
  o.rank = rank;
  const int nb = tree.num_boxes();
  o.owner.assign(size_t(nb), world == 1 ? 0 : -1);
  o.point_bounds = {0, std::int64_t(tree.num_points())};
  if (world == 1) return o;
  // cut level: the first whose frontier (boxes at the level plus the leaves
  // above it) has at least 4 boxes per rank, so point counts can balance
  std::vector<int> frontier;
  for (int lc = 1; lc <= tree.depth(); ++lc) {
    frontier.clear();
    for (const Box& b : tree.boxes())
      if (b.level == lc || (b.level < lc && b.is_leaf())) frontier.push_back(b.id);
    o.cut = lc;
    if (int(frontier.size()) >= 4 * world) break;
  }
  if (tree.depth() == 0) {
    frontier = {0};
    o.cut = 0;
  }
  std::sort(frontier.begin(), frontier.end(),
            [&](int x, int y) { return lay.start[size_t(x)] < lay.start[size_t(y)]; });
  std::vector<double> work(frontier.size());
  for (size_t i = 0; i < frontier.size(); ++i) work[i] = double(lay.count[size_t(frontier[i])]);
  const auto bounds = partition_ranges(work, world);
  o.point_bounds.assign(size_t(world) + 1, std::int64_t(tree.num_points()));
  for (int g = world - 1; g >= 0; --g) {
    for (std::int64_t i = bounds[size_t(g)]; i < bounds[size_t(g) + 1]; ++i) o.owner[size_t(frontier[size_t(i)])] = g;
    if (bounds[size_t(g)] < bounds[size_t(g) + 1])
      o.point_bounds[size_t(g)] = lay.start[size_t(frontier[size_t(bounds[size_t(g)])])];
    else
      o.point_bounds[size_t(g)] = o.point_bounds[size_t(g) + 1];
  }
  o.point_bounds[0] = 0;
  // descendants inherit (ids grow with the level: parents come first)
  for (const Box& b : tree.boxes())
    if (b.parent >= 0 && o.owner[size_t(b.id)] < 0 && o.owner[size_t(b.parent)] >= 0)
      o.owner[size_t(b.id)] = o.owner[size_t(b.parent)];
  return o;
}

// ------------------------------------------------------------------ NCCL

namespace {

// Minimal NCCL ABI (nccl.h 2.x): opaque comm, 128-byte unique id.
struct NcclUniqueId {
  char internal[128];
};
using ncclComm_t = void*;
enum NcclDataType { kNcclInt32 = 2, kNcclFloat64 = 8 };

struct NcclApi {
  int (*GetUniqueId)(NcclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw std::runtime_error(std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) throw std::runtime_error(std::string("libnccl.so.2 lacks ") + name);
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  return api;
}

void check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + ": " + nccl().GetErrorString(rc));
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define HP_CUDA(call) cuda_check((call), #call)

void check_offsets(const std::vector<std::int64_t>& off, int world, const char* what) {
  if (int(off.size()) != world + 1) throw std::invalid_argument(std::string(what) + ": need world + 1 offsets");
}

}  // namespace

void NcclComm::unique_id(unsigned char out[128]) {
  NcclUniqueId id;
  check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

NcclComm::NcclComm(const unsigned char id[128], int rank, int world, int device)
    : rank_(rank), world_(world), device_(device) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank / world size");
  if (world == 1) return;
  NcclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  ncclComm_t c = nullptr;
  check(nccl().CommInitRank(&c, world, uid, rank), "ncclCommInitRank");
  cudaSetDevice(prev);
  comm_ = c;
}

NcclComm::~NcclComm() {
  if (comm_) nccl().CommDestroy(comm_);
}

void NcclComm::bcast(void* buf, const std::vector<std::int64_t>& off, int type, size_t elem, cudaStream_t s) {
  if (world_ == 1) return;
  check_offsets(off, world_, "broadcast_segments");
  check(nccl().GroupStart(), "ncclGroupStart");
  for (int r = 0; r < world_; ++r) {
    const std::int64_t n = off[size_t(r) + 1] - off[size_t(r)];
    if (n <= 0) continue;
    char* p = static_cast<char*>(buf) + size_t(off[size_t(r)]) * elem;
    check(nccl().Broadcast(p, p, size_t(n), type, r, comm_, s), "ncclBroadcast");
  }
  check(nccl().GroupEnd(), "ncclGroupEnd");
}

void NcclComm::a2av(const void* send, const std::vector<std::int64_t>& soff, void* recv,
                    const std::vector<std::int64_t>& roff, int type, size_t elem, cudaStream_t s) {
  if (world_ == 1) return;
  check_offsets(soff, world_, "exchange");
  check_offsets(roff, world_, "exchange");
  check(nccl().GroupStart(), "ncclGroupStart");
  for (int j = 0; j < world_; ++j) {
    if (j == rank_) continue;
    const std::int64_t ns = soff[size_t(j) + 1] - soff[size_t(j)];
    const std::int64_t nr = roff[size_t(j) + 1] - roff[size_t(j)];
    if (ns > 0)
      check(nccl().Send(static_cast<const char*>(send) + size_t(soff[size_t(j)]) * elem, size_t(ns), type, j, comm_, s),
            "ncclSend");
    if (nr > 0)
      check(nccl().Recv(static_cast<char*>(recv) + size_t(roff[size_t(j)]) * elem, size_t(nr), type, j, comm_, s),
            "ncclRecv");
  }
  check(nccl().GroupEnd(), "ncclGroupEnd");
}

void NcclComm::broadcast_segments(double* buf, const std::vector<std::int64_t>& off, cudaStream_t s) {
  bcast(buf, off, kNcclFloat64, sizeof(double), s);
}
void NcclComm::broadcast_segments_i32(int* buf, const std::vector<std::int64_t>& off, cudaStream_t s) {
  bcast(buf, off, kNcclInt32, sizeof(int), s);
}
void NcclComm::exchange(const double* send, const std::vector<std::int64_t>& soff, double* recv,
                        const std::vector<std::int64_t>& roff, cudaStream_t s) {
  a2av(send, soff, recv, roff, kNcclFloat64, sizeof(double), s);
}
void NcclComm::exchange_i32(const int* send, const std::vector<std::int64_t>& soff, int* recv,
                            const std::vector<std::int64_t>& roff, cudaStream_t s) {
  a2av(send, soff, recv, roff, kNcclInt32, sizeof(int), s);
}

// ------------------------------------------------------------------ local group

LocalGroup::LocalGroup(int world) : world_(world), slots_(size_t(world)) {
  if (world < 1) throw std::invalid_argument("world size must be >= 1");
}

void LocalGroup::abort() {
  std::lock_guard<std::mutex> lock(mu_);
  aborted_ = true;
  cv_.notify_all();
}

void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lock(mu_);
  if (aborted_) throw std::runtime_error("emulated rank group aborted by a failing peer");
  const std::uint64_t gen = generation_;
  if (++arrived_ == world_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
    return;
  }
  cv_.wait(lock, [&] { return generation_ != gen || aborted_; });
  if (generation_ == gen) throw std::runtime_error("emulated rank group aborted by a failing peer");
}

LocalComm::LocalComm(std::shared_ptr<LocalGroup> group, int rank, int device)
    : group_(std::move(group)), rank_(rank), device_(device) {
  if (rank < 0 || rank >= group_->world()) throw std::invalid_argument("bad rank / world size");
  HP_CUDA(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
  HP_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
}

LocalComm::~LocalComm() {
  cudaEventDestroy(ready_);
  cudaEventDestroy(done_);
}

void LocalComm::bcast(void* buf, const std::vector<std::int64_t>& off, size_t elem, cudaStream_t s) {
  const int w = world();
  if (w == 1) return;
  check_offsets(off, w, "broadcast_segments");
  LocalGroup& g = *group_;
  HP_CUDA(cudaEventRecord(ready_, s));
  g.slot(rank_).ptr = buf;
  g.slot(rank_).off = off;
  g.slot(rank_).ready = ready_;
  g.barrier();
  for (int r = 0; r < w; ++r) {
    if (r == rank_) continue;
    const auto& sl = g.slot(r);
    const std::int64_t n = off[size_t(r) + 1] - off[size_t(r)];
    if (sl.off != off) throw std::logic_error("broadcast_segments: ranks disagree on the segments");
    if (n <= 0) continue;
    HP_CUDA(cudaStreamWaitEvent(s, sl.ready, 0));
    HP_CUDA(cudaMemcpyAsync(static_cast<char*>(buf) + size_t(off[size_t(r)]) * elem,
                            static_cast<const char*>(sl.ptr) + size_t(off[size_t(r)]) * elem, size_t(n) * elem,
                            cudaMemcpyDeviceToDevice, s));
  }
  HP_CUDA(cudaEventRecord(done_, s));
  g.slot(rank_).done = done_;
  g.barrier();
  // our segment must stay unchanged until every peer has copied it
  for (int r = 0; r < w; ++r)
    if (r != rank_) HP_CUDA(cudaStreamWaitEvent(s, g.slot(r).done, 0));
  g.barrier();
}

void LocalComm::a2av(const void* send, const std::vector<std::int64_t>& soff, void* recv,
                     const std::vector<std::int64_t>& roff, size_t elem, cudaStream_t s) {
  const int w = world();
  if (w == 1) return;
  check_offsets(soff, w, "exchange");
  check_offsets(roff, w, "exchange");
  LocalGroup& g = *group_;
  HP_CUDA(cudaEventRecord(ready_, s));
  g.slot(rank_).ptr = send;
  g.slot(rank_).off = soff;
  g.slot(rank_).ready = ready_;
  g.barrier();
  for (int i = 0; i < w; ++i) {
    if (i == rank_) continue;
    const auto& sl = g.slot(i);
    const std::int64_t n = roff[size_t(i) + 1] - roff[size_t(i)];
    const std::int64_t ns = sl.off[size_t(rank_) + 1] - sl.off[size_t(rank_)];
    if (n != ns) throw std::logic_error("exchange: send and receive counts disagree");
    if (n <= 0) continue;
    HP_CUDA(cudaStreamWaitEvent(s, sl.ready, 0));
    HP_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + size_t(roff[size_t(i)]) * elem,
                            static_cast<const char*>(sl.ptr) + size_t(sl.off[size_t(rank_)]) * elem,
                            size_t(n) * elem, cudaMemcpyDeviceToDevice, s));
  }
  HP_CUDA(cudaEventRecord(done_, s));
  g.slot(rank_).done = done_;
  g.barrier();
  for (int i = 0; i < w; ++i)
    if (i != rank_) HP_CUDA(cudaStreamWaitEvent(s, g.slot(i).done, 0));
  g.barrier();
}

void LocalComm::broadcast_segments(double* buf, const std::vector<std::int64_t>& off, cudaStream_t s) {
  bcast(buf, off, sizeof(double), s);
}
void LocalComm::broadcast_segments_i32(int* buf, const std::vector<std::int64_t>& off, cudaStream_t s) {
  bcast(buf, off, sizeof(int), s);
}
void LocalComm::exchange(const double* send, const std::vector<std::int64_t>& soff, double* recv,
                         const std::vector<std::int64_t>& roff, cudaStream_t s) {
  a2av(send, soff, recv, roff, sizeof(double), s);
}
void LocalComm::exchange_i32(const int* send, const std::vector<std::int64_t>& soff, int* recv,
                             const std::vector<std::int64_t>& roff, cudaStream_t s) {
  a2av(send, soff, recv, roff, sizeof(int), s);
}

}  // namespace hpeel
