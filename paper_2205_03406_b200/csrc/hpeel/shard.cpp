// Work partitioning and the run-time-loaded NCCL communicator (shard.hpp).
#include "shard.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

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

namespace {

// Minimal NCCL ABI (nccl.h 2.x): opaque comm, 128-byte unique id.
struct NcclUniqueId {
  char internal[128];
};
using ncclComm_t = void*;
enum NcclDataType { kNcclInt32 = 2, kNcclFloat64 = 8 };
enum NcclRedOp { kNcclMax = 2 };

struct NcclApi {
  int (*GetUniqueId)(NcclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
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
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  return api;
}

void check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + ": " + nccl().GetErrorString(rc));
}

}  // namespace

void Comm::unique_id(unsigned char out[128]) {
  NcclUniqueId id;
  check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

Comm::Comm(const unsigned char id[128], int rank, int world, int device)
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

Comm::~Comm() {
  if (comm_) nccl().CommDestroy(comm_);
}

void Comm::broadcast_segments(double* buf, const std::vector<std::int64_t>& off, cudaStream_t s) {
  if (world_ == 1) return;
  check(nccl().GroupStart(), "ncclGroupStart");
  for (int r = 0; r < world_; ++r) {
    const std::int64_t n = off[size_t(r) + 1] - off[size_t(r)];
    if (n <= 0) continue;
    double* p = buf + off[size_t(r)];
    check(nccl().Broadcast(p, p, size_t(n), kNcclFloat64, r, comm_, s), "ncclBroadcast");
  }
  check(nccl().GroupEnd(), "ncclGroupEnd");
}

void Comm::broadcast_segments_i32(int* buf, const std::vector<std::int64_t>& off, cudaStream_t s) {
  if (world_ == 1) return;
  check(nccl().GroupStart(), "ncclGroupStart");
  for (int r = 0; r < world_; ++r) {
    const std::int64_t n = off[size_t(r) + 1] - off[size_t(r)];
    if (n <= 0) continue;
    int* p = buf + off[size_t(r)];
    check(nccl().Broadcast(p, p, size_t(n), kNcclInt32, r, comm_, s), "ncclBroadcast");
  }
  check(nccl().GroupEnd(), "ncclGroupEnd");
}

void Comm::all_reduce_max(double* v, cudaStream_t s) {
  if (world_ == 1) return;
  check(nccl().AllReduce(v, v, 1, kNcclFloat64, kNcclMax, comm_, s), "ncclAllReduce");
}

}  // namespace hpeel
