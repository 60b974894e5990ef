// Layout and verification kernels (sm_100a): strided row gather between input
// and tree order, the dense-block part of H1Rep::apply
// (dense_contribution, proj/src/hmatrix.cpp:59-73), and small reductions.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"

namespace hpeel {

namespace {

__global__ void gather_rows_kernel(const double* __restrict__ src, std::int64_t ssr,
                                   std::int64_t ssc, const int* __restrict__ map,
                                   std::int64_t rows, int w, double* __restrict__ dst,
                                   std::int64_t dsr, std::int64_t dsc) {
  const std::int64_t total = rows * w;
  for (std::int64_t e = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; e < total;
       e += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t i = e % rows, c = e / rows;
    const std::int64_t si = map ? map[i] : i;
    dst[i * dsr + c * dsc] = src[si * ssr + c * ssc];
  }
}

// y[(row0 + i) + c * ldy] += sum_partners D x   (x row-major n x w, y col-major)
__global__ void dense_apply_kernel(const DenseTask* __restrict__ tasks,
                                   const int* __restrict__ off, const double* __restrict__ dense,
                                   const double* __restrict__ x, int w, int adjoint,
                                   double* __restrict__ y, std::int64_t ldy) {
  const int box = blockIdx.x;
  const int t0 = off[box], t1 = off[box + 1];
  if (t0 == t1) return;
  const int rows = adjoint ? tasks[t0].cols : tasks[t0].rows;
  const std::int64_t row0 = adjoint ? tasks[t0].col0 : tasks[t0].row0;
  for (int e = threadIdx.x; e < rows * w; e += blockDim.x) {
    const int i = e / w, c = e - i * w;
    double acc = 0.0;
    for (int q = t0; q < t1; ++q) {
      const DenseTask t = tasks[q];
      const double* d = dense + t.d;
      if (!adjoint) {
        for (int j = 0; j < t.cols; ++j) acc = fma(d[i + std::int64_t(j) * t.rows], x[(t.col0 + j) * w + c], acc);
      } else {
        for (int j = 0; j < t.rows; ++j) acc = fma(d[j + std::int64_t(i) * t.rows], x[(t.row0 + j) * w + c], acc);
      }
    }
    y[(row0 + i) + c * ldy] += acc;
  }
}

}  // namespace

void launch_permute_rows(const double* src, std::int64_t ssr, std::int64_t ssc, const int* map,
                         std::int64_t rows, int w, double* dst, std::int64_t dsr, std::int64_t dsc,
                         cudaStream_t s) {
  const std::int64_t total = rows * w;
  if (total == 0) return;
  const unsigned blocks = unsigned(std::min<std::int64_t>((total + 255) / 256, 148 * 16));
  gather_rows_kernel<<<blocks, 256, 0, s>>>(src, ssr, ssc, map, rows, w, dst, dsr, dsc);
  HP_LAUNCHED();
}

void launch_dense_apply(const DenseTask* tasks, const int* box_off, int nboxes,
                        const double* dense, const double* x, int w, bool adjoint, double* y,
                        std::int64_t ldy, cudaStream_t s) {
  if (nboxes == 0) return;
  dense_apply_kernel<<<nboxes, 256, 0, s>>>(tasks, box_off, dense, x, w, adjoint ? 1 : 0, y, ldy);
  HP_LAUNCHED();
}

}  // namespace hpeel

namespace hpeel {
std::int64_t& launch_counter() {
  static std::int64_t count = 0;
  return count;
}
}  // namespace hpeel

#include <cmath>
#include <map>
#include <mutex>
#include <vector>

namespace hpeel {
namespace {
__global__ void find_duplicates_kernel(const double* __restrict__ x, int dim, std::int64_t n,
                                       const std::int64_t* __restrict__ leaf_start,
                                       const std::int64_t* __restrict__ leaf_count, int* flag) {
  const std::int64_t s0 = leaf_start[blockIdx.x];
  const int m = int(leaf_count[blockIdx.x]);
  const std::int64_t pairs = std::int64_t(m) * (m - 1) / 2;
  for (std::int64_t q = threadIdx.x; q < pairs; q += blockDim.x) {
    // q -> (i, j), i < j
    int i = int((sqrt(8.0 * double(q) + 1.0) - 1.0) / 2.0) + 1;
    while (std::int64_t(i) * (i - 1) / 2 > q) --i;
    while (std::int64_t(i + 1) * i / 2 <= q) ++i;
    const int j = int(q - std::int64_t(i) * (i - 1) / 2);
    bool eq = true;
    for (int d = 0; d < dim; ++d) eq = eq && x[d * n + s0 + i] == x[d * n + s0 + j];
    if (eq) atomicOr(flag, 1);
  }
}
}  // namespace

void launch_find_duplicates(const double* x, int dim, std::int64_t n, const std::int64_t* leaf_start,
                            const std::int64_t* leaf_count, int nleaves, int* flag, cudaStream_t s) {
  if (nleaves == 0) return;
  find_duplicates_kernel<<<nleaves, 256, 0, s>>>(x, dim, n, leaf_start, leaf_count, flag);
  HP_LAUNCHED();
}

const double* log_table_device(int device) {
  static std::mutex mu;
  static std::map<int, double*> tabs;
  std::lock_guard<std::mutex> lock(mu);
  auto it = tabs.find(device);
  if (it != tabs.end()) return it->second;
  // T_k = 1 / inv_k exactly (inv_k = 1 / (1 + k/2^kLogBits) rounded); stored:
  // pairs {inv_k / 2, 0.5 log T_k'} (extended precision), where T_k' = T_k
  // below kLogSplit and T_k / 2 from it on (device.cuh half_log)
  std::vector<double> h(2 * kLogTab);
  for (int k = 0; k < kLogTab; ++k) {
    const double inv = double(1.0L / (1.0L + (long double)k / (long double)(1 << kLogBits)));
    long double t = 1.0L / (long double)inv;
    if (k >= kLogSplit) t /= 2.0L;
    h[size_t(2 * k)] = inv / 2.0;
    h[size_t(2 * k + 1)] = double(0.5L * logl(t));
  }
  int prev = 0;
  HP_CUDA(cudaGetDevice(&prev));
  HP_CUDA(cudaSetDevice(device));
  double* d = nullptr;
  HP_CUDA(cudaMalloc(&d, h.size() * sizeof(double)));
  HP_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  HP_CUDA(cudaSetDevice(prev));
  tabs[device] = d;
  return d;
}
}  // namespace hpeel

// ------------------------------------------------------------------ sharding
// Packing of the per-level factor exchanges and the callback
// black box's dense test matrices / sample rows.
namespace hpeel {

namespace {

// one CTA per segment, 16-byte vector copies when both ends are aligned
__global__ void copy_segments_kernel(const double* __restrict__ src, const CopySeg* __restrict__ segs,
                                     double* __restrict__ dst) {
  const CopySeg sg = segs[blockIdx.x];
  const double* a = src + sg.src;
  double* b = dst + sg.dst;
  if (((sg.src | sg.dst) & 1) == 0) {
    const std::int64_t n2 = sg.len >> 1;
    for (std::int64_t e = threadIdx.x; e < n2; e += blockDim.x)
      reinterpret_cast<double2*>(b)[e] = reinterpret_cast<const double2*>(a)[e];
    if ((sg.len & 1) && threadIdx.x == 0) b[sg.len - 1] = a[sg.len - 1];
  } else {
    for (std::int64_t e = threadIdx.x; e < sg.len; e += blockDim.x) b[e] = a[e];
  }
}

__global__ void move_i32_kernel(const int* __restrict__ src, const int* __restrict__ sidx, std::int64_t n,
                                int* __restrict__ dst, const int* __restrict__ didx) {
  for (std::int64_t e = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; e < n;
       e += std::int64_t(gridDim.x) * blockDim.x)
    dst[didx ? didx[e] : e] = src[sidx ? sidx[e] : e];
}

__global__ void gather_sample_rows_kernel(const double* __restrict__ y, std::int64_t ldy,
                                          const int* __restrict__ perm, const GatherRow* __restrict__ rows,
                                          std::int64_t nrows, int w, double* __restrict__ out, int ocol0) {
  const std::int64_t total = nrows * w;
  for (std::int64_t e = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; e < total;
       e += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t i = e % nrows;
    const int c = int(e / nrows);
    const GatherRow r = rows[i];
    if (c < r.cols) out[r.out + std::int64_t(ocol0 + c) * r.ld] = y[perm[r.pos] + std::int64_t(c) * ldy];
  }
}

__global__ void scatter_payload_kernel(const double* __restrict__ g, int gld, int gcol0, int w,
                                       const int* __restrict__ pos, std::int64_t cnt,
                                       const int* __restrict__ perm, double* __restrict__ omega,
                                       std::int64_t ldo) {
  const std::int64_t total = cnt * w;
  for (std::int64_t e = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; e < total;
       e += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t q = e % cnt;
    const int c = int(e / cnt);
    const int p = pos[q];
    omega[perm[p] + std::int64_t(c) * ldo] = g[std::int64_t(p) * gld + gcol0 + c];
  }
}

__global__ void scatter_identity_kernel(const int* __restrict__ boxes, const std::int64_t* __restrict__ box_start,
                                        const std::int64_t* __restrict__ box_count, const int* __restrict__ perm,
                                        int w, double* __restrict__ omega, std::int64_t ldo) {
  const int b = boxes[blockIdx.x];
  const std::int64_t st = box_start[b];
  const int cnt = int(box_count[b] < w ? box_count[b] : w);
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) omega[perm[st + t] + std::int64_t(t) * ldo] = 1.0;
}

unsigned grid_for(std::int64_t total) {
  return unsigned(std::max<std::int64_t>(1, std::min<std::int64_t>((total + 255) / 256, 148 * 16)));
}

}  // namespace

void launch_copy_segments(const double* src, const CopySeg* segs, int nseg, double* dst, cudaStream_t s) {
  if (nseg == 0) return;
  copy_segments_kernel<<<nseg, 256, 0, s>>>(src, segs, dst);
  HP_LAUNCHED();
}

void launch_move_i32(const int* src, const int* sidx, std::int64_t n, int* dst, const int* didx, cudaStream_t s) {
  if (n == 0) return;
  move_i32_kernel<<<grid_for(n), 256, 0, s>>>(src, sidx, n, dst, didx);
  HP_LAUNCHED();
}

void launch_gather_sample_rows(const double* y, std::int64_t ldy, const int* perm, const GatherRow* rows,
                               std::int64_t nrows, int w, double* out, int ocol0, cudaStream_t s) {
  if (nrows == 0 || w == 0) return;
  gather_sample_rows_kernel<<<grid_for(nrows * w), 256, 0, s>>>(y, ldy, perm, rows, nrows, w, out, ocol0);
  HP_LAUNCHED();
}

void launch_scatter_payload(const double* g, int gld, int gcol0, int w, const int* pos, std::int64_t cnt,
                            const int* perm, double* omega, std::int64_t ldo, cudaStream_t s) {
  if (cnt == 0 || w == 0) return;
  scatter_payload_kernel<<<grid_for(cnt * w), 256, 0, s>>>(g, gld, gcol0, w, pos, cnt, perm, omega, ldo);
  HP_LAUNCHED();
}

void launch_scatter_identity(const int* boxes, int nbox, const std::int64_t* box_start,
                             const std::int64_t* box_count, const int* perm, int w, double* omega,
                             std::int64_t ldo, cudaStream_t s) {
  if (nbox == 0) return;
  scatter_identity_kernel<<<nbox, 128, 0, s>>>(boxes, box_start, box_count, perm, w, omega, ldo);
  HP_LAUNCHED();
}

}  // namespace hpeel
