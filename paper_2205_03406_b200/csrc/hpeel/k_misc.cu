// Layout and verification kernels (sm_100a): strided row gather between input
// and tree order, the dense-block part of H1Rep::apply
// (dense_contribution, proj/src/hmatrix.cpp:59-73), and small reductions.
#include <cuda_runtime.h>

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
