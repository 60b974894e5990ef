// K4 batched range finder (sm_100a): qr_orthonormal of every sample block
// (proj/src/linalg.cpp:53-78, via basis_from_sample proj/src/peeling.cpp:63-71).
//
// Blocks that fit in shared memory run column-pivoted Householder QR in one
// CTA (the ColPivHouseholderQR rule: pivot = largest remaining column norm,
// first index on ties; keep = leading |R_jj| > 1e-14 |R_00|, capped at k;
// Q(:, :keep) formed explicitly). Taller blocks go through TSQR: unpivoted
// Householder QR of row chunks, the stacked R factors are reduced the same
// way, the top is pivoted; in exact arithmetic this selects the same pivots and
// span as pivoted QR of the whole block. Q is then back-propagated through the
// chunk reflectors.
#include <cuda_runtime.h>

#include <cmath>

#include "kernels.hpp"

namespace hpeel {

namespace {

constexpr int kQrThreads = 256;
constexpr int kQrWarps = kQrThreads / 32;
constexpr size_t kQrSmemBudget = 216 * 1024;

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kQrWarps; ++w) t += red[w];
  return t;
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Householder step on column j of a (m x n, ld m) in shared memory: LAPACK
// dlarfg convention, v(j) = 1 implicit, reflector stored below the diagonal.
// Applies H = I - tau v v^T to columns j+1..n-1. Returns tau (all threads).
__device__ double householder_step(double* a, int m, int n, int j, double* red) {
  double* col = a + j * m;
  double part = 0.0;
  for (int i = j + 1 + threadIdx.x; i < m; i += kQrThreads) part += col[i] * col[i];
  const double sigma = block_sum(part, red);
  const double alpha = col[j];
  double tau = 0.0;
  if (sigma > 0.0) {
    const double beta = alpha >= 0.0 ? -sqrt(alpha * alpha + sigma) : sqrt(alpha * alpha + sigma);
    tau = (beta - alpha) / beta;
    const double scale = 1.0 / (alpha - beta);
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < m; i += kQrThreads) col[i] *= scale;
    if (threadIdx.x == 0) col[j] = beta;
  }
  __syncthreads();
  if (tau != 0.0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = j + 1 + warp; c < n; c += kQrWarps) {
      double* ac = a + c * m;
      double s = lane == 0 ? ac[j] : 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) s = fma(col[i], ac[i], s);
      s = warp_sum(s) * tau;
      if (lane == 0) ac[j] -= s;
      for (int i = j + 1 + lane; i < m; i += 32) ac[i] = fma(-s, col[i], ac[i]);
    }
  }
  __syncthreads();
  return tau;
}

__device__ void load_block(double* as, const double* src, int m, int n, int ld) {
  for (int e = threadIdx.x; e < m * n; e += kQrThreads) {
    const int i = e % m, j = e / m;
    as[e] = src[i + std::int64_t(j) * ld];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kQrThreads)
qr_chunk_kernel(const QrBlock* __restrict__ blocks, double* data, double* rout, double* tau_out,
                int n) {
  extern __shared__ double sm[];
  __shared__ double red[kQrWarps];
  const QrBlock b = blocks[blockIdx.x];
  const int m = b.rows;
  double* as = sm;
  load_block(as, data + b.a, m, n, b.lda);
  const int kk = m < n ? m : n;
  for (int j = 0; j < kk; ++j) {
    const double tau = householder_step(as, m, n, j, red);
    if (threadIdx.x == 0) tau_out[b.tau + j] = tau;
  }
  // reflectors back in place; R into the parent stacked matrix
  for (int e = threadIdx.x; e < m * n; e += kQrThreads) {
    const int i = e % m, j = e / m;
    data[b.a + i + std::int64_t(j) * b.lda] = as[e];
  }
  for (int e = threadIdx.x; e < kk * n; e += kQrThreads) {
    const int i = e % kk, j = e / kk;
    rout[b.out + i + std::int64_t(j) * b.ldo] = i <= j ? as[i + j * m] : 0.0;
  }
}

__global__ void __launch_bounds__(kQrThreads)
qr_top_kernel(const QrBlock* __restrict__ blocks, double* data, double* outbuf, int* ranks, int n,
              int kmax, double tol) {
  extern __shared__ double sm[];
  __shared__ double red[kQrWarps];
  __shared__ double taus[160];
  __shared__ double norms[160];
  __shared__ int keep_s;
  const QrBlock b = blocks[blockIdx.x];
  const int m = b.rows;
  double* as = sm;
  double* vec = sm + std::int64_t(m) * n;  // kQrWarps vectors of length m
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  load_block(as, data + b.a, m, n, b.lda);
  const int kk = m < n ? m : n;
  for (int j = 0; j < kk; ++j) {
    // exact remaining column norms, pivot = first maximum
    for (int c = j + warp; c < n; c += kQrWarps) {
      const double* ac = as + c * m;
      double s = 0.0;
      for (int i = j + lane; i < m; i += 32) s = fma(ac[i], ac[i], s);
      s = warp_sum(s);
      if (lane == 0) norms[c] = s;
    }
    __syncthreads();
    int p = j;
    double best = norms[j];
    for (int c = j + 1; c < n; ++c)
      if (norms[c] > best) { best = norms[c]; p = c; }
    if (p != j) {
      for (int i = threadIdx.x; i < m; i += kQrThreads) {
        const double t = as[i + j * m];
        as[i + j * m] = as[i + p * m];
        as[i + p * m] = t;
      }
    }
    __syncthreads();
    const double tau = householder_step(as, m, n, j, red);
    if (threadIdx.x == 0) taus[j] = tau;
  }
  if (threadIdx.x == 0) {
    int keep = 0;
    if (kk > 0) {
      const double pivot0 = fabs(as[0]);
      while (keep < kk && fabs(as[keep + keep * m]) > tol * pivot0) ++keep;
    }
    if (keep > kmax) keep = kmax;
    keep_s = keep;
    if (b.rank_slot >= 0) ranks[b.rank_slot] = keep;
  }
  __syncthreads();
  const int keep = keep_s;
  // Q(:, c) = H_0 ... H_c e_c, one column per warp in its own vector.
  double* x = vec + std::int64_t(warp) * m;
  for (int c = warp; c < kmax; c += kQrWarps) {
    double* dst = outbuf + b.out + std::int64_t(c) * b.ldo;
    if (c >= keep) {
      for (int i = lane; i < m; i += 32) dst[i] = 0.0;
      continue;
    }
    for (int i = lane; i < m; i += 32) x[i] = i == c ? 1.0 : 0.0;
    __syncwarp();
    for (int j = c; j >= 0; --j) {
      const double* v = as + j * m;
      double s = lane == 0 ? x[j] : 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) s = fma(v[i], x[i], s);
      s = warp_sum(s) * taus[j];
      __syncwarp();
      if (lane == 0) x[j] -= s;
      for (int i = j + 1 + lane; i < m; i += 32) x[i] = fma(-s, v[i], x[i]);
      __syncwarp();
    }
    for (int i = lane; i < m; i += 32) dst[i] = x[i];
    __syncwarp();
  }
}

// out(rows x kmax) = H_0..H_{kk-1} [C; 0], C = kk x kmax rows of the parent Q.
__global__ void __launch_bounds__(kQrThreads)
qr_backprop_kernel(const QrBlock* __restrict__ blocks, const double* data,
                   const double* __restrict__ tau, const double* parent, double* outbuf, int n,
                   int kmax) {
  extern __shared__ double sm[];
  const QrBlock b = blocks[blockIdx.x];
  const int m = b.rows;
  const int kk = m < n ? m : n;
  double* as = sm;
  double* vec = sm + std::int64_t(m) * kk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < m * kk; e += kQrThreads) {
    const int i = e % m, j = e / m;
    as[e] = data[b.a + i + std::int64_t(j) * b.lda];
  }
  __syncthreads();
  double* x = vec + std::int64_t(warp) * m;
  for (int c = warp; c < kmax; c += kQrWarps) {
    const double* csrc = parent + b.c + std::int64_t(c) * b.ldc;
    for (int i = lane; i < m; i += 32) x[i] = i < kk ? csrc[i] : 0.0;
    __syncwarp();
    for (int j = kk - 1; j >= 0; --j) {
      const double* v = as + j * m;
      double s = lane == 0 ? x[j] : 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) s = fma(v[i], x[i], s);
      s = warp_sum(s) * tau[b.tau + j];
      __syncwarp();
      if (lane == 0) x[j] -= s;
      for (int i = j + 1 + lane; i < m; i += 32) x[i] = fma(-s, v[i], x[i]);
      __syncwarp();
    }
    double* dst = outbuf + b.out + std::int64_t(c) * b.ldo;
    for (int i = lane; i < m; i += 32) dst[i] = x[i];
    __syncwarp();
  }
}

}  // namespace

int qr_rows_max(int cols) {
  const int rows = int(kQrSmemBudget / sizeof(double) / size_t(cols + kQrWarps));
  return std::max(32, std::min(1024, rows / 32 * 32));
}

void launch_qr_chunk(const QrBlock* blocks, int nb, double* data, double* rout, double* tau,
                     int cols, cudaStream_t s) {
  if (nb == 0) return;
  const size_t smem = size_t(qr_rows_max(cols)) * size_t(cols) * sizeof(double);
  HP_CUDA(cudaFuncSetAttribute(qr_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  qr_chunk_kernel<<<nb, kQrThreads, smem, s>>>(blocks, data, rout, tau, cols);
  HP_LAUNCHED();
}

void launch_qr_top(const QrBlock* blocks, int nb, double* data, double* outbuf, int* ranks,
                   int cols, int kmax, double tol, cudaStream_t s) {
  if (nb == 0) return;
  if (cols > 160) throw std::invalid_argument("qr: more than 160 columns");
  const size_t smem = size_t(qr_rows_max(cols)) * size_t(cols + kQrWarps) * sizeof(double);
  HP_CUDA(cudaFuncSetAttribute(qr_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  qr_top_kernel<<<nb, kQrThreads, smem, s>>>(blocks, data, outbuf, ranks, cols, kmax, tol);
  HP_LAUNCHED();
}

void launch_qr_backprop(const QrBlock* blocks, int nb, const double* data, const double* tau,
                        const double* parent, double* outbuf, int cols, int kmax,
                        cudaStream_t s) {
  if (nb == 0) return;
  const size_t smem = size_t(qr_rows_max(cols)) * size_t(cols + kQrWarps) * sizeof(double);
  HP_CUDA(cudaFuncSetAttribute(qr_backprop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  qr_backprop_kernel<<<nb, kQrThreads, smem, s>>>(blocks, data, tau, parent, outbuf, cols, kmax);
  HP_LAUNCHED();
}

}  // namespace hpeel
