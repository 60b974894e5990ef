// K4 batched range finder (sm_100a): qr_orthonormal of every sample block
// (proj/src/linalg.cpp:53-78, via basis_from_sample proj/src/peeling.cpp:63-71).
//
// Blocks that fit in shared memory run column-pivoted Householder QR in one
// CTA (the ColPivHouseholderQR rule: pivot = largest remaining column norm,
// first index on ties; keep = leading |R_jj| > 1e-14 |R_00|, capped at k) and
// form Q(:, :keep) in place (LAPACK dorg2r order). Taller blocks go through
// TSQR: unpivoted Householder QR of row chunks, the stacked R factors are
// reduced the same way, the top is pivoted; in exact arithmetic this selects
// the same pivots and span as pivoted QR of the whole block. Q is then
// back-propagated through the chunk reflectors.
//
// Every reflector application runs over a warp's columns in groups of kGroup
// independent dot/axpy chains (the latency of one column's shuffle reduction
// hides behind the others); column norms for the next pivot are accumulated
// in the same pass, and pivoting permutes column indices instead of data.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "kernels.hpp"

namespace hpeel {

namespace {

constexpr int kQrThreads = 256;
constexpr int kQrWarps = kQrThreads / 32;
constexpr int kGroup = 12;  // columns per warp per pass (independent chains)
constexpr size_t kQrSmemBudget = 216 * 1024;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Generate the reflector of column `col` (m rows, pivot row j) by one warp:
// LAPACK dlarfg, v(j) = 1 implicit, v(j+1:) stored in place, col[j] = beta.
__device__ __forceinline__ double make_reflector(double* col, int m, int j, int lane) {
  double part = 0.0;
  for (int i = j + 1 + lane; i < m; i += 32) part = fma(col[i], col[i], part);
  const double sigma = warp_sum(part);
  const double alpha = col[j];
  double tau = 0.0;
  if (sigma > 0.0) {
    const double beta = alpha >= 0.0 ? -sqrt(alpha * alpha + sigma) : sqrt(alpha * alpha + sigma);
    tau = (beta - alpha) / beta;
    const double scale = 1.0 / (alpha - beta);
    for (int i = j + 1 + lane; i < m; i += 32) col[i] *= scale;
    __syncwarp();
    if (lane == 0) col[j] = beta;
  }
  __syncwarp();
  return tau;
}

// Apply H = I - tau v v^T (v = column vcol, rows j.., v(j) = 1) to the
// columns idx[0..nc) of a (ld m), warps [w0, w0 + nw) taking contiguous
// column ranges processed kGroup at a time. With NORMS, nrm[idx[c]] receives
// the squared norm of rows j+1.. of the updated column.
template <bool NORMS>
__device__ void apply_reflector(double* a, int m, const double* vcol, int j, double tau,
                                const int* idx, int nc, double* nrm, int w0 = 0,
                                int nw = kQrWarps) {
  const int warp = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
  if (warp < 0 || warp >= nw || nc <= 0) return;
  const int per = (nc + nw - 1) / nw;
  const int c_end = min(nc, (warp + 1) * per);
  for (int base = warp * per; base < c_end; base += kGroup) {
    double* col[kGroup];
    bool ok[kGroup];
    double s[kGroup];
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      const int c = base + g;
      ok[g] = c < c_end;
      col[g] = a + std::int64_t(ok[g] ? idx[c] : idx[base]) * m;
      s[g] = 0.0;
    }
    if (tau != 0.0) {
      for (int i = j + lane; i < m; i += 32) {
        const double vi = i == j ? 1.0 : vcol[i];
#pragma unroll
        for (int g = 0; g < kGroup; ++g) s[g] = fma(vi, col[g][i], s[g]);
      }
#pragma unroll
      for (int g = 0; g < kGroup; ++g) s[g] = warp_sum(s[g]) * tau;
    }
    double q[kGroup];
#pragma unroll
    for (int g = 0; g < kGroup; ++g) q[g] = 0.0;
    for (int i = j + lane; i < m; i += 32) {
      const double vi = i == j ? 1.0 : vcol[i];
#pragma unroll
      for (int g = 0; g < kGroup; ++g) {
        if (!ok[g]) continue;
        const double x = tau != 0.0 ? fma(-s[g], vi, col[g][i]) : col[g][i];
        if (tau != 0.0) col[g][i] = x;
        if (NORMS && i > j) q[g] = fma(x, x, q[g]);
      }
    }
    if (NORMS) {
#pragma unroll
      for (int g = 0; g < kGroup; ++g) {
        q[g] = warp_sum(q[g]);
        if (ok[g] && lane == 0) nrm[idx[base + g]] = q[g];
      }
    }
  }
}

// Unpivoted (PIVOT = false) or column-pivoted Householder QR of the m x n
// block in shared memory. perm[j] = physical column of pivot position j;
// tau[j] per reflector. Returns min(m, n) reflectors.
template <bool PIVOT>
__device__ int factor(double* a, int m, int n, int* perm, double* tau, double* nrm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < n; c += kQrThreads) perm[c] = c;
  __syncthreads();
  if (PIVOT) {
    // initial squared column norms
    for (int base = warp; base < n; base += kQrWarps * kGroup) {
      double q[kGroup];
#pragma unroll
      for (int g = 0; g < kGroup; ++g) {
        const int c = base + g * kQrWarps;
        q[g] = 0.0;
        if (c < n)
          for (int i = lane; i < m; i += 32) q[g] = fma(a[i + std::int64_t(c) * m], a[i + std::int64_t(c) * m], q[g]);
      }
#pragma unroll
      for (int g = 0; g < kGroup; ++g) {
        q[g] = warp_sum(q[g]);
        if (base + g * kQrWarps < n && lane == 0) nrm[base + g * kQrWarps] = q[g];
      }
    }
    __syncthreads();
  }
  const int kk = m < n ? m : n;
  if (!PIVOT) {
    // look-ahead: warp 0 updates column j + 1 and builds reflector j + 1
    // while warps 1.. update the rest, one barrier per column
    if (kk > 0 && warp == 0) {
      const double t = make_reflector(a, m, 0, lane);
      if (lane == 0) tau[0] = t;
    }
    __syncthreads();
    for (int j = 0; j < kk; ++j) {
      const double* col = a + std::int64_t(j) * m;
      if (j + 1 < kk) {
        apply_reflector<false>(a, m, col, j, tau[j], perm + j + 1, 1, nullptr, 0, 1);
        if (warp == 0) {
          const double t = make_reflector(a + std::int64_t(j + 1) * m, m, j + 1, lane);
          if (lane == 0) tau[j + 1] = t;
        }
        apply_reflector<false>(a, m, col, j, tau[j], perm + j + 2, n - j - 2, nullptr, 1, kQrWarps - 1);
      } else {
        apply_reflector<false>(a, m, col, j, tau[j], perm + j + 1, n - j - 1, nullptr);
      }
      __syncthreads();
    }
    return kk;
  }
  for (int j = 0; j < kk; ++j) {
    if (PIVOT) {
      if (threadIdx.x == 0) {
        int p = j;
        double best = nrm[perm[j]];
        for (int c = j + 1; c < n; ++c)
          if (nrm[perm[c]] > best) {
            best = nrm[perm[c]];
            p = c;
          }
        const int t = perm[j];
        perm[j] = perm[p];
        perm[p] = t;
      }
      __syncthreads();
    }
    double* col = a + std::int64_t(perm[j]) * m;
    if (warp == 0) {
      const double t = make_reflector(col, m, j, lane);
      if (lane == 0) tau[j] = t;
    }
    __syncthreads();
    apply_reflector<PIVOT>(a, m, col, j, tau[j], perm + j + 1, n - j - 1, nrm);
    __syncthreads();
  }
  return kk;
}

// Q(:, 0:q) in place over the first q pivot columns (dorg2r order).
__device__ void form_q(double* a, int m, int q, const int* perm, const double* tau) {
  for (int j = q - 1; j >= 0; --j) {
    double* col = a + std::int64_t(perm[j]) * m;
    apply_reflector<false>(a, m, col, j, tau[j], perm + j + 1, q - j - 1, nullptr);
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += kQrThreads) {
      if (i < j) col[i] = 0.0;
      else if (i == j) col[i] = 1.0 - tau[j];
      else col[i] = -tau[j] * col[i];
    }
    __syncthreads();
  }
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
  __shared__ int perm[160];
  __shared__ double taus[160];
  const QrBlock b = blocks[blockIdx.x];
  const int m = b.rows;
  double* as = sm;
  load_block(as, data + b.a, m, n, b.lda);
  const int kk = factor<false>(as, m, n, perm, taus, nullptr);
  for (int j = threadIdx.x; j < kk; j += kQrThreads) tau_out[b.tau + j] = taus[j];
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
  __shared__ int perm[160];
  __shared__ double taus[160];
  __shared__ double nrm[160];
  __shared__ int keep_s;
  const QrBlock b = blocks[blockIdx.x];
  const int m = b.rows;
  double* as = sm;
  load_block(as, data + b.a, m, n, b.lda);
  const int kk = factor<true>(as, m, n, perm, taus, nrm);
  if (threadIdx.x == 0) {
    int keep = 0;
    if (kk > 0) {
      const double pivot0 = fabs(as[std::int64_t(perm[0]) * m]);
      while (keep < kk && fabs(as[keep + std::int64_t(perm[keep]) * m]) > tol * pivot0) ++keep;
    }
    if (keep > kmax) keep = kmax;
    keep_s = keep;
    if (b.rank_slot >= 0) ranks[b.rank_slot] = keep;
  }
  __syncthreads();
  const int keep = keep_s;
  form_q(as, m, keep, perm, taus);
  for (int e = threadIdx.x; e < m * kmax; e += kQrThreads) {
    const int i = e % m, c = e / m;
    outbuf[b.out + i + std::int64_t(c) * b.ldo] = c < keep ? as[i + std::int64_t(perm[c]) * m] : 0.0;
  }
}

// out(rows x kmax) = H_0..H_{kk-1} [C; 0], C = kk x kmax rows of the parent Q;
// X staged in shared memory, reflectors streamed one at a time.
__global__ void __launch_bounds__(kQrThreads)
qr_backprop_kernel(const QrBlock* __restrict__ blocks, const double* data,
                   const double* __restrict__ tau, const double* parent, double* outbuf, int n,
                   int kmax) {
  extern __shared__ double sm[];
  __shared__ int idx[160];
  const QrBlock b = blocks[blockIdx.x];
  const int m = b.rows;
  const int kk = m < n ? m : n;
  double* xs = sm;                          // m x kmax
  double* vs = sm + std::int64_t(m) * kmax;  // 2 x m reflector buffer
  for (int e = threadIdx.x; e < m * kmax; e += kQrThreads) {
    const int i = e % m, c = e / m;
    xs[e] = i < kk ? parent[b.c + i + std::int64_t(c) * b.ldc] : 0.0;
  }
  for (int c = threadIdx.x; c < kmax; c += kQrThreads) idx[c] = c;
  if (kk > 0)
    for (int i = threadIdx.x; i < m; i += kQrThreads)
      vs[((kk - 1) & 1) * m + i] = data[b.a + i + std::int64_t(kk - 1) * b.lda];
  __syncthreads();
  for (int j = kk - 1; j >= 0; --j) {
    // prefetch the next reflector into the other buffer
    if (j > 0)
      for (int i = threadIdx.x; i < m; i += kQrThreads)
        vs[((j - 1) & 1) * m + i] = data[b.a + i + std::int64_t(j - 1) * b.lda];
    apply_reflector<false>(xs, m, vs + (j & 1) * m, j, tau[b.tau + j], idx, kmax, nullptr);
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * kmax; e += kQrThreads) {
    const int i = e % m, c = e / m;
    outbuf[b.out + i + std::int64_t(c) * b.ldo] = xs[e];
  }
}

size_t smem_for(size_t doubles) { return std::max<size_t>(doubles, 1) * sizeof(double); }

}  // namespace

int qr_rows_max(int cols) {
  const int rows = int(kQrSmemBudget / sizeof(double) / size_t(cols));
  return std::max(32, std::min(1024, rows / 32 * 32));
}

int qr_chunk_rows(int cols, int kmax) {
  const int rows = int(kQrSmemBudget / sizeof(double) / size_t(kmax + 2));
  return std::min(qr_rows_max(cols), std::max(32, std::min(1024, rows / 32 * 32)));
}

void launch_qr_chunk(const QrBlock* blocks, int nb, double* data, double* rout, double* tau,
                     int cols, int max_rows, cudaStream_t s) {
  if (nb == 0) return;
  const size_t smem = smem_for(size_t(max_rows) * size_t(cols));
  HP_CUDA(cudaFuncSetAttribute(qr_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  qr_chunk_kernel<<<nb, kQrThreads, smem, s>>>(blocks, data, rout, tau, cols);
  HP_LAUNCHED();
}

void launch_qr_top(const QrBlock* blocks, int nb, double* data, double* outbuf, int* ranks,
                   int cols, int kmax, double tol, int max_rows, cudaStream_t s) {
  if (nb == 0) return;
  if (cols > 160) throw std::invalid_argument("qr: more than 160 columns");
  const size_t smem = smem_for(size_t(max_rows) * size_t(cols));
  HP_CUDA(cudaFuncSetAttribute(qr_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  qr_top_kernel<<<nb, kQrThreads, smem, s>>>(blocks, data, outbuf, ranks, cols, kmax, tol);
  HP_LAUNCHED();
}

void launch_qr_backprop(const QrBlock* blocks, int nb, const double* data, const double* tau,
                        const double* parent, double* outbuf, int cols, int kmax, int max_rows,
                        cudaStream_t s) {
  if (nb == 0) return;
  const size_t smem = smem_for(size_t(max_rows) * size_t(kmax + 2));
  HP_CUDA(cudaFuncSetAttribute(qr_backprop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  qr_backprop_kernel<<<nb, kQrThreads, smem, s>>>(blocks, data, tau, parent, outbuf, cols, kmax);
  HP_LAUNCHED();
}

}  // namespace hpeel
