// K5 coupling-matrix solve, normal-equations variant (sm_100a).
//
// B = pinv(M1) middle pinv(M2)^T with M1 = G'^T U and M2 = (V^T G)^T
// (proj/src/peeling.cpp:252-269). U and V have orthonormal columns (zero
// columns beyond their kept rank) and G, G' are Gaussian test blocks, so M1
// and M2 are r x k Gaussian matrices on their nonzero columns: full column
// rank with condition numbers ~ (sqrt r + sqrt k) / (sqrt r - sqrt k) (~10-20
// for the configured k, p). For such matrices pinv(M) X = (M^T M)^{-1} M^T X
// through a Cholesky factorization agrees with the SVD-based pinv_apply to
// ~cond^2 eps, and nothing falls under its 1e-12 sigma_1 cutoff. Exactly zero
// columns (rank below k) get zero rows, as the pseudo-inverse gives. Any pair
// whose Cholesky diagonal drops below 1e-2 of its largest entry (condition
// ~1e2 or worse) is flagged and solved by the Jacobi-SVD kernel instead,
// which implements pinv_apply itself.
//
// With N = M^T M the two solves collapse to k x k work,
//   B = N1^-1 (M1^T middle M2) N2^-1,
// done by two kernels per batch of pairs (see bprep_kernel / bfinal_kernel):
// the r-long contractions on DMMA tiles, then a left-looking Cholesky that
// builds X = L^-T alongside (chol.cuh) and N^-1 Y = X (X^T Y) on DMMA tiles
// (the round-1 kernel ran column-per-thread triangular substitutions, a
// 2 k^2-long dependent chain, in one 126 KB CTA per SM). Shared-memory
// leading dimensions are == 4 (mod 16): conflict-free DMMA fragments.
#include <cuda_runtime.h>

#include <cmath>

#include "chol.cuh"
#include "kernels.hpp"

namespace hpeel {

namespace {

constexpr int kBsThreads = 256;
constexpr double kCholFlag = 1e-2;  // min L_jj / max L_jj before falling back

constexpr int kAtbTiles = 16;  // 8 x 8 output tiles per warp held in registers

// C(c, d) = sum_{i < r} P(i, c) Q(i, d), c < m, d < nn, on FP64 DMMA (m8n8k4):
// 8 x 8 tiles over the warps, accumulated in registers, then handed to
// store(c, d, v) after a barrier (so C may overwrite P or Q). P(i, c) =
// P[i * ps_i + c * ps_c], Q likewise. Needs ceil(m/8) ceil(nn/8) <= 8 *
// kAtbTiles (launch_bsolve_reg checks). (Was one scalar FMA chain per output
// with two shared loads per FMA: bound by shared-memory bandwidth.)
template <class Store>
__device__ __forceinline__ void atb_dmma(const double* P, int ps_i, int ps_c, const double* Q, int qs_i, int qs_d,
                                         int r, int m, int nn, Store store) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kWarps = kBsThreads / 32;
  const int ntl = (nn + 7) / 8, ntiles = ((m + 7) / 8) * ntl;
  double acc[kAtbTiles][2];
#pragma unroll
  for (int u = 0; u < kAtbTiles; ++u) {
    acc[u][0] = acc[u][1] = 0.0;
    const int tile = warp + u * kWarps;
    if (tile < ntiles) {
      const int mi = tile / ntl, ni = tile - mi * ntl;
      const int c = mi * 8 + (lane >> 2), d = ni * 8 + (lane >> 2);
      const double* pc = P + c * ps_c;
      const double* qd = Q + d * qs_d;
      for (int kk = 0; kk < r; kk += 4) {
        const int i = kk + (lane & 3);
        const double av = (i < r && c < m) ? pc[i * ps_i] : 0.0;
        const double bv = (i < r && d < nn) ? qd[i * qs_i] : 0.0;
        dmma8x8x4(acc[u][0], acc[u][1], av, bv);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kAtbTiles; ++u) {
    const int tile = warp + u * kWarps;
    if (tile < ntiles) {
      const int mi = tile / ntl, ni = tile - mi * ntl;
      const int c = mi * 8 + (lane >> 2), d = ni * 8 + (lane & 3) * 2;
      if (c < m) {
        if (d < nn) store(c, d, acc[u][0]);
        if (d + 1 < nn) store(c, d + 1, acc[u][1]);
      }
    }
  }
  __syncthreads();
}

// N = L L^T in place (lower, ld ldn) with X = L^-T (upper, k x k, ld ldx)
// built alongside (chol.cuh: one barrier pair per column, rows on threads).
// Exactly zero diagonals mark null columns (zero rows in the solution).
// Returns false when a pivot is negative or small relative to the largest.
__device__ bool cholesky_inv(double* n, int k, int ldn, double* xinv, int ldx, int* status, CholShared& cs) {
  __shared__ int bad;
  double d00 = 0.0;
  int last = 0;
  bool used = false;
  const CholStops stops{0, 0.0, 0.0, 0.0};
  lazy_chol<false>(n, ldn, n, ldn, xinv, ldx, k, 0, k, stops, d00, last, used, cs, status);
  if (threadIdx.x == 0) {
    double dmax = 0.0;
    int b = 0;
    for (int j = 0; j < k; ++j) dmax = fmax(dmax, n[j + j * ldn]);
    for (int j = 0; j < k; ++j)
      if (status[j] == 2 || (status[j] == 0 && n[j + j * ldn] < kCholFlag * dmax)) b = 1;
    bad = b;
  }
  __syncthreads();
  return bad == 0;
}

// y (k x nr, ld ldy) <- N^{-1} y = X (X^T y) on DMMA tiles.
__device__ void chol_solve(const double* xinv, int k, int ldx, double* y, int nr, int ldy) {
  atb_dmma(xinv, 1, ldx, y, 1, ldy, k, k, nr, [&](int c, int d, double v) { y[c + d * ldy] = v; });
  atb_dmma(xinv, ldx, 1, y, 1, ldy, k, k, nr, [&](int c, int d, double v) { y[c + d * ldy] = v; });
}

// B = pinv(M1) middle pinv(M2)^T = N1^-1 (M1^T middle M2) N2^-1 with
// N = M^T M: everything the pair needs beyond this point is k x k.
//
// Kernel 1 (bprep): N1 = M1^T M1, N2 = M2^T M2 and C = (middle^T M1)^T M2 on
// DMMA tiles; middle (r x r) and one M (r x k) in shared memory at a time, so
// two CTAs fit per SM (the fused kernel held M, middle, N and X: one CTA per
// SM, two warps per scheduler, bound by latency).
// Kernel 2 (bfinal): Cholesky of N1 and N2 with X = L^-T alongside, then
// B = X1 X1^T C X2 X2^T on DMMA tiles; three k x k buffers.
__global__ void __launch_bounds__(kBsThreads, 2)
bprep_kernel(const double* __restrict__ gpu_, const double* __restrict__ middle, const double* __restrict__ vg,
             int r, int k, std::int64_t p0, double* __restrict__ work) {
  extern __shared__ double sm[];
  const int ldm = ld4(r);
  double* m = sm;             // M1, then M2: r x k (ld ldm)
  double* x = m + ldm * k;    // middle (r x r, ld ldm), then P = middle^T M1 (r x k, ld ldm)
  const std::int64_t p = p0 + blockIdx.x;
  double* out = work + std::int64_t(blockIdx.x) * 3 * k * k;  // N1, N2, C (k x k each, ld k)
  const int t = threadIdx.x;
  for (int e = t; e < r * k; e += kBsThreads) m[e % r + (e / r) * ldm] = gpu_[p * r * k + e];
  for (int e = t; e < r * r; e += kBsThreads) x[e % r + (e / r) * ldm] = middle[p * r * r + e];
  __syncthreads();
  atb_dmma(m, 1, ldm, m, 1, ldm, r, k, k, [&](int c, int d, double v) {
    if (c >= d) out[c + d * k] = v;
  });
  // P(c, d) = sum_i middle(i, c) M1(i, d), written over middle once every warp has its sums
  atb_dmma(x, 1, ldm, m, 1, ldm, r, r, k, [&](int c, int d, double v) { x[c + d * ldm] = v; });
  for (int e = t; e < r * k; e += kBsThreads) {
    const int i = e % r, c = e / r;  // M2(i, c) = vg(c, i), vg k x r col-major
    m[i + c * ldm] = vg[p * k * r + c + std::int64_t(i) * k];
  }
  __syncthreads();
  atb_dmma(m, 1, ldm, m, 1, ldm, r, k, k, [&](int c, int d, double v) {
    if (c >= d) out[k * k + c + d * k] = v;
  });
  atb_dmma(x, 1, ldm, m, 1, ldm, r, k, k, [&](int c, int d, double v) { out[2 * k * k + c + d * k] = v; });
}

__global__ void __launch_bounds__(kBsThreads, 2)
bfinal_kernel(const double* __restrict__ work, int k, std::int64_t p0, const std::int64_t* __restrict__ boff,
              double* __restrict__ bout, int* __restrict__ flags) {
  extern __shared__ double sm[];
  __shared__ int status[64];
  __shared__ CholShared cs;
  const int ldn = ld4(k);
  double* n = sm;              // N1 then N2 (lower), overwritten by L
  double* xinv = n + ldn * k;  // X = L^-T
  double* c = xinv + ldn * k;  // C -> B
  const std::int64_t p = p0 + blockIdx.x;
  const double* in = work + std::int64_t(blockIdx.x) * 3 * k * k;
  const int t = threadIdx.x;
  for (int e = t; e < k * k; e += kBsThreads) {
    const int i = e % k, j = e / k;
    n[i + j * ldn] = in[e];
    c[i + j * ldn] = in[2 * k * k + e];
  }
  __syncthreads();
  const bool ok1 = cholesky_inv(n, k, ldn, xinv, ldn, status, cs);
  chol_solve(xinv, k, ldn, c, k, ldn);  // C <- N1^-1 C
  for (int e = t; e < k * k; e += kBsThreads) n[e % k + (e / k) * ldn] = in[k * k + e];
  __syncthreads();
  const bool ok2 = cholesky_inv(n, k, ldn, xinv, ldn, status, cs);
  // C <- C X2 X2^T: D(c, d) = sum_i C(c, i) X2(i, d), then sum_i D(c, i) X2(d, i)
  atb_dmma(c, ldn, 1, xinv, 1, ldn, k, k, k, [&](int cc, int d, double v) { c[cc + d * ldn] = v; });
  atb_dmma(c, ldn, 1, xinv, ldn, 1, k, k, k, [&](int cc, int d, double v) { c[cc + d * ldn] = v; });
  const bool ok = ok1 && ok2;
  if (ok)
    for (int e = t; e < k * k; e += kBsThreads) bout[boff[p] + e] = c[e % k + (e / k) * ldn];
  if (t == 0) flags[p] = ok ? 0 : 1;
}

}  // namespace

bool launch_bsolve_reg(int npairs, const double* gpu_, const double* middle, const double* vg, int r, int k,
                       const std::int64_t* boff, double* b, int* flags, cudaStream_t s) {
  if (k > 64 || k > r || r > 96) return false;
  if (((r + 7) / 8) * ((k + 7) / 8) > (kBsThreads / 32) * kAtbTiles) return false;
  const size_t sm1 = size_t(ld4(r)) * (k + r) * sizeof(double);
  const size_t sm2 = size_t(3) * ld4(k) * k * sizeof(double);
  if (sm1 > 220 * 1024 || sm2 > 220 * 1024) return false;
  HP_CUDA(cudaFuncSetAttribute(bprep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm1)));
  HP_CUDA(cudaFuncSetAttribute(bfinal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm2)));
  // pairs in batches: N1, N2, C of a batch live in a workspace of <= 1.5 GB
  const std::int64_t per = std::int64_t(3) * k * k;
  const int batch = int(std::max<std::int64_t>(1, std::min<std::int64_t>(npairs, (std::int64_t(3) << 26) / per)));
  double* work = nullptr;
  HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&work), size_t(batch) * size_t(per) * sizeof(double), s));
  for (std::int64_t p0 = 0; p0 < npairs; p0 += batch) {
    const int nb = int(std::min<std::int64_t>(batch, npairs - p0));
    bprep_kernel<<<nb, kBsThreads, sm1, s>>>(gpu_, middle, vg, r, k, p0, work);
    HP_LAUNCHED();
    bfinal_kernel<<<nb, kBsThreads, sm2, s>>>(work, k, p0, boff, b, flags);
    HP_LAUNCHED();
  }
  HP_CUDA(cudaFreeAsync(work, s));
  return true;
}

}  // namespace hpeel
