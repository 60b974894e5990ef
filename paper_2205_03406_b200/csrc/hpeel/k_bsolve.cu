// K5 coupling-matrix solve (sm_100a): the per-pair B of run_h1
// (proj/src/peeling.cpp:252-269)
//   middle = G'^T Y(I_a)            (r x r)
//   left   = pinv(G'^T U) middle    (k x r)
//   B      = (pinv((V^T G)^T) left^T)^T
// with pinv_apply's SVD cutoff 1e-12 * sigma_1 (proj/src/linalg.cpp:110-127).
// The row reductions (G'^T Y, G'^T U, V^T G) run as chunked Gram tasks with a
// fixed-order partial sum; the pseudo-inverses use one-sided Jacobi SVD in
// shared memory, one CTA per pair.
#include <cuda_runtime.h>

#include <cmath>

#include "kernels.hpp"

namespace hpeel {

namespace {

constexpr int kGramThreads = 256;
constexpr int kGramRows = 32;

// Row stride of a staged operand: >= the 8-padded width and == 4 mod 16
// doubles: a DMMA fragment read is served per half warp (4 rows x 4 columns),
// which then hits 16 distinct bank pairs (== 8 mod 16 gave two-way conflicts
// on half of the shared loads, profiles/r02_ncu_kernels.txt).
__host__ __device__ constexpr int gram_stride(int n) { return ((((n + 7) / 8) * 8 + 11) / 16) * 16 + 4; }

// out (nx x ny, col-major) = X^T Y over t.rows rows, on FP64 DMMA (m8n8k4):
// 32-row chunks of X and Y staged row-major in shared memory (rows past the
// end zeroed), 8 x 8 output tiles spread over the warps, TPW tiles per warp.
// (Was one scalar FMA chain per output element with two shared loads per
// FMA.)
template <int TPW>
__global__ void __launch_bounds__(kGramThreads)
gram_kernel(const GramTask* __restrict__ tasks, const double* __restrict__ xb,
            const double* __restrict__ yb, int nx, int ny, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int XS = gram_stride(nx), YS = gram_stride(ny);
  double* xs = sm;                    // kGramRows x XS (row-major)
  double* ys = sm + kGramRows * XS;   // kGramRows x YS (row-major)
  const GramTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kWarps = kGramThreads / 32;
  const int ntl = (ny + 7) / 8, ntiles = ((nx + 7) / 8) * ntl;
  int ao[TPW], bo[TPW];
  double acc[TPW][2];
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    const int tile = warp + u * kWarps;
    const int mi = tile / ntl, ni = tile - mi * ntl;
    ao[u] = mi * 8 + (lane >> 2);
    bo[u] = ni * 8 + (lane >> 2);
    acc[u][0] = acc[u][1] = 0.0;
  }
  auto stage = [&](double* dst, int ld, int n, const double* src, std::int64_t off, std::int64_t lsrc,
                   bool rowmajor, int r0, int cnt) {
    static_assert(kGramRows == 32, "one lane per chunk row");
    if (rowmajor) {
      for (int i = warp; i < kGramRows; i += kWarps)
        for (int a = lane; a < n; a += 32)
          dst[i * ld + a] = i < cnt ? src[off + std::int64_t(r0 + i) * lsrc + a] : 0.0;
    } else {
      for (int a = warp; a < n; a += kWarps)
        dst[lane * ld + a] = lane < cnt ? src[off + r0 + lane + std::int64_t(a) * lsrc] : 0.0;
    }
  };
  for (int r0 = 0; r0 < t.rows; r0 += kGramRows) {
    const int cnt = t.rows - r0 < kGramRows ? t.rows - r0 : kGramRows;
    __syncthreads();
    stage(xs, XS, nx, xb, t.x, t.lx, t.x_rowmajor, r0, cnt);
    stage(ys, YS, ny, yb, t.y, t.ly, t.y_rowmajor, r0, cnt);
    __syncthreads();
    const int kend = (cnt + 3) & ~3;
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      if (warp + u * kWarps >= ntiles) break;
      const double* ap = xs + (lane & 3) * XS + ao[u];
      const double* bp = ys + (lane & 3) * YS + bo[u];
      for (int kk = 0; kk < kend; kk += 4) dmma8x8x4(acc[u][0], acc[u][1], ap[kk * XS], bp[kk * YS]);
    }
  }
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    if (warp + u * kWarps >= ntiles) break;
    const int m = ao[u], n = bo[u] - (lane >> 2) + (lane & 3) * 2;
    if (m < nx) {
      if (n < ny) out[t.out + m + std::int64_t(n) * nx] = acc[u][0];
      if (n + 1 < ny) out[t.out + m + std::int64_t(n + 1) * nx] = acc[u][1];
    }
  }
}

__global__ void sum_partials_kernel(const std::int64_t* __restrict__ off, const double* src,
                                    int len, double* dst) {
  const int d = blockIdx.x;
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    double s = 0.0;
    for (std::int64_t p = off[d]; p < off[d + 1]; ++p) s += src[p * len + i];
    dst[std::int64_t(d) * len + i] = s;
  }
}

constexpr int kSvdThreads = 256;
constexpr int kSvdWarps = kSvdThreads / 32;

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One-sided Jacobi on the n columns of c (m x n, ld m) with v (n x n) = I
// accumulated: afterwards c = W (orthogonal columns), sigma_j = |W_j|.
// Round-robin pair schedule; warps take disjoint pairs.
__device__ void jacobi(double* c, double* v, int m, int n, int* done) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < n * n; e += kSvdThreads) v[e] = (e % n == e / n) ? 1.0 : 0.0;
  const int np = n + (n & 1);  // even player count (one dummy when n is odd)
  const double conv = 4.0e-16 * sqrt(double(m));
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) *done = 1;
    __syncthreads();
    for (int round = 0; round < np - 1; ++round) {
      for (int pr = warp; pr < np / 2; pr += kSvdWarps) {
        // circle method: player np-1 fixed, others rotate
        int p = pr == 0 ? np - 1 : (round + pr) % (np - 1);
        int q = pr == 0 ? round : (round + np - 1 - pr) % (np - 1);
        if (p >= n || q >= n) continue;
        if (p > q) { const int t = p; p = q; q = t; }
        double* cp = c + p * m;
        double* cq = c + q * m;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = lane; i < m; i += 32) {
          a = fma(cp[i], cp[i], a);
          b = fma(cq[i], cq[i], b);
          g = fma(cp[i], cq[i], g);
        }
        a = wsum(a);
        b = wsum(b);
        g = wsum(g);
        if (g == 0.0 || fabs(g) <= conv * sqrt(a * b)) continue;
        if (lane == 0) *done = 0;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int i = lane; i < m; i += 32) {
          const double x = cp[i], y = cq[i];
          cp[i] = cs * x - sn * y;
          cq[i] = sn * x + cs * y;
        }
        double* vp = v + p * n;
        double* vq = v + q * n;
        for (int i = lane; i < n; i += 32) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
      }
      __syncthreads();
    }
    if (*done) break;
    __syncthreads();
  }
  __syncthreads();
}

// inv2[j] = 1 / sigma_j^2 for sigma_j > tol * sigma_max else 0.
__device__ void pinv_weights(const double* c, int m, int n, double tol, double* inv2) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < n; j += kSvdWarps) {
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s = fma(c[j * m + i], c[j * m + i], s);
    s = wsum(s);
    if (lane == 0) inv2[j] = sqrt(s);
  }
  __syncthreads();
  __shared__ double smax;
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int j = 0; j < n; ++j) mx = fmax(mx, inv2[j]);
    smax = mx;
  }
  __syncthreads();
  const double cut = tol * smax;
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += kSvdThreads) {
    const double sg = inv2[j];
    inv2[j] = sg > cut && sg > 0.0 ? 1.0 / (sg * sg) : 0.0;
  }
  __syncthreads();
}

// Column-pivoted Householder QR of the first `ncand` columns of the m x ntot
// shared matrix a (ld m); every reflector is also applied to the trailing
// columns (right-hand sides), which end up holding Q^T rhs. perm[j] = original
// column at pivot position j; the R diagonal stays on a's diagonal.
__device__ void pivqr_augmented(double* a, int m, int ncand, int ntot, int* perm, double* nrm,
                                double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = threadIdx.x; j < ncand; j += kSvdThreads) perm[j] = j;
  __syncthreads();
  const int kk = m < ncand ? m : ncand;
  for (int j = 0; j < kk; ++j) {
    for (int c = j + warp; c < ncand; c += kSvdWarps) {
      const double* ac = a + c * m;
      double s = 0.0;
      for (int i = j + lane; i < m; i += 32) s = fma(ac[i], ac[i], s);
      s = wsum(s);
      if (lane == 0) nrm[c] = s;
    }
    __syncthreads();
    int p = j;
    double best = nrm[j];
    for (int c = j + 1; c < ncand; ++c)
      if (nrm[c] > best) { best = nrm[c]; p = c; }
    if (p != j) {
      for (int i = threadIdx.x; i < m; i += kSvdThreads) {
        const double t = a[i + j * m];
        a[i + j * m] = a[i + p * m];
        a[i + p * m] = t;
      }
      if (threadIdx.x == 0) {
        const int t = perm[j];
        perm[j] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    // reflector from column j (dlarfg), applied to columns j+1 .. ntot-1
    double* col = a + j * m;
    double part = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += kSvdThreads) part += col[i] * col[i];
    part = wsum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    double sigma = 0.0;
    for (int w = 0; w < kSvdWarps; ++w) sigma += red[w];
    const double alpha = col[j];
    double tau = 0.0;
    if (sigma > 0.0) {
      const double beta = alpha >= 0.0 ? -sqrt(alpha * alpha + sigma) : sqrt(alpha * alpha + sigma);
      tau = (beta - alpha) / beta;
      const double scale = 1.0 / (alpha - beta);
      __syncthreads();
      for (int i = j + 1 + threadIdx.x; i < m; i += kSvdThreads) col[i] *= scale;
      if (threadIdx.x == 0) col[j] = beta;
    }
    __syncthreads();
    if (tau != 0.0) {
      for (int c = j + 1 + warp; c < ntot; c += kSvdWarps) {
        double* ac = a + c * m;
        double s = lane == 0 ? ac[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) s = fma(col[i], ac[i], s);
        s = wsum(s) * tau;
        if (lane == 0) ac[j] -= s;
        for (int i = j + 1 + lane; i < m; i += 32) ac[i] = fma(-s, col[i], ac[i]);
      }
    }
    __syncthreads();
  }
}

// pinv(C) X through the pivoted QR above (C = a[:, :n], X = a[:, n:n+nr]):
// out (n x nr, ld n) = P R^{-1} (Q^T X)[:rank] with zero rows for exactly-zero
// pivots. Returns false (uniformly) when a nonzero |R_jj| <= 1e-10 |R_00|,
// i.e. when the SVD cutoff 1e-12 sigma_1 of pinv_apply could drop a value.
__device__ bool qr_pinv_apply(double* a, int m, int n, int nr, int* perm, double* nrm,
                              double* red, double* out) {
  pivqr_augmented(a, m, n, n + nr, perm, nrm, red);
  const int kk = m < n ? m : n;
  __shared__ int rank_s, ok_s;
  if (threadIdx.x == 0) {
    const double r0 = kk > 0 ? fabs(a[0]) : 0.0;
    int rank = 0;
    int ok = 1;
    while (rank < kk && fabs(a[rank + rank * m]) > 0.0) {
      if (fabs(a[rank + rank * m]) <= 1e-10 * r0) ok = 0;
      ++rank;
    }
    rank_s = rank;
    ok_s = ok;
  }
  __syncthreads();
  const int rank = rank_s;
  for (int e = threadIdx.x; e < n * nr; e += kSvdThreads) out[e] = 0.0;
  __syncthreads();
  for (int c = threadIdx.x; c < nr; c += kSvdThreads) {
    const double* y = a + (n + c) * m;
    for (int i = rank - 1; i >= 0; --i) {
      double s = y[i];
      for (int l = i + 1; l < rank; ++l) s = fma(-a[i + l * m], out[perm[l] + c * n], s);
      out[perm[i] + c * n] = s / a[i + i * m];
    }
  }
  __syncthreads();
  return ok_s != 0;
}

// B for every pair by pivoted-QR least squares; pairs whose conditioning
// could interact with the SVD cutoff are flagged for bsolve_kernel.
__global__ void __launch_bounds__(kSvdThreads)
bsolve_qr_kernel(const double* __restrict__ gpu_, const double* __restrict__ middle,
                 const double* __restrict__ vg, int r, int k, const std::int64_t* __restrict__ boff,
                 double* __restrict__ bout, int* __restrict__ flags) {
  extern __shared__ double sm[];
  double* a = sm;                   // r x (k + max(r, k))
  double* left = a + r * (k + (r > k ? r : k));  // k x r
  double* out2 = left + k * r;      // k x k
  double* nrm = out2 + k * k;       // k
  __shared__ double red[kSvdWarps];
  __shared__ int perm[160];
  const std::int64_t p = blockIdx.x;
  const int tid = threadIdx.x;
  for (int e = tid; e < r * k; e += kSvdThreads) a[e] = gpu_[p * r * k + e];
  for (int e = tid; e < r * r; e += kSvdThreads) a[r * k + e] = middle[p * r * r + e];
  __syncthreads();
  const bool ok1 = qr_pinv_apply(a, r, k, r, perm, nrm, red, left);
  // [ (V^T G)^T | left^T ]
  for (int e = tid; e < r * k; e += kSvdThreads) {
    const int i = e % r, j = e / r;
    a[e] = vg[p * k * r + j + std::int64_t(i) * k];
  }
  for (int e = tid; e < r * k; e += kSvdThreads) {
    const int i = e % r, j = e / r;  // column j of left^T = row j of left
    a[r * k + e] = left[j + i * k];
  }
  __syncthreads();
  const bool ok2 = qr_pinv_apply(a, r, k, k, perm, nrm, red, out2);
  if (ok1 && ok2) {
    for (int e = tid; e < k * k; e += kSvdThreads) {
      const int i = e % k, j = e / k;
      bout[boff[p] + e] = out2[j + i * k];  // B = out2^T
    }
  }
  if (tid == 0) flags[p] = (ok1 && ok2) ? 0 : 1;
}

__global__ void __launch_bounds__(kSvdThreads)
bsolve_kernel(const double* __restrict__ gpu_, const double* __restrict__ middle,
              const double* __restrict__ vg, int r, int k, double tol,
              const std::int64_t* __restrict__ boff, double* __restrict__ bout,
              const int* __restrict__ flags) {
  if (flags && flags[blockIdx.x] == 0) return;
  extern __shared__ double sm[];
  double* c = sm;              // r x k
  double* v = c + r * k;       // k x k
  double* mid = v + k * k;     // r x r
  double* left = mid + r * r;  // k x r
  double* tmp = left + k * r;  // k x r (scratch)
  double* inv2 = tmp + k * r;  // k
  __shared__ int done;
  const std::int64_t p = blockIdx.x;
  const int tid = threadIdx.x;

  // 1) pinv(G'^T U) middle
  for (int e = tid; e < r * k; e += kSvdThreads) c[e] = gpu_[p * r * k + e];
  for (int e = tid; e < r * r; e += kSvdThreads) mid[e] = middle[p * r * r + e];
  __syncthreads();
  jacobi(c, v, r, k, &done);
  pinv_weights(c, r, k, tol, inv2);
  // tmp = diag(inv2) W^T mid  (k x r)
  for (int e = tid; e < k * r; e += kSvdThreads) {
    const int i = e % k, j = e / k;
    double s = 0.0;
    if (inv2[i] != 0.0)
      for (int l = 0; l < r; ++l) s = fma(c[i * r + l], mid[l + j * r], s);
    tmp[e] = s * inv2[i];
  }
  __syncthreads();
  // left = V tmp  (k x r)
  for (int e = tid; e < k * r; e += kSvdThreads) {
    const int i = e % k, j = e / k;
    double s = 0.0;
    for (int l = 0; l < k; ++l) s = fma(v[i + l * k], tmp[l + j * k], s);
    left[e] = s;
  }
  __syncthreads();
  // 2) D = (V^T G)^T = vg^T (r x k)
  for (int e = tid; e < r * k; e += kSvdThreads) {
    const int i = e % r, j = e / r;  // D(i, j) = vg(j, i), vg is k x r col-major
    c[e] = vg[p * k * r + j + std::int64_t(i) * k];
  }
  __syncthreads();
  jacobi(c, v, r, k, &done);
  pinv_weights(c, r, k, tol, inv2);
  // B = left W2 diag(inv2) V2^T : tmp = left W2 (k x k) scaled, then * V2^T
  for (int e = tid; e < k * k; e += kSvdThreads) {
    const int i = e % k, j = e / k;
    double s = 0.0;
    if (inv2[j] != 0.0)
      for (int l = 0; l < r; ++l) s = fma(left[i + l * k], c[j * r + l], s);
    tmp[e] = s * inv2[j];
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += kSvdThreads) {
    const int i = e % k, j = e / k;
    double s = 0.0;
    for (int l = 0; l < k; ++l) s = fma(tmp[i + l * k], v[j + l * k], s);
    bout[boff[p] + e] = s;
  }
}

}  // namespace

void launch_gram(const GramTask* tasks, int ntasks, const double* xbase, const double* ybase,
                 int nx, int ny, double* out, cudaStream_t s) {
  if (ntasks == 0) return;
  const int e = (((nx + 7) / 8) * ((ny + 7) / 8) + kGramThreads / 32 - 1) / (kGramThreads / 32);  // tiles per warp
  const size_t smem = size_t(kGramRows) * size_t(gram_stride(nx) + gram_stride(ny)) * sizeof(double);
#define HP_G(EE)                                                                            \
  if (e <= EE) {                                                                            \
    HP_CUDA(cudaFuncSetAttribute(gram_kernel<EE>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 int(smem)));                                               \
    gram_kernel<EE><<<ntasks, kGramThreads, smem, s>>>(tasks, xbase, ybase, nx, ny, out);   \
    HP_LAUNCHED();                                                            \
    return;                                                                                 \
  }
  HP_G(1) HP_G(2) HP_G(4) HP_G(8) HP_G(13) HP_G(18) HP_G(25) HP_G(32)
#undef HP_G
  throw std::invalid_argument("gram block too large (more than 256 output tiles)");
}

void launch_sum_partials(const std::int64_t* off, int ndst, const double* src, int len,
                         double* dst, cudaStream_t s) {
  if (ndst == 0) return;
  sum_partials_kernel<<<ndst, 128, 0, s>>>(off, src, len, dst);
  HP_LAUNCHED();
}

void launch_bsolve(int npairs, const double* gpu_, const double* middle, const double* vg, int r,
                   int k, double tol, const std::int64_t* boff, double* b, cudaStream_t s) {
  if (npairs == 0) return;
  if (r > 160 || k > 160) throw std::invalid_argument("bsolve: widths above 160 unsupported");
  int* flags = nullptr;
  HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flags), size_t(npairs) * sizeof(int), s));
  if (!launch_bsolve_reg(npairs, gpu_, middle, vg, r, k, boff, b, flags, s)) {
    const size_t smem_qr =
        size_t(r * (k + std::max(r, k)) + k * r + k * k + k) * sizeof(double);
    HP_CUDA(cudaFuncSetAttribute(bsolve_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_qr)));
    bsolve_qr_kernel<<<npairs, kSvdThreads, smem_qr, s>>>(gpu_, middle, vg, r, k, boff, b, flags);
    HP_LAUNCHED();
  }
  // fallback: one-sided Jacobi SVD with the 1e-12 cutoff for flagged pairs
  const size_t smem = size_t(r * k + k * k + r * r + 2 * k * r + k) * sizeof(double);
  HP_CUDA(cudaFuncSetAttribute(bsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  bsolve_kernel<<<npairs, kSvdThreads, smem, s>>>(gpu_, middle, vg, r, k, tol, boff, b, flags);
  HP_LAUNCHED();
  HP_CUDA(cudaFreeAsync(flags, s));
}

}  // namespace hpeel
