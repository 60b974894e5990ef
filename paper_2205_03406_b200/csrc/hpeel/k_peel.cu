// K3 peeling subtraction (sm_100a): the level-truncated H1 apply
// A^(l-1) Omega_c of H1Rep::apply_truncated(_adjoint)
// (proj/src/hmatrix.cpp:86-116), restricted to the sample rows the driver
// reads and to the nonzero rows of Omega_c.
//
// For a coarse pair q = (x, y) and a color c the reference computes
// U_q (B_q (V_q^T Omega_c(I_y))) for every color over all N rows. Here
// coefficient tasks form T_{q,c} = B_q * sum_{v in P_c, v in y} V_q[v]^T G_v
// once (k x r), and apply tasks subtract U_q[rows of a] T_{q,c} from each
// level-l sample block whose box a lies under x.
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace hpeel {

namespace {

constexpr int kCoeffThreads = 256;

// M (k x w) accumulated in registers, E entries per thread; then T = op(B) M
// through shared memory.
template <int E>
__global__ void __launch_bounds__(kCoeffThreads)
peel_coeff_kernel(const CoeffTask* __restrict__ tasks, const double* __restrict__ factors,
                  const double* __restrict__ bmat, const std::int64_t* __restrict__ seg_start,
                  const std::int64_t* __restrict__ seg_count, const double* __restrict__ g,
                  int gld, int gcol0, int k, int w, double* __restrict__ tbuf) {
  extern __shared__ double sm[];  // k*w (M) then k*k (B)
  const CoeffTask task = tasks[blockIdx.x];
  const int tid = threadIdx.x;
  const int kw = k * w;
  double acc[E];
#pragma unroll
  for (int u = 0; u < E; ++u) acc[u] = 0.0;
  const double* f = factors + task.f;

  for (int sg = task.seg_begin; sg < task.seg_end; ++sg) {
    const std::int64_t s0 = seg_start[sg] - task.f_row0;
    const std::int64_t cnt = seg_count[sg];
    if (gcol0 >= 0) {
      // Gaussian payload: M[i][c] += sum_t F[s0+t][i] * G[pos][c]
      for (std::int64_t t = 0; t < cnt; ++t) {
        const std::int64_t row = s0 + t;
        const double* grow = g + (seg_start[sg] + t) * gld + gcol0;
#pragma unroll
        for (int u = 0; u < E; ++u) {
          const int e = tid + u * kCoeffThreads;
          if (e < kw) {
            const int i = e % k, c = e / k;
            acc[u] = fma(f[row + std::int64_t(i) * task.frows], grow[c], acc[u]);
          }
        }
      }
    } else {
      // Identity payload [I | 0]: M[i][t] += F[s0+t][i] for t < min(cnt, w)
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const int e = tid + u * kCoeffThreads;
        if (e < kw) {
          const int i = e % k, c = e / k;
          if (c < cnt) acc[u] += f[s0 + c + std::int64_t(i) * task.frows];
        }
      }
    }
  }
  double* ms = sm;
  double* bs = sm + kw;
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const int e = tid + u * kCoeffThreads;
    if (e < kw) ms[e] = acc[u];  // (i, c) at i + c*k: col-major k x w
  }
  for (int e = tid; e < k * k; e += kCoeffThreads) bs[e] = bmat[task.b + e];
  __syncthreads();
  for (int e = tid; e < kw; e += kCoeffThreads) {
    const int i = e % k, c = e / k;
    double t = 0.0;
    if (task.btrans) {
      for (int l = 0; l < k; ++l) t = fma(bs[l + i * k], ms[l + c * k], t);
    } else {
      for (int l = 0; l < k; ++l) t = fma(bs[i + l * k], ms[l + c * k], t);
    }
    tbuf[task.t_out + e] = t;
  }
}

constexpr int kApplyThreads = 256;
constexpr int kApplyRows = 64;

// acc (64 x w) in registers (E = ceil(64 w / 256) entries per thread).
template <int E>
__global__ void __launch_bounds__(kApplyThreads)
peel_apply_kernel(const PeelTask* __restrict__ tasks, const PeelTerm* __restrict__ terms,
                  const double* __restrict__ factors, const double* __restrict__ tbuf, int k,
                  int w, double* __restrict__ out, int ocol0, double alpha) {
  extern __shared__ double sm[];  // F tile (64 x k, col-major) then T (k x w)
  double* fs = sm;
  double* ts = sm + kApplyRows * k;
  const PeelTask task = tasks[blockIdx.x];
  const int tid = threadIdx.x;
  double acc[E];
#pragma unroll
  for (int u = 0; u < E; ++u) acc[u] = 0.0;
  for (int q = task.term_begin; q < task.term_end; ++q) {
    const PeelTerm term = terms[q];
    __syncthreads();
    for (int e = tid; e < kApplyRows * k; e += kApplyThreads) {
      const int i = e % kApplyRows, l = e / kApplyRows;
      fs[e] = i < task.rows ? factors[term.f + i + std::int64_t(l) * term.fld] : 0.0;
    }
    for (int e = tid; e < k * w; e += kApplyThreads) ts[e] = tbuf[term.t + e];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < E; ++u) {
      const int e = tid + u * kApplyThreads;
      const int i = e % kApplyRows, c = e / kApplyRows;
      if (c < w) {
        double t = acc[u];
        for (int l = 0; l < k; ++l) t = fma(fs[i + l * kApplyRows], ts[l + c * k], t);
        acc[u] = t;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const int e = tid + u * kApplyThreads;
    const int i = e % kApplyRows, c = e / kApplyRows;
    if (c < w && i < task.rows) out[task.out + i + std::int64_t(ocol0 + c) * task.ld] += alpha * acc[u];
  }
}

}  // namespace

void launch_peel_coeff(const CoeffTask* tasks, int ntasks, const double* factors,
                       const double* bmat, const std::int64_t* seg_start,
                       const std::int64_t* seg_count, const double* g, int gld, int gcol0, int k,
                       int w, double* tbuf, cudaStream_t s) {
  if (ntasks == 0) return;
  const int e = (k * w + kCoeffThreads - 1) / kCoeffThreads;
  const size_t smem = size_t(k * w + k * k) * sizeof(double);
#define HP_C(EE)                                                                              \
  if (e <= EE) {                                                                              \
    HP_CUDA(cudaFuncSetAttribute(peel_coeff_kernel<EE>,                                       \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));    \
    peel_coeff_kernel<EE><<<ntasks, kCoeffThreads, smem, s>>>(tasks, factors, bmat, seg_start, \
                                                              seg_count, g, gld, gcol0, k, w, tbuf); \
    HP_CUDA(cudaGetLastError());                                                              \
    return;                                                                                   \
  }
  HP_C(2) HP_C(4) HP_C(8) HP_C(12) HP_C(16) HP_C(24) HP_C(32) HP_C(48) HP_C(64)
#undef HP_C
  throw std::invalid_argument("peel coefficient block too large (k * w > 16384)");
}

void launch_peel_apply(const PeelTask* tasks, int ntasks, const PeelTerm* terms,
                       const double* factors, const double* tbuf, int k, int w, double* out,
                       int ocol0, double alpha, cudaStream_t s) {
  if (ntasks == 0) return;
  const int e = (kApplyRows * w + kApplyThreads - 1) / kApplyThreads;
  const size_t smem = size_t(kApplyRows * k + k * w) * sizeof(double);
#define HP_A(EE)                                                                              \
  if (e <= EE) {                                                                              \
    HP_CUDA(cudaFuncSetAttribute(peel_apply_kernel<EE>,                                       \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));    \
    peel_apply_kernel<EE><<<ntasks, kApplyThreads, smem, s>>>(tasks, terms, factors, tbuf, k, w, \
                                                              out, ocol0, alpha);                    \
    HP_CUDA(cudaGetLastError());                                                              \
    return;                                                                                   \
  }
  HP_A(2) HP_A(4) HP_A(8) HP_A(12) HP_A(16) HP_A(20) HP_A(24) HP_A(32) HP_A(48) HP_A(64)
#undef HP_A
  throw std::invalid_argument("peel apply width too large (w > 256)");
}

}  // namespace hpeel
