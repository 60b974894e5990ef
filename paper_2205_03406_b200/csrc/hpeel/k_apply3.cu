// K2 colored black-box apply, fused variant (sm_100a): every warp evaluates
// its own kernel entries straight into the DMMA A fragments and runs the
// DMMAs on them, instead of handing kernel tiles from evaluation warps to
// DMMA warps through shared memory (k_apply2.cu). Same contract as
// launch_sample_apply (kernels.hpp); replaces the same reference step
// (residual_samples, proj/src/peeling.cpp:165-170).
//
// Why: the kernel evaluation (12 FP64 ops per entry) and the DMMA share the
// one FP64 datapath. With separate warps the hand-off couples them through
// barriers and the datapath idles whenever one side waits; inside one warp
// the evaluation of k-step s+1 is independent of the DMMAs of k-step s, so
// the scheduler interleaves both streams and no kernel tile touches smem.
#include <cuda_runtime.h>

#include "async.cuh"
#include "kernels.hpp"

namespace hpeel {

namespace {

constexpr int kFK = 32;  // payload rows per ring stage (8 DMMA k-steps)
constexpr int kFStages = 4;

__host__ __device__ constexpr int fstride(int nt) { return nt * 8 + 4; }

__host__ __device__ constexpr size_t fused_smem_bytes(int nt) {
  return size_t(kFStages) * kFK * fstride(nt) * sizeof(double);
}

/// CTA = WARPS warps x 16 rows; the lane owning A-fragment element
/// (row lane/4 [+8], k lane%4) evaluates K(row, payload row k) itself.
template <int NT, int KIND, int DIM, bool TRANS, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, WARPS <= 8 ? 2 : 1)
fused_apply_kernel(DevOp op, const K2Task* __restrict__ tasks, const K2Row* __restrict__ rowtab,
                   const std::int64_t* __restrict__ pay_off, const int* __restrict__ pc,
                   const double* __restrict__ gc, int gld, int gcol0, int ncols,
                   const double* __restrict__ xc, std::int64_t nnz, double* __restrict__ out,
                   int ocol0) {
  constexpr int S = fstride(NT);
  constexpr int D = DIM > 0 ? DIM : 1;
  constexpr int kThreads = WARPS * 32;
  extern __shared__ __align__(16) double gsm[];  // [kFStages][kFK * S] payload ring
  __shared__ __align__(16) double xs[kFStages][D][kFK];
  __shared__ __align__(16) int js[kFStages][kFK];
  const double* lts = op.ltab;  // half_log table read through L1

  const K2Task task = tasks[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::int64_t n = op.n;

  for (int e = tid; e < kFStages * kFK * S; e += kThreads) gsm[e] = 0.0;
  for (int e = tid; e < kFStages * kFK; e += kThreads) {
    (&js[0][0])[e] = -1;
    for (int d = 0; d < D; ++d) xs[e / kFK][d][e % kFK] = 0.0;
  }

  // this lane's two A rows and their points
  const int r0 = warp * 16 + (lane >> 2), r1 = r0 + 8;
  const int ip0 = k2_row(task, rowtab, r0 < task.rows ? r0 : task.rows - 1).pos;
  const int ip1 = k2_row(task, rowtab, r1 < task.rows ? r1 : task.rows - 1).pos;
  double xi0[D], xi1[D];
  if constexpr (KIND != kOpDense) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      xi0[d] = op.x[d * n + ip0];
      xi1[d] = op.x[d * n + ip1];
    }
  }
  __syncthreads();

  const std::int64_t p0 = pay_off[task.color], p1 = pay_off[task.color + 1];
  const int nchunks = int((p1 - p0 + kFK - 1) / kFK);
  const bool even_cols = ((gld | gcol0 | ncols) & 1) == 0;

  auto load_chunk = [&](int c) {
    if (c < nchunks) {
      const int st = c % kFStages;
      const std::int64_t base = p0 + std::int64_t(c) * kFK;
      const int cnt = int(p1 - base < kFK ? p1 - base : kFK);
      if (tid < cnt) {
        cp_async4(&js[st][tid], pc + base + tid);
        if constexpr (KIND != kOpDense) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) cp_async8(&xs[st][d][tid], xc + d * nnz + base + tid);
        }
      }
      double* gb = gsm + st * kFK * S;
      const double* gsrc = gc + base * gld + gcol0;
      if (even_cols) {
        const int half = ncols >> 1;
        for (int idx = tid; idx < cnt * half; idx += kThreads) {
          const int t = idx / half, cc = (idx - t * half) * 2;
          cp_async16(gb + t * S + cc, gsrc + std::int64_t(t) * gld + cc);
        }
      } else {
        for (int idx = tid; idx < cnt * ncols; idx += kThreads) {
          const int t = idx / ncols, cc = idx - t * ncols;
          cp_async8(gb + t * S + cc, gsrc + std::int64_t(t) * gld + cc);
        }
      }
    }
    cp_async_commit();  // one group per chunk slot, empty past the end
  };

  // K(row, payload row `col` of stage st) for both A rows; 0 past the chunk end
  auto eval2 = [&](int st, int col, int cnt, double& a0, double& a1) {
    const int jp = js[st][col];
    if constexpr (KIND == kOpDense) {
      const int jj0 = col < cnt ? jp : ip0, jj1 = col < cnt ? jp : ip1;
      const double v0 = TRANS ? op.a[std::int64_t(jj0) + std::int64_t(ip0) * n]
                              : op.a[std::int64_t(ip0) + std::int64_t(jj0) * n];
      const double v1 = TRANS ? op.a[std::int64_t(jj1) + std::int64_t(ip1) * n]
                              : op.a[std::int64_t(ip1) + std::int64_t(jj1) * n];
      a0 = col < cnt ? v0 : 0.0;
      a1 = col < cnt ? v1 : 0.0;
    } else {
      double xj[D];
#pragma unroll
      for (int d = 0; d < DIM; ++d) xj[d] = xs[st][d][col];
      const double v0 = kernel_value<KIND, DIM>(xi0, xj, ip0 == jp, op.param, lts);
      const double v1 = kernel_value<KIND, DIM>(xi1, xj, ip1 == jp, op.param, lts);
      a0 = col < cnt ? v0 : 0.0;
      a1 = col < cnt ? v1 : 0.0;
    }
  };

  double acc[2][NT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;

#pragma unroll
  for (int c = 0; c < kFStages - 1; ++c) load_chunk(c);

  const int kc = lane & 3;
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<kFStages - 2>();  // chunk c landed (this thread's copies)
    __syncthreads();                // ... everyone's; and stage (c-1) is free
    load_chunk(c + kFStages - 1);
    const int st = c % kFStages;
    const int cnt = int(p1 - p0 - std::int64_t(c) * kFK < kFK ? p1 - p0 - std::int64_t(c) * kFK : kFK);
    const double* brow = gsm + st * kFK * S + kc * S + (lane >> 2);
    double a0, a1;
    eval2(st, kc, cnt, a0, a1);
#pragma unroll
    for (int kk = 0; kk < kFK / 4; ++kk) {
      double n0 = 0.0, n1 = 0.0;
      if (kk + 1 < kFK / 4) eval2(st, (kk + 1) * 4 + kc, cnt, n0, n1);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double bb = brow[kk * 4 * S + nt * 8];
        dmma8x8x4(acc[0][nt][0], acc[0][nt][1], a0, bb);
        dmma8x8x4(acc[1][nt][0], acc[1][nt][1], a1, bb);
      }
      a0 = n0;
      a1 = n1;
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int rr = warp * 16 + m * 8 + (lane >> 2);
    if (rr >= task.rows) continue;
    const K2Row dst = k2_row(task, rowtab, rr);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = nt * 8 + (lane & 3) * 2 + h;
        if (c < ncols) out[dst.out + std::int64_t(ocol0 + c) * dst.ld] = acc[m][nt][h];
      }
    }
  }
}

template <int NT, int KIND, int DIM>
void fused_kind_dim(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab,
                    int ntasks, const std::int64_t* pay_off, const int* pc, const double* gc,
                    int gld, int gcol0, int ncols, const double* xc, std::int64_t nnz, double* out,
                    int ocol0, cudaStream_t s) {
  constexpr int W = kFusedRows / 16;
  constexpr size_t smem = fused_smem_bytes(NT);
  if (KIND == kOpDense && trans) {
    auto* fn = fused_apply_kernel<NT, KIND, DIM, KIND == kOpDense, W>;
    HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn<<<ntasks, W * 32, smem, s>>>(op, tasks, rowtab, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz,
                                    out, ocol0);
  } else {
    auto* fn = fused_apply_kernel<NT, KIND, DIM, false, W>;
    HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn<<<ntasks, W * 32, smem, s>>>(op, tasks, rowtab, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz,
                                    out, ocol0);
  }
}

template <int NT>
void fused_nt(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab, int ntasks,
              const std::int64_t* pay_off, const int* pc, const double* gc, int gld, int gcol0,
              int ncols, const double* xc, std::int64_t nnz, double* out, int ocol0, cudaStream_t s) {
#define HP_ARGS op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out, ocol0, s
  switch (op.kind) {
    case kOpDense: return fused_kind_dim<NT, kOpDense, 0>(HP_ARGS);
    case kOpLog:
      if (op.dim == 1) return fused_kind_dim<NT, kOpLog, 1>(HP_ARGS);
      if (op.dim == 2) return fused_kind_dim<NT, kOpLog, 2>(HP_ARGS);
      return fused_kind_dim<NT, kOpLog, 3>(HP_ARGS);
    case kOpInvDist4Pi:
      if (op.dim == 1) return fused_kind_dim<NT, kOpInvDist4Pi, 1>(HP_ARGS);
      if (op.dim == 2) return fused_kind_dim<NT, kOpInvDist4Pi, 2>(HP_ARGS);
      return fused_kind_dim<NT, kOpInvDist4Pi, 3>(HP_ARGS);
    default:
      if (op.dim == 1) return fused_kind_dim<NT, kOpExp, 1>(HP_ARGS);
      if (op.dim == 2) return fused_kind_dim<NT, kOpExp, 2>(HP_ARGS);
      return fused_kind_dim<NT, kOpExp, 3>(HP_ARGS);
  }
#undef HP_ARGS
}

}  // namespace

void launch_sample_apply_fused(const DevOp& op, bool trans, const K2Task* tasks,
                               const K2Row* rowtab, int ntasks, const std::int64_t* pay_off,
                               const int* pc, const double* gc, int gld, int gcol0, int ncols,
                               const double* xc, std::int64_t nnz, double* out, int ocol0,
                               cudaStream_t s) {
  if (ntasks == 0) return;
  const int nt = (ncols + 7) / 8;
#define HP_CASE(NT)                                                                              \
  case NT:                                                                                       \
    fused_nt<NT>(op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz,  \
                 out, ocol0, s);                                                                 \
    break;
  switch (nt) {
    HP_CASE(1) HP_CASE(2) HP_CASE(3) HP_CASE(4) HP_CASE(5) HP_CASE(6) HP_CASE(7) HP_CASE(8)
    HP_CASE(9) HP_CASE(10) HP_CASE(11)
    default:
      throw std::invalid_argument("fused apply kernel supports sample width 2r <= 88");
  }
#undef HP_CASE
  HP_LAUNCHED();
}

}  // namespace hpeel
