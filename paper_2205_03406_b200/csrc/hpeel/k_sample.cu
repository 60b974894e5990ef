// K1 colored Gaussian payload and K2 colored black-box apply (sm_100a).
//
// K1 replaces BlockTestMatrix::realize / payload_gaussian / gaussian_matrix
// (proj/src/coloring.cpp:252-291, proj/src/rng.cpp:35-59): instead of a dense
// N x r zero-filled Omega per color, each level stores one compact row per
// tree position, because G_beta is keyed by (seed, level, box, phase) only and
// is identical in every color that carries beta.
//
// K2 replaces the per-color black-box call Y_c = A * Omega_c of
// residual_samples (proj/src/peeling.cpp:165-170) for the rows the driver
// reads back (Y_c(I_alpha, :) of the pairs served by color c): a CTA owns 64
// rows of one box and streams the payload rows of that color through shared
// memory; each lane evaluates one kernel entry per m8n8k4 step directly into
// the DMMA A fragment, so K(i, j) is computed once and reused for all 2r
// forward+adjoint columns.
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "rng.hpp"

namespace hpeel {

namespace {

__global__ void payload_gaussian_kernel(double* g, int gld, int r, std::int64_t n,
                                        const int* __restrict__ pos_box,
                                        const int* __restrict__ local, std::uint64_t seed,
                                        int level) {
  const std::int64_t total = n * gld;
  for (std::int64_t idx = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t pos = idx / gld;
    const int col = int(idx - pos * gld);
    const int box = pos_box[pos];
    if (box < 0) continue;
    double v = 0.0;
    if (col < 2 * r) {
      const int phase = col < r ? 0 : 1;
      const int c = col < r ? col : col - r;
      const std::uint64_t s = payload_seed(seed, level, box, phase);
      v = gaussian_entry(s, std::uint64_t(local[pos]) * std::uint64_t(r) + std::uint64_t(c));
    }
    g[idx] = v;
  }
}

constexpr int kBM = 64;       // rows per CTA (4 warps x 16)
constexpr int kBK = 32;       // payload rows per shared-memory stage
constexpr int kThreads = 128;
constexpr int kKS = kBK + 4;  // kernel-tile row stride (== 4 mod 16: conflict-free A fragments)

__host__ __device__ constexpr int smem_stride(int nt) {
  // payload row stride (doubles) == 4 mod 16: conflict-free B-fragment reads
  return ((nt * 8 + 11) / 16) * 16 + 4;
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Per payload chunk (32 rows): (1) all 128 threads evaluate the 64 x 32 kernel
// tile into shared memory (16 independent evaluations per thread: full ILP
// on the FP64 pipe), (2) each warp runs 2 x NT DMMA.8x8x4 per k-step over its
// 16 rows. The next chunk's payload rows stream in with cp.async meanwhile.
template <int NT>
constexpr size_t sample_smem_bytes() {
  return size_t(2 * kBK * smem_stride(NT) + kBM * kKS) * sizeof(double);
}

template <int NT, int KIND, int DIM, bool TRANS>
__global__ void __launch_bounds__(kThreads, NT <= 10 ? 4 : (NT <= 14 ? 3 : 2))
sample_apply_kernel(DevOp op, const SampleTask* __restrict__ tasks,
                    const std::int64_t* __restrict__ pay_off, const int* __restrict__ pay_pos,
                    const double* __restrict__ g, int gld, int gcol0, int ncols,
                    double* __restrict__ out, int ocol0) {
  constexpr int S = smem_stride(NT);
  constexpr int D = DIM > 0 ? DIM : 1;
  extern __shared__ __align__(16) double dyn_smem[];
  double(*gs)[kBK * S] = reinterpret_cast<double(*)[kBK * S]>(dyn_smem);
  double* ks = dyn_smem + 2 * kBK * S;
  __shared__ double xs[2][D][kBK];
  __shared__ double xr[D][kBM];
  __shared__ int js[2][kBK];

  const SampleTask task = tasks[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::int64_t n = op.n;

  for (int e = tid; e < 2 * kBK * S; e += kThreads) (&gs[0][0])[e] = 0.0;
  if (tid < kBM) {
    const int rr = tid < task.rows ? tid : task.rows - 1;
    if constexpr (KIND != kOpDense) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) xr[d][tid] = op.x[d * n + task.row0 + rr];
    }
  }
  __syncthreads();

  const std::int64_t p0 = pay_off[task.color], p1 = pay_off[task.color + 1];
  auto issue = [&](int buf, std::int64_t base) {
    const int cnt = int(p1 - base < kBK ? p1 - base : kBK);
    for (int idx = tid; idx < cnt * ncols; idx += kThreads) {
      const int t = idx / ncols, c = idx - t * ncols;
      cp_async8(&gs[buf][t * S + c], g + std::int64_t(pay_pos[base + t]) * gld + gcol0 + c);
    }
    cp_async_commit();
    if (tid < kBK) {
      const int pos = tid < cnt ? pay_pos[base + tid] : -1;
      js[buf][tid] = pos;
      if constexpr (KIND != kOpDense) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) xs[buf][d][tid] = pos >= 0 ? op.x[d * n + pos] : 0.0;
      }
    }
  };

  double acc[2][NT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;

  if (p0 < p1) issue(0, p0);
  int buf = 0;
  for (std::int64_t base = p0; base < p1; base += kBK, buf ^= 1) {
    cp_async_wait_all();
    __syncthreads();
    if (base + kBK < p1) issue(buf ^ 1, base + kBK);

    // (1) kernel tile: lane = payload column, warp strides over the 64 rows
    {
      const int jpos = js[buf][lane];
      double xj[D];
      if constexpr (KIND != kOpDense) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) xj[d] = xs[buf][d][lane];
      }
#pragma unroll
      for (int u = 0; u < kBM / 4; ++u) {
        const int row = warp + 4 * u;
        const std::int64_t ipos = task.row0 + (row < task.rows ? row : task.rows - 1);
        double v = 0.0;
        if (jpos >= 0) {
          if constexpr (KIND == kOpDense) {
            v = TRANS ? op.a[std::int64_t(jpos) + ipos * n] : op.a[ipos + std::int64_t(jpos) * n];
          } else {
            double xi[D];
#pragma unroll
            for (int d = 0; d < DIM; ++d) xi[d] = xr[d][row];
            v = kernel_value<KIND, DIM>(xi, xj, ipos == jpos, op.param);
          }
        }
        ks[row * kKS + lane] = v;
      }
    }
    __syncthreads();

    // (2) DMMA over the tile
    const double* arow0 = ks + (warp * 16 + (lane >> 2)) * kKS + (lane & 3);
    const double* arow1 = arow0 + 8 * kKS;
    const double* brow = gs[buf] + (lane & 3) * S + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      const double a0 = arow0[kk * 4], a1 = arow1[kk * 4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double b = brow[kk * 4 * S + nt * 8];
        dmma8x8x4(acc[0][nt][0], acc[0][nt][1], a0, b);
        dmma8x8x4(acc[1][nt][0], acc[1][nt][1], a1, b);
      }
    }
  }

#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int rr = warp * 16 + m * 8 + (lane >> 2);
    if (rr >= task.rows) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = nt * 8 + (lane & 3) * 2 + h;
        if (c < ncols) out[task.out + rr + std::int64_t(ocol0 + c) * task.ld] = acc[m][nt][h];
      }
    }
  }
}
template <int NT, int KIND, int DIM>
void launch_nt_kind_dim(const DevOp& op, bool trans, const SampleTask* tasks, int ntasks,
                        const std::int64_t* pay_off, const int* pay_pos, const double* g, int gld,
                        int gcol0, int ncols, double* out, int ocol0, cudaStream_t s) {
  // kernel kinds are symmetric: only the explicit dense operator has a transpose
  constexpr size_t smem = sample_smem_bytes<NT>();
  if (KIND == kOpDense && trans) {
    auto* fn = sample_apply_kernel<NT, KIND, DIM, KIND == kOpDense>;
    HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn<<<ntasks, kThreads, smem, s>>>(op, tasks, pay_off, pay_pos, g, gld, gcol0, ncols, out, ocol0);
  } else {
    auto* fn = sample_apply_kernel<NT, KIND, DIM, false>;
    HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn<<<ntasks, kThreads, smem, s>>>(op, tasks, pay_off, pay_pos, g, gld, gcol0, ncols, out, ocol0);
  }
}

template <int NT>
void launch_nt(const DevOp& op, bool trans, const SampleTask* tasks, int ntasks,
               const std::int64_t* pay_off, const int* pay_pos, const double* g, int gld, int gcol0,
               int ncols, double* out, int ocol0, cudaStream_t s) {
#define HP_ARGS op, trans, tasks, ntasks, pay_off, pay_pos, g, gld, gcol0, ncols, out, ocol0, s
  switch (op.kind) {
    case kOpDense: return launch_nt_kind_dim<NT, kOpDense, 0>(HP_ARGS);
    case kOpLog:
      if (op.dim == 1) return launch_nt_kind_dim<NT, kOpLog, 1>(HP_ARGS);
      if (op.dim == 2) return launch_nt_kind_dim<NT, kOpLog, 2>(HP_ARGS);
      return launch_nt_kind_dim<NT, kOpLog, 3>(HP_ARGS);
    case kOpInvDist4Pi:
      if (op.dim == 1) return launch_nt_kind_dim<NT, kOpInvDist4Pi, 1>(HP_ARGS);
      if (op.dim == 2) return launch_nt_kind_dim<NT, kOpInvDist4Pi, 2>(HP_ARGS);
      return launch_nt_kind_dim<NT, kOpInvDist4Pi, 3>(HP_ARGS);
    default:
      if (op.dim == 1) return launch_nt_kind_dim<NT, kOpExp, 1>(HP_ARGS);
      if (op.dim == 2) return launch_nt_kind_dim<NT, kOpExp, 2>(HP_ARGS);
      return launch_nt_kind_dim<NT, kOpExp, 3>(HP_ARGS);
  }
#undef HP_ARGS
}

// Leaf identity probes: one thread per (row, column t); sums kernel columns.
template <int KIND, int DIM>
__global__ void identity_apply_kernel(DevOp op, const SampleTask* __restrict__ tasks,
                                      const std::int64_t* __restrict__ pay_off,
                                      const int* __restrict__ pay_box,
                                      const std::int64_t* __restrict__ box_start,
                                      const std::int64_t* __restrict__ box_count, int w,
                                      double* __restrict__ out) {
  const SampleTask task = tasks[blockIdx.x];
  const std::int64_t n = op.n;
  for (int idx = threadIdx.x; idx < task.rows * w; idx += blockDim.x) {
    const int t = idx / task.rows, i = idx - t * task.rows;
    const std::int64_t ip = task.row0 + i;
    double xi[DIM > 0 ? DIM : 1];
    if constexpr (KIND != kOpDense) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) xi[d] = op.x[d * n + ip];
    }
    double acc = 0.0;
    for (std::int64_t q = pay_off[task.color]; q < pay_off[task.color + 1]; ++q) {
      const int v = pay_box[q];
      if (t >= box_count[v]) continue;
      const std::int64_t jp = box_start[v] + t;
      if constexpr (KIND == kOpDense) {
        acc += op.a[ip + jp * n];
      } else {
        double xj[DIM > 0 ? DIM : 1];
#pragma unroll
        for (int d = 0; d < DIM; ++d) xj[d] = op.x[d * n + jp];
        acc += kernel_value<KIND, DIM>(xi, xj, ip == jp, op.param);
      }
    }
    out[task.out + i + std::int64_t(t) * task.ld] = acc;
  }
}

// Full apply y = K x for the power method (proj/src/linalg.cpp:179-196).
template <int KIND, int DIM, bool TRANS>
__global__ void full_apply_kernel(DevOp op, const double* __restrict__ x, int w,
                                  double* __restrict__ y) {
  const std::int64_t n = op.n;
  const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  __shared__ double xs[DIM > 0 ? DIM : 1][256];
  __shared__ double vs[256];
  double xi[DIM > 0 ? DIM : 1];
  if constexpr (KIND != kOpDense) if (i < n) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) xi[d] = op.x[d * n + i];
  }
  for (int c = 0; c < w; ++c) {
    double acc = 0.0;
    for (std::int64_t j0 = 0; j0 < n; j0 += 256) {
      __syncthreads();
      const std::int64_t jl = j0 + threadIdx.x;
      if (jl < n) {
        vs[threadIdx.x] = x[jl + std::int64_t(c) * n];
        if constexpr (KIND != kOpDense) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) xs[d][threadIdx.x] = op.x[d * n + jl];
        }
      }
      __syncthreads();
      if (i < n) {
        const int cnt = int(n - j0 < 256 ? n - j0 : 256);
        for (int t = 0; t < cnt; ++t) {
          double kv;
          if constexpr (KIND == kOpDense) {
            kv = TRANS ? op.a[(j0 + t) + i * n] : op.a[i + (j0 + t) * n];
          } else {
            double xj[DIM > 0 ? DIM : 1];
#pragma unroll
            for (int d = 0; d < DIM; ++d) xj[d] = xs[d][t];
            kv = kernel_value<KIND, DIM>(xi, xj, i == j0 + t, op.param);
          }
          acc = fma(kv, vs[t], acc);
        }
      }
    }
    if (i < n) y[i + std::int64_t(c) * n] = acc;
  }
}

}  // namespace

void launch_payload_gaussian(double* g, int gld, int r, std::int64_t n, const int* pos_box,
                             const int* local, std::uint64_t seed, int level, cudaStream_t s) {
  const std::int64_t total = n * gld;
  const unsigned blocks = unsigned(std::min<std::int64_t>((total + 255) / 256, 148 * 32));
  payload_gaussian_kernel<<<blocks, 256, 0, s>>>(g, gld, r, n, pos_box, local, seed, level);
  HP_LAUNCHED();
}

void launch_sample_apply(const DevOp& op, bool trans, const SampleTask* tasks, int ntasks,
                         const std::int64_t* pay_off, const int* pay_pos, const double* g,
                         int gld, int gcol0, int ncols, double* out, int ocol0,
                         cudaStream_t s) {
  if (ntasks == 0) return;
  const int nt = (ncols + 7) / 8;
#define HP_CASE(NT)                                                                         \
  case NT:                                                                                  \
    launch_nt<NT>(op, trans, tasks, ntasks, pay_off, pay_pos, g, gld, gcol0, ncols, out, ocol0, \
                  s);                                                                       \
    break;
  switch (nt) {
    HP_CASE(1) HP_CASE(2) HP_CASE(3) HP_CASE(4) HP_CASE(5) HP_CASE(6) HP_CASE(7) HP_CASE(8)
    HP_CASE(9) HP_CASE(10) HP_CASE(11) HP_CASE(12) HP_CASE(13) HP_CASE(14) HP_CASE(15)
    HP_CASE(16) HP_CASE(17) HP_CASE(18) HP_CASE(19) HP_CASE(20)
    default:
      throw std::invalid_argument("sample width 2r > 160 is not supported by the apply kernel");
  }
#undef HP_CASE
  HP_LAUNCHED();
}

void launch_identity_apply(const DevOp& op, const SampleTask* tasks, int ntasks,
                           const std::int64_t* pay_off, const int* pay_box,
                           const std::int64_t* box_start, const std::int64_t* box_count, int w,
                           double* out, cudaStream_t s) {
  if (ntasks == 0) return;
#define HP_ID(K, D)                                                                          \
  identity_apply_kernel<K, D><<<ntasks, 256, 0, s>>>(op, tasks, pay_off, pay_box, box_start, \
                                                     box_count, w, out)
  if (op.kind == kOpDense) HP_ID(kOpDense, 0);
  else if (op.kind == kOpLog) { if (op.dim == 1) HP_ID(kOpLog, 1); else if (op.dim == 2) HP_ID(kOpLog, 2); else HP_ID(kOpLog, 3); }
  else if (op.kind == kOpInvDist4Pi) { if (op.dim == 1) HP_ID(kOpInvDist4Pi, 1); else if (op.dim == 2) HP_ID(kOpInvDist4Pi, 2); else HP_ID(kOpInvDist4Pi, 3); }
  else { if (op.dim == 1) HP_ID(kOpExp, 1); else if (op.dim == 2) HP_ID(kOpExp, 2); else HP_ID(kOpExp, 3); }
#undef HP_ID
  HP_LAUNCHED();
}

void launch_full_apply(const DevOp& op, bool trans, const double* x, int w, double* y,
                       cudaStream_t s) {
  const unsigned blocks = cdiv(op.n, 256);
#define HP_FA(K, D)                                                                  \
  do {                                                                               \
    if (trans) full_apply_kernel<K, D, true><<<blocks, 256, 0, s>>>(op, x, w, y);    \
    else full_apply_kernel<K, D, false><<<blocks, 256, 0, s>>>(op, x, w, y);         \
  } while (0)
  if (op.kind == kOpDense) HP_FA(kOpDense, 0);
  else if (op.kind == kOpLog) { if (op.dim == 1) HP_FA(kOpLog, 1); else if (op.dim == 2) HP_FA(kOpLog, 2); else HP_FA(kOpLog, 3); }
  else if (op.kind == kOpInvDist4Pi) { if (op.dim == 1) HP_FA(kOpInvDist4Pi, 1); else if (op.dim == 2) HP_FA(kOpInvDist4Pi, 2); else HP_FA(kOpInvDist4Pi, 3); }
  else { if (op.dim == 1) HP_FA(kOpExp, 1); else if (op.dim == 2) HP_FA(kOpExp, 2); else HP_FA(kOpExp, 3); }
#undef HP_FA
  HP_LAUNCHED();
}

}  // namespace hpeel
