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

#include <cstdlib>

#include "k2_ws.cuh"
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

// profiling switch (hp_debug_set_k2_mode): bit 0 skips kernel evaluation,
// bit 1 skips the DMMA, bit 2 selects the fused kernel (k_apply3.cu); 0 in production
int& k2_mode_ref() {
  static int mode = 0;
  return mode;
}

// Leaf identity probes: one thread per (row, column t); sums kernel columns.
template <int KIND, int DIM>
__global__ void identity_apply_kernel(DevOp op, const SampleTask* __restrict__ tasks,
                                      const std::int64_t* __restrict__ pay_off,
                                      const int* __restrict__ pay_box,
                                      const std::int64_t* __restrict__ box_start,
                                      const std::int64_t* __restrict__ box_count, int w,
                                      double* __restrict__ out) {
  // the color's payload boxes (start, count) staged in shared memory in
  // chunks, and the half_log table for log kernels: the per-box loop then has
  // no dependent global loads before the coordinate reads
  constexpr int kBoxChunk = 512;
  __shared__ std::int64_t s_start[kBoxChunk];
  __shared__ int s_count[kBoxChunk];
  __shared__ __align__(16) double s_tab[KIND == kOpLog ? 2 * kLogTab : 2];
  const SampleTask task = tasks[blockIdx.x];
  const std::int64_t n = op.n;
  if constexpr (KIND == kOpLog) {
    for (int e = threadIdx.x; e < 2 * kLogTab; e += blockDim.x) s_tab[e] = op.ltab[e];
  }
  const double* tab = KIND == kOpLog ? s_tab : op.ltab;
  const std::int64_t q0 = pay_off[task.color], q1 = pay_off[task.color + 1];
  // compact dense blocks: only the |I_mu| columns the block keeps (task.pad)
  const int nidx = task.rows * (task.pad > 0 && task.pad < w ? task.pad : w);
  // per-thread accumulators for kPer (row, column) entries per pass
  constexpr int kPer = 16;
  for (int base = 0; base < nidx; base += kPer * int(blockDim.x)) {
    double acc[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) acc[u] = 0.0;
    for (std::int64_t qc = q0; qc < q1; qc += kBoxChunk) {
      const int nb = int(q1 - qc < kBoxChunk ? q1 - qc : kBoxChunk);
      __syncthreads();
      for (int e = threadIdx.x; e < nb; e += blockDim.x) {
        const int v = pay_box[qc + e];
        s_start[e] = box_start[v];
        s_count[e] = int(box_count[v]);
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int idx = base + threadIdx.x + u * int(blockDim.x);
        if (idx >= nidx) break;
        const int t = idx / task.rows, i = idx - t * task.rows;
        const std::int64_t ip = task.row0 + i;
        double xi[DIM > 0 ? DIM : 1];
        if constexpr (KIND != kOpDense) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) xi[d] = op.x[d * n + ip];
        }
        double a = acc[u];
        for (int b = 0; b < nb; ++b) {
          if (t >= s_count[b]) continue;
          const std::int64_t jp = s_start[b] + t;
          if constexpr (KIND == kOpDense) {
            a += op.a[ip + jp * n];
          } else {
            double xj[DIM > 0 ? DIM : 1];
#pragma unroll
            for (int d = 0; d < DIM; ++d) xj[d] = op.x[d * n + jp];
            a += kernel_value<KIND, DIM>(xi, xj, ip == jp, op.param, tab);
          }
        }
        acc[u] = a;
      }
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int idx = base + threadIdx.x + u * int(blockDim.x);
      if (idx >= nidx) break;
      const int t = idx / task.rows, i = idx - t * task.rows;
      out[task.out + i + std::int64_t(t) * task.ld] = acc[u];
    }
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
            kv = kernel_value<KIND, DIM>(xi, xj, i == j0 + t, op.param, op.ltab);
          }
          acc = fma(kv, vs[t], acc);
        }
      }
    }
    if (i < n) y[i + std::int64_t(c) * n] = acc;
  }
}

}  // namespace

int k2_mode() { return k2_mode_ref(); }

// K2 arithmetic path: int8 tensor-core digit products (k2_i8.cuh) where
// eligible, unless switched off (hp_debug_set_k2_path(1) or HP_K2_FP64=1).
static int& k2_path_ref() {
  static int path = std::getenv("HP_K2_FP64") ? 1 : 0;
  return path;
}
bool k2_int8_enabled() { return k2_path_ref() != 1; }
int k2_int8_debug() { return k2_path_ref() >= 2 ? k2_path_ref() - 1 : 0; }  // 2: no MMA, 3: no eval, 5: MMAs x2, 7: no eval + MMAs x2
void set_k2_path(int path) { k2_path_ref() = path; }

int k2_tile_rows(int ncols) {
  const int nt = (ncols + 7) / 8;
  return ((k2_mode() & 4) && nt <= 11) ? kFusedRows : k2::k2_rows_for(nt);
}

void set_k2_mode(int m) { k2_mode_ref() = m; }

void launch_payload_gaussian(double* g, int gld, int r, std::int64_t n, const int* pos_box,
                             const int* local, std::uint64_t seed, int level, cudaStream_t s) {
  const std::int64_t total = n * gld;
  const unsigned blocks = unsigned(std::min<std::int64_t>((total + 255) / 256, 148 * 32));
  payload_gaussian_kernel<<<blocks, 256, 0, s>>>(g, gld, r, n, pos_box, local, seed, level);
  HP_LAUNCHED();
}

void launch_sample_apply(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab, int ntasks,
                         const std::int64_t* pay_off, const int* pc, const double* gc, int gld,
                         int gcol0, int ncols, const double* xc, std::int64_t nnz, double* out,
                         int ocol0, bool checked, cudaStream_t s) {
  if (ntasks == 0) return;
  const int flags = checked ? 8 : 0;
  const int nt = (ncols + 7) / 8;
  if ((k2_mode() & 4) && nt <= 11) {
    launch_sample_apply_fused(op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld, gcol0, ncols,
                              xc, nnz, out, ocol0, s);
    return;
  }
#define HP_ARGS op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out, ocol0, flags, s
  if (nt > 20) throw std::invalid_argument("sample width 2r > 160 is not supported by the apply kernel");
  switch (op.kind) {
    case kOpDense: k2::launch_dense(HP_ARGS); break;
    case kOpLog: k2::launch_log(HP_ARGS); break;
    case kOpInvDist4Pi: k2::launch_invdist(HP_ARGS); break;
    default: k2::launch_exp(HP_ARGS); break;
  }
#undef HP_ARGS
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
