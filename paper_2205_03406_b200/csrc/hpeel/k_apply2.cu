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

constexpr int kBK = 32;        // payload rows per stage
constexpr int kBarFull = 1;    // named barriers: 1,2 tile b full; 3,4 tile b empty; 5 eval warps
constexpr int kBarEmpty = 3;
constexpr int kBarEval = 5;

__host__ __device__ constexpr int smem_stride(int nt) {
  // payload row stride (doubles) == 4 or 12 mod 16: the B-fragment pattern
  // (lane%4) * S + lane/4 then hits 16 distinct 8-byte bank pairs per half warp
  return nt * 8 + 4;
}

constexpr int kStages = 3;     // payload ring: chunk c+1 streams in while chunk c is evaluated

template <int NT, int ROWS>
constexpr size_t sample_smem_bytes() {
  return size_t(kStages * kBK * smem_stride(NT) + 2 * kBK * (ROWS + 4)) * sizeof(double);
}

/// Rows per K2 CTA: 128 (8 DMMA + 8 evaluation warps, one CTA per SM) when the
/// accumulators fit 128 registers (2r <= 88), else 64 (4 + 4 warps).
constexpr int k2_rows_for(int nt) { return nt <= 11 ? 128 : 64; }

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Warp-specialized colored apply. The payload rows of each color are stored
// contiguously in color order (gc, xc, pc: payload values, coordinates and
// tree positions), so a 32-row chunk is one contiguous copy.
// Upper half of the warps ("eval"): per chunk, cp.async the chunk's coordinates/positions
// (group 1) and payload rows (group 2), then evaluate the 64 x 32 kernel
// tile into K[b] (column-major; each thread owns one row and 16 columns).
// Lower half ("DMMA"): each owns 16 output rows and runs 2 x NT DMMA.8x8x4
// per k-step from K[b] / G[b]. Double-buffered; full/empty hand-off through
// named barriers, so evaluation of chunk c+1 overlaps the DMMA of chunk c.
template <int NT, int KIND, int DIM, bool TRANS, int ROWS>
__global__ void __launch_bounds__(ROWS * 4, 1)
sample_apply_kernel(DevOp op, const K2Task* __restrict__ tasks, const K2Row* __restrict__ rowtab,
                    const std::int64_t* __restrict__ pay_off, const int* __restrict__ pc,
                    const double* __restrict__ gc, int gld, int gcol0, int ncols,
                    const double* __restrict__ xc, std::int64_t nnz, double* __restrict__ out,
                    int ocol0, int mode) {
  constexpr int S = smem_stride(NT);
  constexpr int D = DIM > 0 ? DIM : 1;
  constexpr int kThreads = ROWS * 4;   // ROWS/16 DMMA warps + ROWS/16 evaluation warps
  constexpr int kEval = ROWS * 2;      // evaluation threads
  constexpr int kKR = ROWS + 4;        // kernel tile column stride (== 4 mod 16)
  constexpr int kBM = ROWS;
  extern __shared__ __align__(16) double dyn_smem[];
  double* gsm = dyn_smem;                        // [kStages][kBK * S] payload ring
  double* ksm = dyn_smem + kStages * kBK * S;    // [2][kBK * kKR] kernel tiles
  __shared__ __align__(16) double xs[kStages][D][kBK];
  __shared__ __align__(16) int js[kStages][kBK];
  __shared__ __align__(16) double lts[KIND == kOpLog ? 2 * kLogTab : 1];

  const K2Task task = tasks[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::int64_t n = op.n;
  const K2Row* rt = rowtab + task.rbeg;

  if constexpr (KIND == kOpLog) {
    for (int e = tid; e < 2 * kLogTab; e += kThreads) lts[e] = op.ltab[e];
  }
  for (int e = tid; e < kStages * kBK * S; e += kThreads) gsm[e] = 0.0;
  for (int e = tid; e < kStages * kBK; e += kThreads) {
    (&js[0][0])[e] = rt[0].pos;
    for (int d = 0; d < D; ++d) xs[e / kBK][d][e % kBK] = 0.0;
  }
  __syncthreads();

  const std::int64_t p0 = pay_off[task.color], p1 = pay_off[task.color + 1];
  const int nchunks = int((p1 - p0 + kBK - 1) / kBK);

  if (warp >= ROWS / 16) {
    // ------------------------------------------------ evaluation warps
    const int et = tid - kEval;
    const int row = et & (kBM - 1), cgrp = et / kBM;
    const int ipos = rt[row < task.rows ? row : task.rows - 1].pos;
    double xi[D];
    if constexpr (KIND != kOpDense) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) xi[d] = op.x[d * n + ipos];
    }
    const bool even_cols = ((gld | gcol0 | ncols) & 1) == 0;
    // stage chunk c: positions/coordinates, then payload rows (one group)
    auto load_chunk = [&](int c) {
      const int st = c % kStages;
      const std::int64_t base = p0 + std::int64_t(c) * kBK;
      const int cnt = int(p1 - base < kBK ? p1 - base : kBK);
      if (et < cnt) {
        cp_async4(&js[st][et], pc + base + et);
        if constexpr (KIND != kOpDense) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) cp_async8(&xs[st][d][et], xc + d * nnz + base + et);
        }
      }
      double* gb = gsm + st * kBK * S;
      const double* gsrc = gc + base * gld + gcol0;
      if (even_cols) {
        const int half = ncols >> 1;
        for (int idx = et; idx < cnt * half; idx += kEval) {
          const int t = idx / half, cc = (idx - t * half) * 2;
          cp_async16(gb + t * S + cc, gsrc + std::int64_t(t) * gld + cc);
        }
      } else {
        for (int idx = et; idx < cnt * ncols; idx += kEval) {
          const int t = idx / ncols, cc = idx - t * ncols;
          cp_async8(gb + t * S + cc, gsrc + std::int64_t(t) * gld + cc);
        }
      }
      cp_async_commit();
    };
    if (nchunks > 0) load_chunk(0);
    for (int c = 0; c < nchunks; ++c) {
      const int b = c & 1, st = c % kStages;
      // DMMA is done with chunk c-2 (K tile b and payload stage (c+1) % 3)
      if (c >= 2) bar_sync(kBarEmpty + b, kThreads);
      if (c + 1 < nchunks) {
        load_chunk(c + 1);
        cp_async_wait_1();  // chunk c landed (this thread's copies)
      } else {
        cp_async_wait_all();
      }
      bar_sync(kBarEval, kEval);  // ... and every eval thread's copies
      const std::int64_t base = p0 + std::int64_t(c) * kBK;
      const int cnt = int(p1 - base < kBK ? p1 - base : kBK);
      double* kb = ksm + b * kBK * kKR;
      const bool skip = (mode & 1) != 0;
      // branch-free: stale/padded columns are evaluated and masked to 0.
      // Loads, evaluations and stores are grouped so the 8 independent
      // evaluation chains of a group interleave (shared-memory stores would
      // otherwise order them).
      constexpr int kGrp = 8;
      if (skip) {
        for (int u = 0; u < kBK / 2; ++u) kb[(cgrp + 2 * u) * kKR + row] = 0.0;
        bar_arrive(kBarFull + b, kThreads);
        continue;
      }
#pragma unroll
      for (int h = 0; h < kBK / 2; h += kGrp) {
        int jp[kGrp];
        double xj[kGrp][D];
        double v[kGrp];
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
          const int col = cgrp + 2 * (h + u);
          jp[u] = js[st][col];
          if constexpr (KIND != kOpDense) {
#pragma unroll
            for (int d = 0; d < DIM; ++d) xj[u][d] = xs[st][d][col];
          }
        }
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
          const int col = cgrp + 2 * (h + u);
          if constexpr (KIND == kOpDense) {
            const int jj = col < cnt ? jp[u] : ipos;
            v[u] = TRANS ? op.a[std::int64_t(jj) + std::int64_t(ipos) * n]
                         : op.a[std::int64_t(ipos) + std::int64_t(jj) * n];
          } else {
            v[u] = kernel_value<KIND, DIM>(xi, xj[u], ipos == jp[u], op.param, lts);
          }
        }
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
          const int col = cgrp + 2 * (h + u);
          kb[col * kKR + row] = col < cnt ? v[u] : 0.0;
        }
      }
      bar_arrive(kBarFull + b, kThreads);
    }
    return;
  }

  // -------------------------------------------------- DMMA warps
  double acc[2][NT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;

  for (int c = 0; c < nchunks; ++c) {
    const int b = c & 1;
    bar_sync(kBarFull + b, kThreads);
    if (mode & 2) {
      if (c + 2 < nchunks) bar_arrive(kBarEmpty + b, kThreads);
      continue;
    }
    const double* arow = ksm + b * kBK * kKR + (lane & 3) * kKR + warp * 16 + (lane >> 2);
    const double* brow = gsm + (c % kStages) * kBK * S + (lane & 3) * S + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      const double a0 = arow[kk * 4 * kKR], a1 = arow[kk * 4 * kKR + 8];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double bb = brow[kk * 4 * S + nt * 8];
        dmma8x8x4(acc[0][nt][0], acc[0][nt][1], a0, bb);
        dmma8x8x4(acc[1][nt][0], acc[1][nt][1], a1, bb);
      }
    }
    if (c + 2 < nchunks) bar_arrive(kBarEmpty + b, kThreads);
  }

#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int rr = warp * 16 + m * 8 + (lane >> 2);
    if (rr >= task.rows) continue;
    const K2Row dst = rt[rr];
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

// profiling switch (hp_debug_set_k2_mode): bit 0 skips kernel evaluation,
// bit 1 skips the DMMA; 0 in production
int& k2_mode() {
  static int mode = 0;
  return mode;
}

template <int NT, int KIND, int DIM, int R>
void launch_rows(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab, int ntasks,
                 const std::int64_t* pay_off, const int* pc, const double* gc, int gld, int gcol0,
                 int ncols, const double* xc, std::int64_t nnz, double* out, int ocol0, cudaStream_t s) {
  constexpr size_t smem = sample_smem_bytes<NT, R>();
  if (KIND == kOpDense && trans) {
    auto* fn = sample_apply_kernel<NT, KIND, DIM, KIND == kOpDense, R>;
    HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn<<<ntasks, R * 4, smem, s>>>(op, tasks, rowtab, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out, ocol0, k2_mode());
  } else {
    auto* fn = sample_apply_kernel<NT, KIND, DIM, false, R>;
    HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn<<<ntasks, R * 4, smem, s>>>(op, tasks, rowtab, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out, ocol0, k2_mode());
  }
}

template <int NT, int KIND, int DIM>
void launch_nt_kind_dim(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab, int ntasks,
                        const std::int64_t* pay_off, const int* pc, const double* gc, int gld,
                        int gcol0, int ncols, const double* xc, std::int64_t nnz, double* out,
                        int ocol0, cudaStream_t s) {
  // kernel kinds are symmetric: only the explicit dense operator has a transpose
  launch_rows<NT, KIND, DIM, k2_rows_for(NT)>(op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld,
                                              gcol0, ncols, xc, nnz, out, ocol0, s);
}

template <int NT>
void launch_nt(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab, int ntasks,
               const std::int64_t* pay_off, const int* pc, const double* gc, int gld, int gcol0,
               int ncols, const double* xc, std::int64_t nnz, double* out, int ocol0, cudaStream_t s) {
#define HP_ARGS op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out, ocol0, s
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
        acc += kernel_value<KIND, DIM>(xi, xj, ip == jp, op.param, op.ltab);
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

int k2_tile_rows(int ncols) { return k2_rows_for((ncols + 7) / 8); }

void set_k2_mode(int m) { k2_mode() = m; }

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
                         int ocol0, cudaStream_t s) {
  if (ntasks == 0) return;
  const int nt = (ncols + 7) / 8;
#define HP_CASE(NT)                                                                            \
  case NT:                                                                                     \
    launch_nt<NT>(op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out,  \
                  ocol0, s);                                                                   \
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
