// K2 warp-specialized colored apply: kernel template shared by the per-kind
// instantiation units k2_<kind>.cu (split so they compile in parallel).
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "async.cuh"
#include "kernels.hpp"

namespace hpeel {

/// K2 profiling switch (hp_debug_set_k2_mode, k_apply2.cu).
int k2_mode();

namespace k2 {

constexpr int kBK = 32;        // payload rows per stage

__host__ __device__ constexpr int smem_stride(int nt) {
  // payload row stride (doubles) == 4 or 12 mod 16: the B-fragment pattern
  // (lane%4) * S + lane/4 then hits 16 distinct 8-byte bank pairs per half warp
  return nt * 8 + 4;
}

/// Dynamic shared memory of a K2 CTA: NK kernel tiles (kBK x (ROWS + 4)), a
/// payload ring of NK + 1 stages (chunk c + 1 streams in while chunk c is
/// evaluated and the DMMA warps may still be NK - 1 chunks behind) and,
/// when `tab`, a shared-memory copy of the half_log table.
__host__ __device__ constexpr size_t sample_smem_bytes(int nt, int rows, int nk, bool tab) {
  return size_t((nk + 1) * kBK * smem_stride(nt) + nk * kBK * (rows + 4) + (tab ? 2 * kLogTab : 0)) *
         sizeof(double);
}
/// Static shared memory: coordinates/positions ring.
__host__ __device__ constexpr size_t sample_static_bytes(int nk) {
  return size_t(nk + 1) * kBK * (4 * 8 + 4);
}
__host__ __device__ constexpr bool k2_fits(int nt, int rows, int nk, bool tab) {
  return sample_smem_bytes(nt, rows, nk, tab) + sample_static_bytes(nk) + 1024 <= 232448;
}
/// Shared-memory plan: kernel tiles in flight (3 if they fit the 227 KB
/// per-CTA budget, else 2) and whether the log table is staged in shared
/// memory (log kernels; else it is read through L1). Encoded nk + 4 * tab.
__host__ __device__ constexpr int k2_plan(int nt, int rows, bool log_kind) {
  return (log_kind && k2_fits(nt, rows, 3, true))    ? 3 + 4
         : (log_kind && k2_fits(nt, rows, 2, true))  ? 2 + 4
         : k2_fits(nt, rows, 3, false)               ? 3
                                                     : 2;
}

/// Rows per K2 CTA: 128 (8 DMMA + 8 evaluation warps, one CTA per SM) when the
/// accumulators fit 128 registers (2r <= 88), else 64.
__host__ __device__ constexpr int k2_rows_for(int nt) { return nt <= 11 ? 128 : 64; }
/// 8-row tiles per DMMA warp: 2 at 128 rows, 1 at 64 rows (8 DMMA warps either
/// way, half the accumulators per thread at 64 rows).
__host__ __device__ constexpr int k2_mt_for(int rows) { return rows == 128 ? 2 : 1; }
/// Evaluation threads: 8 warps either way. At 64 rows four column groups share
/// a row (8 kernel values per thread and chunk): with 4 + 4 warps the probe
/// (tools/k2_modes.py, config 4 scaled) showed 0.48 s of the 1.71 s apply
/// exposed in the evaluation (one evaluation warp per scheduler, bound by its
/// own latency) on top of a 0.67 s streaming skeleton.
__host__ __device__ constexpr int k2_eval_for(int rows) { return 256; }
__host__ __device__ constexpr int k2_threads_for(int rows) {
  return rows / (8 * k2_mt_for(rows)) * 32 + k2_eval_for(rows);
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
__global__ void __launch_bounds__(k2_threads_for(ROWS), 1)
sample_apply_kernel(DevOp op, const K2Task* __restrict__ tasks, const K2Row* __restrict__ rowtab,
                    const std::int64_t* __restrict__ pay_off, const int* __restrict__ pc,
                    const double* __restrict__ gc, int gld, int gcol0, int ncols,
                    const double* __restrict__ xc, std::int64_t nnz, double* __restrict__ out,
                    int ocol0, int mode) {
  constexpr int S = smem_stride(NT);
  constexpr int D = DIM > 0 ? DIM : 1;
  constexpr int MT = k2_mt_for(ROWS);            // 8-row tiles per DMMA warp
  constexpr int kDmmaWarps = ROWS / (8 * MT);
  constexpr int kEval = k2_eval_for(ROWS);       // evaluation threads
  constexpr int NG = kEval / ROWS;               // column groups sharing a row (2 or 4)
  constexpr int kThreads = kDmmaWarps * 32 + kEval;
  constexpr int kKR = ROWS + 4;        // kernel tile column stride (== 4 mod 16)
  constexpr int kBM = ROWS;
  constexpr int kPlan = k2_plan(NT, ROWS, KIND == kOpLog);
  constexpr int NK = kPlan & 3;                 // kernel tiles in flight
  constexpr bool kTabSmem = (kPlan & 4) != 0;   // half_log table in shared memory
  constexpr int kStages = NK + 1;          // payload ring stages
  // named barriers: 1..NK tile b full, NK+1..2NK tile b empty, 2NK+1 eval warps
  constexpr int kBarFull = 1, kBarEmpty = 1 + NK, kBarEval = 1 + 2 * NK;
  extern __shared__ __align__(16) double dyn_smem[];
  double* gsm = dyn_smem;                        // [kStages][kBK * S] payload ring
  double* ksm = dyn_smem + kStages * kBK * S;    // [NK][kBK * kKR] kernel tiles
  double* lts = ksm + NK * kBK * kKR;            // [2 * kLogTab] (kTabSmem)
  const double* tab = kTabSmem ? lts : op.ltab;
  constexpr int DP = D == 3 ? 4 : D;  // point stride in smem (16-byte reads)
  __shared__ __align__(16) double xs[kStages][kBK][DP];
  __shared__ __align__(16) int js[kStages][kBK];

  const K2Task task = tasks[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::int64_t n = op.n;

  if constexpr (KIND == kOpLog && kTabSmem) {
    for (int e = tid; e < 2 * kLogTab; e += kThreads) lts[e] = op.ltab[e];
  }
  for (int e = tid; e < kStages * kBK * S; e += kThreads) gsm[e] = 0.0;
  for (int e = tid; e < kStages * kBK; e += kThreads) {
    (&js[0][0])[e] = k2_row(task, rowtab, 0).pos;
    for (int d = 0; d < DP; ++d) xs[e / kBK][e % kBK][d] = 0.0;
  }
  __syncthreads();

  const std::int64_t p0 = pay_off[task.color], p1 = pay_off[task.color + 1];
  const int nchunks = int((p1 - p0 + kBK - 1) / kBK);
  // probe bit 4: payload chunks in reverse order (another FP64 summation
  // order; the results stay valid)
  const bool rev = (mode & 16) != 0;
  auto chunk_base = [&](int c) { return p0 + std::int64_t(rev ? nchunks - 1 - c : c) * kBK; };

  if (warp >= kDmmaWarps) {
    // ------------------------------------------------ evaluation warps
    const int et = tid - kDmmaWarps * 32;
    const int row = et & (kBM - 1), cgrp = et / kBM;
    const int ipos = k2_row(task, rowtab, row < task.rows ? row : task.rows - 1).pos;
    double xi[D];
    if constexpr (KIND != kOpDense) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) xi[d] = op.x[d * n + ipos];
    }
    const bool even_cols = ((gld | gcol0 | ncols) & 1) == 0;
    // stage chunk c: positions/coordinates, then payload rows (one group)
    auto load_chunk = [&](int c) {
      const int st = c % kStages;
      const std::int64_t base = chunk_base(c);
      const int cnt = int(p1 - base < kBK ? p1 - base : kBK);
      if (et < cnt) {
        cp_async4(&js[st][et], pc + base + et);
        if constexpr (KIND != kOpDense) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) cp_async8(&xs[st][et][d], xc + d * nnz + base + et);
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
      if (cnt < kBK) {
        // partial (last) chunk: zero payload rows and far-away points in the
        // padding, so padded columns need no masking in the evaluation
        for (int idx = et; idx < (kBK - cnt) * ncols; idx += kEval) {
          const int t = cnt + idx / ncols, cc = idx % ncols;
          gb[t * S + cc] = 0.0;
        }
        if (et < kBK - cnt) {
          js[st][cnt + et] = -1;
#pragma unroll
          for (int d = 0; d < D; ++d) xs[st][cnt + et][d] = 1e150;
        }
      }
    };
    if (nchunks > 0) load_chunk(0);
    for (int c = 0; c < nchunks; ++c) {
      const int b = c % NK, st = c % kStages;
      // DMMA is done with chunk c-NK (K tile b and payload stage (c+1) % kStages)
      if (c >= NK) bar_sync(kBarEmpty + b, kThreads);
      if (c + 1 < nchunks) {
        load_chunk(c + 1);
        cp_async_wait_1();  // chunk c landed (this thread's copies)
      } else {
        cp_async_wait_all();
      }
      bar_sync(kBarEval, kEval);  // ... and every eval thread's copies
      const std::int64_t base = chunk_base(c);
      const int cnt = int(p1 - base < kBK ? p1 - base : kBK);
      double* kb = ksm + b * kBK * kKR;
      const bool skip = (mode & 1) != 0;
      // branch-free: padded columns evaluate far-away points against zero
      // payload rows (dense: masked). Loads, evaluations and stores are
      // grouped so the 8 independent evaluation chains of a group interleave
      // (shared-memory stores would otherwise order them). Unchecked tiles
      // (mode bit 3 clear) skip the i == j / coincident-point tests.
      constexpr int kGrp = 8;
      static_assert((kBK / NG) % kGrp == 0, "kernel values per thread and chunk in groups of kGrp");
      if (skip) {
        for (int u = 0; u < kBK / NG; ++u) kb[(cgrp + NG * u) * kKR + row] = 0.0;
        bar_arrive(kBarFull + b, kThreads);
        continue;
      }
      auto eval_tile = [&](auto check) {
        constexpr bool C = decltype(check)::value;
#pragma unroll
        for (int h = 0; h < kBK / NG; h += kGrp) {
          int jp[kGrp];
          double xj[kGrp][DP];
          double v[kGrp];
#pragma unroll
          for (int u = 0; u < kGrp; ++u) {
            const int col = cgrp + NG * (h + u);
            if (KIND == kOpDense || C) jp[u] = js[st][col];
            if constexpr (KIND != kOpDense) {
#pragma unroll
              for (int d = 0; d < DP; d += 2) {
                if (d + 1 < DP) {
                  const double2 p = *reinterpret_cast<const double2*>(&xs[st][col][d]);
                  xj[u][d] = p.x;
                  xj[u][d + 1] = p.y;
                } else {
                  xj[u][d] = xs[st][col][d];
                }
              }
            }
          }
#pragma unroll
          for (int u = 0; u < kGrp; ++u) {
            const int col = cgrp + NG * (h + u);
            if constexpr (KIND == kOpDense) {
              const int jj = col < cnt ? jp[u] : ipos;
              v[u] = TRANS ? op.a[std::int64_t(jj) + std::int64_t(ipos) * n]
                           : op.a[std::int64_t(ipos) + std::int64_t(jj) * n];
            } else {
              v[u] = kernel_value<KIND, DIM, C>(xi, xj[u], C && ipos == jp[u], op.param, tab);
            }
          }
#pragma unroll
          for (int u = 0; u < kGrp; ++u) {
            const int col = cgrp + NG * (h + u);
            kb[col * kKR + row] = (KIND != kOpDense || col < cnt) ? v[u] : 0.0;
          }
        }
      };
      if (mode & 8) {
        eval_tile(std::true_type{});
      } else {
        eval_tile(std::false_type{});
      }
      bar_arrive(kBarFull + b, kThreads);
    }
    return;
  }

  // -------------------------------------------------- DMMA warps
  double acc[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;

  for (int c = 0; c < nchunks; ++c) {
    const int b = c % NK;
    bar_sync(kBarFull + b, kThreads);
    if (mode & 2) {
      if (c + NK < nchunks) bar_arrive(kBarEmpty + b, kThreads);
      continue;
    }
    const double* arow = ksm + b * kBK * kKR + (lane & 3) * kKR + warp * 8 * MT + (lane >> 2);
    const double* brow = gsm + (c % kStages) * kBK * S + (lane & 3) * S + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      double a[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) a[m] = arow[kk * 4 * kKR + 8 * m];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double bb = brow[kk * 4 * S + nt * 8];
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma8x8x4(acc[m][nt][0], acc[m][nt][1], a[m], bb);
      }
    }
    if (c + NK < nchunks) bar_arrive(kBarEmpty + b, kThreads);
  }

#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const int rr = warp * 8 * MT + m * 8 + (lane >> 2);
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

template <int NT, int KIND, int DIM, int R>
void launch_rows(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab, int ntasks,
                 const std::int64_t* pay_off, const int* pc, const double* gc, int gld, int gcol0,
                 int ncols, const double* xc, std::int64_t nnz, double* out, int ocol0, int flags, cudaStream_t s) {
  constexpr int plan = k2_plan(NT, R, KIND == kOpLog);
  constexpr size_t smem = sample_smem_bytes(NT, R, plan & 3, (plan & 4) != 0);
  if (KIND == kOpDense && trans) {
    auto* fn = sample_apply_kernel<NT, KIND, DIM, KIND == kOpDense, R>;
    HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn<<<ntasks, k2_threads_for(R), smem, s>>>(op, tasks, rowtab, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out, ocol0, k2_mode() | flags);
  } else {
    auto* fn = sample_apply_kernel<NT, KIND, DIM, false, R>;
    HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn<<<ntasks, k2_threads_for(R), smem, s>>>(op, tasks, rowtab, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out, ocol0, k2_mode() | flags);
  }
}

template <int NT, int KIND, int DIM>
void launch_nt_kind_dim(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab, int ntasks,
                        const std::int64_t* pay_off, const int* pc, const double* gc, int gld,
                        int gcol0, int ncols, const double* xc, std::int64_t nnz, double* out,
                        int ocol0, int flags, cudaStream_t s) {
  // kernel kinds are symmetric: only the explicit dense operator has a transpose
  launch_rows<NT, KIND, DIM, k2_rows_for(NT)>(op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld,
                                              gcol0, ncols, xc, nnz, out, ocol0, flags, s);
}


/// Per-kind launch entry points (k2_<kind>.cu): dispatch on NT = ceil(ncols/8) and dim.
#define HP_K2_LAUNCH_ARGS                                                                        \
  const DevOp &op, bool trans, const K2Task *tasks, const K2Row *rowtab, int ntasks,            \
      const std::int64_t *pay_off, const int *pc, const double *gc, int gld, int gcol0,          \
      int ncols, const double *xc, std::int64_t nnz, double *out, int ocol0, int flags, cudaStream_t s
void launch_dense(HP_K2_LAUNCH_ARGS);
void launch_log(HP_K2_LAUNCH_ARGS);
void launch_invdist(HP_K2_LAUNCH_ARGS);
void launch_exp(HP_K2_LAUNCH_ARGS);

}  // namespace k2
}  // namespace hpeel
