// K4 batched range finder, register-resident variant (sm_100a).
//
// Same contract as k_qr.cu (qr_top / qr_chunk / qr_backprop), for blocks of
// at most 4 * RPT rows and NC >= cols columns: every column lives in the
// registers of the four threads of one "column group" (rows g*RPT .. +RPT in
// thread g), so a Householder step is
//   - one broadcast of the reflector through shared memory,
//   - per column a local dot product + a 2-step shuffle reduction over the
//     four row groups, and a local axpy,
// with no shared-memory traffic for the block itself and two barriers per
// step. Column pivoting (largest remaining norm, first index on ties) keeps
// columns in place and tracks the order in shared memory; remaining norms
// are downdated with LAPACK dlaqp2's cancellation guard and recomputed
// exactly when it trips (the ColPivHouseholderQR norm-update rule of the
// reference, proj/src/linalg.cpp:53-78 via Eigen). The dynamic row index of
// the pivot row is resolved with a warp-uniform switch, never through local
// memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "kernels.hpp"

namespace hpeel {

namespace {

// x[i] for a warp-uniform runtime i < RPT: a jump table, not local memory
#define HP_R4(M, b) M(b) M(b + 1) M(b + 2) M(b + 3)
#define HP_R16(M, b) HP_R4(M, b) HP_R4(M, b + 4) HP_R4(M, b + 8) HP_R4(M, b + 12)
#define HP_R64(M) HP_R16(M, 0) HP_R16(M, 16) HP_R16(M, 32) HP_R16(M, 48)
template <int RPT>
__device__ __forceinline__ double get_row(const double (&x)[RPT], int i) {
  double v = 0.0;
#define HP_GET(K)                      \
  case K:                              \
    if constexpr ((K) < RPT) v = x[K]; \
    break;
  switch (i) { HP_R64(HP_GET) default: break; }
#undef HP_GET
  return v;
}
template <int RPT>
__device__ __forceinline__ void set_row(double (&x)[RPT], int i, double v) {
#define HP_SET(K)                      \
  case K:                              \
    if constexpr ((K) < RPT) x[K] = v; \
    break;
  switch (i) { HP_R64(HP_SET) default: break; }
#undef HP_SET
}

// sum over the TPC threads of one column (lanes CPW apart, CPW = 32 / TPC)
template <int TPC>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = 32 / TPC; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum of x[i]^2 over this thread's rows r0 + i > j
template <int RPT>
__device__ __forceinline__ double tail_sq(const double (&x)[RPT], int r0, int j) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < RPT; ++i)
    if (r0 + i > j) s = fma(x[i], x[i], s);
  return s;
}

template <int NC, int RPT, int TPC>
struct QrShared {
  double v[2][TPC][RPT + 2];  // reflector (double-buffered), per row group (padded)
  double tau[NC];
  double beta[NC];
  double best[2][NC * TPC / 32];   // per-warp argmax of the next step (double-buffered)
  int bidx[2][NC * TPC / 32];
  int perm[NC];
  int keep;
};

// Broadcast reflector j from column owner threads into sm.v: rows < j -> 0,
// row j -> 1, rows > j -> x.
template <int RPT>
__device__ __forceinline__ void publish_v(double (*vs)[RPT + 2], const double (&x)[RPT], int g,
                                          int r0, int j) {
#pragma unroll
  for (int i = 0; i < RPT; ++i) vs[g][i] = r0 + i > j ? x[i] : (r0 + i == j ? 1.0 : 0.0);
}

__device__ __forceinline__ double2 lds2(const double* p) {
  double2 r;
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return r;
}

// x -= tau * v * (v^T x) over the column (all four row groups reduce). The
// reflector is read in 8-row slices through volatile loads fenced on the
// running sums, so at most one slice is live in registers next to the column.
template <int TPC, int RPT>
__device__ __forceinline__ double reflect(double (&x)[RPT], const double* v, double tau) {
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int i0 = 0; i0 < RPT; i0 += 8) {
#pragma unroll
    for (int i = i0; i < i0 + 8 && i < RPT; i += 2) {
      const double2 vv = lds2(v + i);
      s0 = fma(vv.x, x[i], s0);
      s1 = fma(vv.y, x[i + 1], s1);
    }
    asm volatile("" : "+d"(s0), "+d"(s1));
  }
  const double w = group_sum<TPC>(s0 + s1) * tau;
#pragma unroll
  for (int i0 = 0; i0 < RPT; i0 += 8) {
#pragma unroll
    for (int i = i0; i < i0 + 8 && i < RPT; i += 2) {
      const double2 vv = lds2(v + i);
      x[i] = fma(-w, vv.x, x[i]);
      x[i + 1] = fma(-w, vv.y, x[i + 1]);
    }
    asm volatile("" : "+d"(x[i0]));
  }
  return w;
}

// MODE 0: pivoted top (keep rule, Q(:, :keep) in place, Q to out).
// MODE 1: unpivoted TSQR chunk (reflectors back in place, tau, R stacked).
// Each step j: the pivot column's threads build the reflector from the tail
// norm and pivot-row value they computed in step j - 1 and publish it; one
// barrier; every column applies it, then computes its exact remaining norm
// (rows >= j + 1) and the warp-local argmax for step j + 1; a second barrier
// in MODE 0 only.
// CTAs per SM the register budget allows (x[RPT] doubles + ~48 registers)
__host__ __device__ constexpr int qr_min_blocks(int threads, int rpt) {
  return threads * (rpt * 2 + 48) <= 32768 ? 2 : 1;
}

template <int NC, int RPT, int MODE, int TPC>
__global__ void __launch_bounds__(NC * TPC, qr_min_blocks(NC * TPC, RPT))
qr_reg_kernel(const QrBlock* __restrict__ blocks, double* data, double* out, double* tau_out,
              int* ranks, int n, int kmax, double tol) {
  constexpr int CPW = 32 / TPC;  // columns per warp
  __shared__ __align__(16) QrShared<NC, RPT, TPC> sm;
  const QrBlock b = blocks[blockIdx.x];
  const int m = b.rows;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane / CPW;
  const int c = warp * CPW + (lane % CPW);
  const int r0 = g * RPT;
  const bool valid = c < n;

  double x[RPT];
  {
    const double* src = data + b.a + r0 + std::int64_t(valid ? c : 0) * b.lda;
    const int lim = valid ? m - r0 : 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) x[i] = i < lim ? src[i] : 0.0;
  }

  const int kk = m < n ? m : n;
  const int steps = MODE == 0 ? (kk < kmax ? kk : kmax) : kk;
  bool done = !valid;
  int li = -1;  // logical (pivot) position of this column

  // column statistics for step j: sig = sum of squares of rows > j, arow =
  // row j; MODE 0 also publishes the warp argmax of sig + arow^2
  double sig = 0.0, arow = 0.0;
  auto stats = [&](int j, int buf) {
    // MODE 1 (no pivoting): only column j's warp needs its tail norm
    if (MODE == 1 && j / CPW != warp) return;
    const int gj = j / RPT, ij = j - gj * RPT;
    sig = group_sum<TPC>(tail_sq(x, r0, j));
    arow = __shfl_sync(0xffffffffu, get_row(x, ij), (lane % CPW) + gj * CPW);
    if (MODE == 0) {
      double key = done ? -1.0 : fma(arow, arow, sig);
      int kidx = c;
#pragma unroll
      for (int o = 1; o < CPW; o <<= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, key, o);
        const int oi = __shfl_xor_sync(0xffffffffu, kidx, o);
        if (ok > key || (ok == key && oi < kidx)) {
          key = ok;
          kidx = oi;
        }
      }
      if (lane == 0) {
        sm.best[buf][warp] = key;
        sm.bidx[buf][warp] = kidx;
      }
    }
  };
  if (steps > 0) stats(0, 0);
  __syncthreads();

  for (int j = 0; j < steps; ++j) {
    const int gj = j / RPT, ij = j - gj * RPT;
    int p = j;
    if (MODE == 0) {
      // first maximum of the remaining norms
      double bk = sm.best[j & 1][0];
      p = sm.bidx[j & 1][0];
#pragma unroll
      for (int w = 1; w < NC / CPW; ++w)
        if (sm.best[j & 1][w] > bk) {
          bk = sm.best[j & 1][w];
          p = sm.bidx[j & 1][w];
        }
    }
    double (*vj)[RPT + 2] = sm.v[j & 1];
    if (c == p) {
      // dlarfg from this column's tail norm and pivot-row value
      const double alpha = arow;
      double tau = 0.0, beta = alpha;
      if (sig > 0.0) {
        beta = alpha >= 0.0 ? -sqrt(alpha * alpha + sig) : sqrt(alpha * alpha + sig);
        tau = (beta - alpha) / beta;
        const double scale = 1.0 / (alpha - beta);
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          if (r0 + i > j) x[i] *= scale;
      }
      if (g == gj) set_row(x, ij, beta);
      publish_v(vj, x, g, r0, j);
      if (g == 0) {
        sm.tau[j] = tau;
        sm.beta[j] = beta;
        sm.perm[j] = p;
      }
      done = true;
      li = j;
    }
    __syncthreads();
    const double tau = sm.tau[j];
    if (tau != 0.0) reflect<TPC>(x, vj[g], done ? 0.0 : tau);
    if (j + 1 < steps) stats(j + 1, (j + 1) & 1);
    // MODE 0: every thread reads the next pivot from the warps' argmax.
    // MODE 1 needs no second barrier: the next reflector goes to the other
    // buffer (its previous readers all passed this step's barrier), and the
    // next pivot column's tail norm is reduced inside its own warp.
    if (MODE == 0) __syncthreads();
  }

  if (MODE == 1) {
    // reflectors and R back in place, tau, R rows into the stacked parent
    if (valid) {
      double* dst = data + b.a + r0 + std::int64_t(c) * b.lda;
      double* rdst = out + b.out + r0 + std::int64_t(c) * b.ldo;
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (i < m - r0) dst[i] = x[i];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (i < kk - r0) rdst[i] = r0 + i <= c ? x[i] : 0.0;
    }
    for (int jj = t; jj < kk; jj += NC * TPC) tau_out[b.tau + jj] = sm.tau[jj];
    return;
  }

  // keep rule on the R diagonal
  if (t == 0) {
    int keep = 0;
    if (steps > 0) {
      const double r00 = fabs(sm.beta[0]);
      while (keep < steps && fabs(sm.beta[keep]) > tol * r00) ++keep;
    }
    sm.keep = keep;
    if (b.rank_slot >= 0) ranks[b.rank_slot] = keep;
  }
  __syncthreads();
  const int keep = sm.keep;
  // Q(:, :keep) in place, dorg2r order; double-buffered reflector, one
  // barrier per column
  for (int j = keep - 1; j >= 0; --j) {
    double (*vj)[RPT + 2] = sm.v[j & 1];
    const bool owner = li == j;
    if (owner) publish_v(vj, x, g, r0, j);
    __syncthreads();
    const double tau = sm.tau[j];
    if (tau != 0.0) reflect<TPC>(x, vj[g], li > j && li < keep ? tau : 0.0);
    if (owner) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = r0 + i;
        x[i] = r < j ? 0.0 : (r == j ? 1.0 - tau : -tau * x[i]);
      }
    }
  }
  // Q columns to out (zero beyond keep)
  for (int e = t; e < m * kmax; e += NC * TPC) {
    const int col = e / m;
    if (col >= keep) out[b.out + (e - col * m) + std::int64_t(col) * b.ldo] = 0.0;
  }
  if (li >= 0 && li < keep) {
    double* dst = out + b.out + r0 + std::int64_t(li) * b.ldo;
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i < m - r0) dst[i] = x[i];
  }
}

// out(rows x kmax) = H_0..H_{kk-1} [C; 0]: X columns on threads, reflectors
// streamed from the chunk's in-place storage.
template <int NC, int RPT, int TPC>
__global__ void __launch_bounds__(NC * TPC, qr_min_blocks(NC * TPC, RPT))
qr_reg_backprop_kernel(const QrBlock* __restrict__ blocks, const double* data,
                       const double* __restrict__ tau, const double* parent, double* outbuf, int n,
                       int kmax) {
  constexpr int CPW = 32 / TPC;
  __shared__ __align__(16) double vs[2][TPC][RPT + 2];
  const QrBlock b = blocks[blockIdx.x];
  const int m = b.rows;
  const int kk = m < n ? m : n;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane / CPW;
  const int c = warp * CPW + (lane % CPW);
  const int r0 = g * RPT;
  const bool valid = c < kmax;
  double x[RPT];
  {
    const double* src = parent + b.c + r0 + std::int64_t(valid ? c : 0) * b.ldc;
    const int lim = valid ? kk - r0 : 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) x[i] = i < lim ? src[i] : 0.0;
  }
  auto stage = [&](int j, int buf) {
    for (int r = t; r < TPC * RPT; r += NC * TPC) {
      const int gg = r / RPT, ii = r - gg * RPT;
      vs[buf][gg][ii] = r > j && r < m ? data[b.a + r + std::int64_t(j) * b.lda] : (r == j ? 1.0 : 0.0);
    }
  };
  if (kk > 0) stage(kk - 1, (kk - 1) & 1);
  __syncthreads();
  for (int j = kk - 1; j >= 0; --j) {
    if (j > 0) stage(j - 1, (j - 1) & 1);
    const double tj = tau[b.tau + j];
    if (tj != 0.0) reflect<TPC>(x, vs[j & 1][g], valid ? tj : 0.0);
    __syncthreads();
  }
  if (valid) {
    double* dst = outbuf + b.out + r0 + std::int64_t(c) * b.ldo;
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i < m - r0) dst[i] = x[i];
  }
}

}  // namespace

int qr_reg_cols(int cols) { return cols <= 32 ? 32 : cols <= 48 ? 48 : cols <= 64 ? 64 : cols <= 80 ? 80 : cols <= 96 ? 96 : 0; }

// Layout per block-size class, code = threads per column * 100 + rows per
// thread (a block's arithmetic depends only on its class, so batches are
// launched per class and sharded runs reproduce the unsharded factors):
//  - up to 64 columns: 8 threads per column for <= 128 rows (8 or 16 rows
//    each), 16 threads per column for 129..256 rows (16 rows each: half the
//    dependent chain of a Householder step; for <= 128 rows the wider layout
//    measured 1.6-2.3x slower, its threads mostly idle);
//  - 80 columns (config 5): 8 threads per column, <= 24 rows each (640
//    threads, 96 registers; the 4-thread layout held 168 registers, one
//    320-thread CTA per SM and half of its stall samples at the step
//    barriers, profiles/r02_ncu_kernels.txt);
//  - 96 columns: 4 threads per column, <= 48 rows each.
namespace {
int variant_for(int nc, int max_rows) {
  if (nc <= 64) {
    const int need = (max_rows + 7) / 8;
    return need <= 8 ? 808 : need <= 16 ? 816 : 1616;
  }
  if (nc <= 80) {
    const int need = (max_rows + 7) / 8;
    return need <= 8 ? 808 : need <= 16 ? 816 : 824;
  }
  const int need = (max_rows + 3) / 4;
  return need <= 16 ? 416 : need <= 32 ? 432 : 448;
}
constexpr int vt(int v) { return v / 100; }
constexpr int vr(int v) { return v % 100; }
}  // namespace

int qr_reg_rows_max(int cols) {
  const int nc = qr_reg_cols(cols);
  if (nc == 0) return 0;
  return nc <= 64 ? 256 : 192;
}

namespace {

template <int NC, int V>
void launch_reg(int mode, const QrBlock* blocks, int nb, double* data, double* out, double* tau, int* ranks,
                int cols, int kmax, double tol, cudaStream_t s) {
  constexpr int T = vt(V), R = vr(V);
  if (mode == 0)
    qr_reg_kernel<NC, R, 0, T><<<nb, NC * T, 0, s>>>(blocks, data, out, tau, ranks, cols, kmax, tol);
  else
    qr_reg_kernel<NC, R, 1, T><<<nb, NC * T, 0, s>>>(blocks, data, out, tau, ranks, cols, kmax, tol);
}

template <int NC>
void launch_reg_nc(int mode, int v, const QrBlock* blocks, int nb, double* data, double* out, double* tau,
                   int* ranks, int cols, int kmax, double tol, cudaStream_t s) {
#define HP_V(V)                                                                  \
  case V:                                                                        \
    return launch_reg<NC, V>(mode, blocks, nb, data, out, tau, ranks, cols, kmax, tol, s);
  if constexpr (NC <= 64) {
    switch (v) { HP_V(808) HP_V(816) HP_V(1616) default: break; }
  } else if constexpr (NC <= 80) {
    switch (v) { HP_V(808) HP_V(816) HP_V(824) default: break; }
  } else {
    switch (v) { HP_V(416) HP_V(432) HP_V(448) default: break; }
  }
#undef HP_V
  throw std::logic_error("qr_reg: no kernel for this block class");
}

template <int NC, int V>
void launch_bp(const QrBlock* blocks, int nb, const double* data, const double* tau, const double* parent,
               double* outbuf, int cols, int kmax, cudaStream_t s) {
  constexpr int T = vt(V), R = vr(V);
  qr_reg_backprop_kernel<NC, R, T><<<nb, NC * T, 0, s>>>(blocks, data, tau, parent, outbuf, cols, kmax);
}

template <int NC>
void launch_bp_nc(int v, const QrBlock* blocks, int nb, const double* data, const double* tau,
                  const double* parent, double* outbuf, int cols, int kmax, cudaStream_t s) {
#define HP_V(V)    \
  case V:          \
    return launch_bp<NC, V>(blocks, nb, data, tau, parent, outbuf, cols, kmax, s);
  if constexpr (NC <= 64) {
    switch (v) { HP_V(808) HP_V(816) HP_V(1616) default: break; }
  } else if constexpr (NC <= 80) {
    switch (v) { HP_V(808) HP_V(816) HP_V(824) default: break; }
  } else {
    switch (v) { HP_V(416) HP_V(432) HP_V(448) default: break; }
  }
#undef HP_V
  throw std::logic_error("qr_reg backprop: no kernel for this block class");
}
}  // namespace

int qr_reg_rpt(int cols, int rows) { return variant_for(qr_reg_cols(cols), rows); }

void launch_qr_reg(int mode, const QrBlock* blocks, int nb, double* data, double* out, double* tau,
                   int* ranks, int cols, int kmax, double tol, int max_rows, cudaStream_t s) {
  if (nb == 0) return;
  const int nc = qr_reg_cols(cols);
  const int v = variant_for(nc, max_rows);
  if (nc == 0 || max_rows > vt(v) * vr(v)) throw std::invalid_argument("qr_reg: block too large");
  switch (nc) {
    case 32: launch_reg_nc<32>(mode, v, blocks, nb, data, out, tau, ranks, cols, kmax, tol, s); break;
    case 48: launch_reg_nc<48>(mode, v, blocks, nb, data, out, tau, ranks, cols, kmax, tol, s); break;
    case 64: launch_reg_nc<64>(mode, v, blocks, nb, data, out, tau, ranks, cols, kmax, tol, s); break;
    case 80: launch_reg_nc<80>(mode, v, blocks, nb, data, out, tau, ranks, cols, kmax, tol, s); break;
    default: launch_reg_nc<96>(mode, v, blocks, nb, data, out, tau, ranks, cols, kmax, tol, s); break;
  }
  HP_LAUNCHED();
}

void launch_qr_reg_backprop(const QrBlock* blocks, int nb, const double* data, const double* tau,
                            const double* parent, double* outbuf, int cols, int kmax, int max_rows,
                            cudaStream_t s) {
  if (nb == 0) return;
  const int nc = qr_reg_cols(kmax);
  const int v = variant_for(nc, max_rows);
  if (nc == 0 || max_rows > vt(v) * vr(v)) throw std::invalid_argument("qr_reg backprop: block too large");
  switch (nc) {
    case 32: launch_bp_nc<32>(v, blocks, nb, data, tau, parent, outbuf, cols, kmax, s); break;
    case 48: launch_bp_nc<48>(v, blocks, nb, data, tau, parent, outbuf, cols, kmax, s); break;
    case 64: launch_bp_nc<64>(v, blocks, nb, data, tau, parent, outbuf, cols, kmax, s); break;
    case 80: launch_bp_nc<80>(v, blocks, nb, data, tau, parent, outbuf, cols, kmax, s); break;
    default: launch_bp_nc<96>(v, blocks, nb, data, tau, parent, outbuf, cols, kmax, s); break;
  }
  HP_LAUNCHED();
}

}  // namespace hpeel
