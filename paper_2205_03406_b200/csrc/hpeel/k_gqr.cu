// K4 batched range finder on FP64 DMMA: staged pivoted Cholesky-QR (sm_100a).
//
// qr_orthonormal (proj/src/linalg.cpp:53-78) is a column-pivoted Householder
// QR of an m x r sample block Y: keep = #{j : |R_jj| > tol |R_00|} capped at
// kmax, Q(:, :keep) returned. The Householder recurrence is a chain of r
// dependent reflections over the whole block (k_qr2.cu: ~3% of the FP64
// peak). Here the same pivots and the same span come from the Gram matrix:
//
//   stage:  G = Y^T Y                          (DMMA, rows streamed once)
//           pivoted Cholesky of G              (one small CTA per block):
//             the pivot order and the diagonal L_jj = |R_jj| of QRCP on Y,
//             stopped where the Schur diagonal falls under theta = 1e-12 of
//             the stage's first pivot (G carries ~1e-15 of noise), at the
//             rank threshold or at kmax; the same eliminations applied to
//             an identity give W1 = P L^-T
//           Q1 = Y W1                          (DMMA)
//           [H; G1] = [Q_prev Q1]^T Q1         (DMMA)
//           Cholesky of G1 - H^T H (~ I)       -> W2 = [-H X; X], X = L2^-T
//           Q_new = [Q_prev Q1] W2             (DMMA; the second Cholesky-QR
//                                               pass and the re-projection)
//           if pivots are still owed: Y -= Q_new (Q_new^T Y)   (DMMA)
//   and the next stage factors the deflated Y (its columns now ~1e-6 of the
//   first stage's), so every stage sees a Gram matrix of condition <= 1e12.
//   Three stages reach the 1e-14 rank threshold (1e-28 in G).
//
// In exact arithmetic the pivots, |R_jj| and span(Q(:, :j)) equal those of
// the Householder factorization; in floating point Q is orthonormal to
// machine precision and the projection residual matches LAPACK's dgeqp3
// (tools/qr_bench.py). Blocks of any height take the same path: Gram
// products and Y W are sums / maps over row tasks of <= 256 rows, partial
// Gram matrices are added in task order by their consumer (deterministic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "async.cuh"
#include "chol.cuh"
#include "kernels.hpp"

namespace hpeel {

namespace {

// runner-up margin in units of the stage's first pivot (chol.cuh); HP_GQR_GAP overrides (probe)
static const double kGqrGapHost = std::getenv("HP_GQR_GAP") ? std::atof(std::getenv("HP_GQR_GAP")) : 3e-13;
constexpr unsigned long long kGqrNonFinite = 0x7ff8000000000000ull;  // amax of a block holding NaN / Inf
constexpr int kGqrThreads = 256;  // 8 warps: Gram / apply kernels
constexpr int kSlice = 64;        // rows per shared-memory slice
constexpr int kLds = 68;          // slice leading dimension: == 4 (mod 16) doubles, conflict-free fragments

__host__ __device__ constexpr int up(int n, int q) { return (n + q - 1) / q * q; }

// rows [row0, row0 + rows) x cols [0, nc) of a col-major global block into a
// slice (ld kLds) with cp.async (the caller commits and waits), zero-filled up
// to rows_pad x nc_pad
__device__ __forceinline__ void load_slice(double* dst, const double* src, std::int64_t ld, int rows, int nc,
                                           int rows_pad, int nc_pad) {
  // 64 consecutive threads take one column's rows (coalesced)
  const int t = threadIdx.x;
  const int rr = t & (kSlice - 1), c0 = t / kSlice;
  if (rr < rows_pad)
    for (int c = c0; c < nc_pad; c += kGqrThreads / kSlice) {
      double* d = dst + c * kLds + rr;
      if (rr < rows && c < nc)
        cp_async8(d, src + std::int64_t(c) * ld + rr);
      else
        *d = 0.0;
    }
}

// ------------------------------------------------------------------ Gram
// MODE 0: G  = Y^T Y                      (r x r)
// MODE 1: HG = Q(:, 0:kq+j)^T Q(:, kq:kq+j)   ((kq + j) x j)
// MODE 2: Wd = Q(:, kq:kq+j)^T Y          (j x r)
// One CTA per row task; partial at part + task * psz (col-major, ld = nx).
// NV / NU: 8 x 8 output tiles per warp along X (half of the tile rows) / Y
// (every fourth tile column) - sized by the launcher from r
template <int MODE, int NV, int NU>
__global__ void __launch_bounds__(kGqrThreads, (NV * NU <= 8 ? 3 : 2))
gqr_gram_kernel(const GqrBlock* __restrict__ blocks, const GqrTask* __restrict__ tasks,
                const GqrState* __restrict__ state, const double* data, const double* q, double* part, int r,
                std::int64_t psz, int nbuf, int bufsz) {
  extern __shared__ __align__(16) double sm[];
  const GqrTask tk = tasks[blockIdx.x];
  const GqrBlock b = blocks[tk.block];
  const GqrState* st = state + tk.block;
  if (st->done) return;
  const int kq = st->kq, j = st->j;
  if (MODE == 0 && st->last) return;  // finished in the previous stage
  if (MODE != 0 && j == 0) return;
  if (MODE == 2 && st->last) return;

  const double *xb, *yb;
  std::int64_t ldx, ldy;
  int nx, ny;
  if (MODE == 0) {
    xb = yb = data + b.a + tk.row0;
    ldx = ldy = b.lda;
    nx = ny = r;
  } else if (MODE == 1) {
    xb = q + b.out + tk.row0;
    yb = xb + std::int64_t(kq) * b.ldo;
    ldx = ldy = b.ldo;
    nx = kq + j;
    ny = j;
  } else {
    xb = q + b.out + tk.row0 + std::int64_t(kq) * b.ldo;
    ldx = b.ldo;
    nx = j;
    yb = data + b.a + tk.row0;
    ldy = b.lda;
    ny = r;
  }
  const int nx8 = up(nx, 8), ny8 = up(ny, 8);
  double* xs = sm;
  double* ys = MODE == 0 ? xs : (MODE == 1 ? xs + kq * kLds : xs + nx8 * kLds);
  // MODE 1: the Y columns are columns [kq, kq + j) of the X slice; the X slice
  // is padded to cover ys + ny8 columns
  const int xcols_pad = MODE == 1 ? max(nx8, kq + ny8) : nx8;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wi = warp & 1, wj = warp >> 1;  // tile-row half, tile-column residue (mod 4)
  const int ntx = nx8 / 8, nty = ny8 / 8;
  const int ti0 = wi * ((ntx + 1) / 2), ti1 = wi ? ntx : (ntx + 1) / 2;
  double acc[NU][NV][2];
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;

  // slices stream through one or two buffers (the next slice's cp.async
  // copies overlap this slice's DMMAs when two fit)
  auto issue = [&](int s0, int buf) {
    const int rows = min(kSlice, tk.rows - s0), rows4 = up(rows, 4);
    load_slice(xs + buf * bufsz, xb + s0, ldx, rows, nx, rows4, xcols_pad);
    if (MODE == 2) load_slice(ys + buf * bufsz, yb + s0, ldy, rows, ny, rows4, ny8);
    cp_async_commit();
  };
  issue(0, 0);
  for (int s0 = 0, it = 0; s0 < tk.rows; s0 += kSlice, ++it) {
    const int rows4 = up(min(kSlice, tk.rows - s0), 4);
    const bool more = s0 + kSlice < tk.rows;
    const int cur = nbuf == 2 ? (it & 1) : 0;
    if (nbuf == 2 && more) {
      issue(s0 + kSlice, cur ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    const double* xc = xs + cur * bufsz;
    const double* yc = ys + cur * bufsz;
    for (int k0 = 0; k0 < rows4; k0 += 4) {
      double af[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) af[v] = ti0 + v < ti1 ? xc[((ti0 + v) * 8 + g) * kLds + k0 + t4] : 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const int tj = wj + 4 * u;
        if (tj < nty) {
          const double bf = yc[(tj * 8 + g) * kLds + k0 + t4];
#pragma unroll
          for (int v = 0; v < NV; ++v)
            if (ti0 + v < ti1) dmma8x8x4(acc[u][v][0], acc[u][v][1], af[v], bf);
        }
      }
    }
    if (more) {
      __syncthreads();
      if (nbuf == 1) issue(s0 + kSlice, 0);
    }
  }
  double* out = part + std::int64_t(blockIdx.x) * psz;
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    const int tj = wj + 4 * u;
    if (tj >= nty) continue;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (ti0 + v >= ti1) continue;
      const int c = (ti0 + v) * 8 + g, d = tj * 8 + 2 * t4;
      if (c < nx) {
        if (d < ny) out[std::int64_t(d) * nx + c] = acc[u][v][0];
        if (d + 1 < ny) out[std::int64_t(d + 1) * nx + c] = acc[u][v][1];
      }
    }
  }
}

// ------------------------------------------------------------------ apply
// MODE 0: Q(:, kq:kq+j)  = Y W1                 W1: r x j       (ld r)
// MODE 1: Q(:, kq:kq+j)  = Q(:, 0:kq+j) W2      W2: (kq+j) x j  (ld kq+j), in place
// MODE 2: Y             -= Q(:, kq:kq+j) Wd     Wd: j x r = the block's summed MODE-2 Gram matrix
// NT: 8-column output tiles per warp (every second tile column)
template <int MODE, int NT>
__global__ void __launch_bounds__(kGqrThreads, (NT <= 4 ? 3 : 2))
gqr_apply_kernel(const GqrBlock* __restrict__ blocks, const GqrTask* __restrict__ tasks,
                 const GqrState* __restrict__ state, double* data, double* q, const double* wbuf,
                 const double* part, int r, std::int64_t wsz, std::int64_t psz, int nbuf, int bufsz) {
  extern __shared__ __align__(16) double sm[];
  const GqrTask tk = tasks[blockIdx.x];
  const GqrBlock b = blocks[tk.block];
  const GqrState* st = state + tk.block;
  if (st->done) return;
  const int kq = st->kq, j = st->j;
  if (j == 0) return;
  if (MODE == 2 && st->last) return;

  const double* xb;
  double* ob;
  std::int64_t ldx, ldo;
  int nin, nout;
  if (MODE == 0) {
    xb = data + b.a + tk.row0;
    ldx = b.lda;
    nin = r;
    ob = q + b.out + tk.row0 + std::int64_t(kq) * b.ldo;
    ldo = b.ldo;
    nout = j;
  } else if (MODE == 1) {
    xb = q + b.out + tk.row0;
    ldx = b.ldo;
    nin = kq + j;
    ob = q + b.out + tk.row0 + std::int64_t(kq) * b.ldo;
    ldo = b.ldo;
    nout = j;
  } else {
    xb = q + b.out + tk.row0 + std::int64_t(kq) * b.ldo;
    ldx = b.ldo;
    nin = j;
    ob = data + b.a + tk.row0;
    ldo = b.lda;
    nout = r;
  }
  const int nin4 = up(nin, 4), nout8 = up(nout, 8), ldw = ld4(nin4);
  double* ws = sm;                // nout8 columns x ldw
  double* xs = sm + nout8 * ldw;  // nin4 columns x kLds
  // W into shared memory (zero-padded)
  if (MODE == 2) {
    const double* p0 = part + std::int64_t(b.task0) * psz;
    for (int e = threadIdx.x; e < nout8 * nin4; e += kGqrThreads) {
      const int c = e / nin4, i = e - c * nin4;
      ws[c * ldw + i] = (c < nout && i < nin) ? -p0[std::int64_t(c) * nin + i] : 0.0;
    }
  } else {
    const double* w = wbuf + std::int64_t(tk.block) * wsz;
    for (int e = threadIdx.x; e < nout8 * nin4; e += kGqrThreads) {
      const int c = e / nin4, i = e - c * nin4;
      ws[c * ldw + i] = (c < nout && i < nin) ? w[std::int64_t(c) * nin + i] : 0.0;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;  // m-tile pair, n-tile parity
  const int ntn = nout8 / 8;
  auto issue = [&](int s0, int buf) {
    const int rows = min(kSlice, tk.rows - s0);
    load_slice(xs + buf * bufsz, xb + s0, ldx, rows, nin, up(rows, 8), nin4);
    cp_async_commit();
  };
  issue(0, 0);
  for (int s0 = 0, it = 0; s0 < tk.rows; s0 += kSlice, ++it) {
    const int rows = min(kSlice, tk.rows - s0), rows8 = up(rows, 8);
    const bool more = s0 + kSlice < tk.rows;
    const int cur = nbuf == 2 ? (it & 1) : 0;
    if (nbuf == 2 && more) {
      issue(s0 + kSlice, cur ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();  // (also orders the W fill before its first use)
    const double* xc = xs + cur * bufsz;
    if (wm * 16 < rows8) {
      double acc[2][NT][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < NT; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
      const bool two = wm * 16 + 8 < rows8;
      for (int k0 = 0; k0 < nin4; k0 += 4) {
        const double a0 = xc[(k0 + t4) * kLds + wm * 16 + g];
        const double a1 = two ? xc[(k0 + t4) * kLds + wm * 16 + 8 + g] : 0.0;
#pragma unroll
        for (int v = 0; v < NT; ++v) {
          const int tn = wn + 2 * v;
          if (tn < ntn) {
            const double bf = ws[(tn * 8 + g) * ldw + k0 + t4];
            dmma8x8x4(acc[0][v][0], acc[0][v][1], a0, bf);
            if (two) dmma8x8x4(acc[1][v][0], acc[1][v][1], a1, bf);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int row = wm * 16 + u * 8 + g;
        if (row >= rows) continue;
#pragma unroll
        for (int v = 0; v < NT; ++v) {
          const int tn = wn + 2 * v;
          if (tn >= ntn) continue;
          const int d = tn * 8 + 2 * t4;
          double* o = ob + s0 + row + std::int64_t(d) * ldo;
          if (MODE == 2) {
            if (d < nout) o[0] += acc[u][v][0];
            if (d + 1 < nout) o[ldo] += acc[u][v][1];
          } else {
            if (d < nout) o[0] = acc[u][v][0];
            if (d + 1 < nout) o[ldo] = acc[u][v][1];
          }
        }
      }
    }
    if (more) {
      __syncthreads();
      if (nbuf == 1) issue(s0 + kSlice, 0);
    }
  }
}

// ------------------------------------------------------------------ small factorizations
// Partial Gram matrices of a block's row tasks summed into the first task's
// slot, in task order (blocks of one task: nothing to do). MODE as in
// gqr_gram_kernel (the element count).
template <int MODE>
__global__ void gqr_sum_kernel(const GqrBlock* __restrict__ blocks, const GqrState* __restrict__ state,
                               double* part, int r, std::int64_t psz) {
  const GqrBlock b = blocks[blockIdx.x];
  if (b.ntasks <= 1) return;
  const GqrState* st = state + blockIdx.x;
  if (st->done) return;
  if (MODE == 0 && st->last) return;
  if (MODE != 0 && st->j == 0) return;
  if (MODE == 2 && st->last) return;
  const int ne = MODE == 0 ? r * r : MODE == 1 ? (st->kq + st->j) * st->j : st->j * r;
  double* p0 = part + std::int64_t(b.task0) * psz;
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    double v = p0[e];
    for (int q = 1; q < b.ntasks; ++q) v += p0[std::int64_t(q) * psz + e];
    p0[e] = v;
  }
}

// Stage factorization: one CTA per block on the block's (summed) Gram
// matrix: pivoted Cholesky with the stage / rank / kmax stops; writes
// W1 = P X (r x j, ld r) and the block's state.
__global__ void __launch_bounds__(kCholThreads, 3)
gqr_pchol_kernel(const GqrBlock* __restrict__ blocks, GqrState* state, const double* part, double* wbuf,
                 int r, int kmax, double theta, double tol, int stage, std::int64_t psz, std::int64_t wsz,
                 int g_shared, double gap) {
  extern __shared__ __align__(16) double sm[];
  __shared__ CholShared cs;
  const GqrBlock b = blocks[blockIdx.x];
  GqrState* st = state + blockIdx.x;
  if (st->done) return;
  int kq = 0;
  if (stage > 0) {
    if (st->last) {
      if (threadIdx.x == 0) st->done = 1;
      return;
    }
    kq = st->kq + st->j;
  }
  const int ldl = r | 1, ldx = kmax | 1;
  double* L = sm;              // kmax columns x ldl
  double* X = sm + kmax * ldl;  // kmax columns x ldx
  const int t = threadIdx.x;
  const int steps = min(min(b.rows, r), kmax);
  const double* G = part + std::int64_t(b.task0) * psz;
  int ldg = r;
  if (g_shared) {  // the Gram matrix staged in shared memory: no L2 round trip per step
    double* Gs = X + kmax * ldx;
    for (int e = t; e < r * r; e += kCholThreads) {
      const int c = e / r;
      Gs[c * ldl + (e - c * r)] = G[e];
    }
    G = Gs;
    ldg = ldl;
    __syncthreads();
  }
  double d00 = stage > 0 ? st->d00 : 0.0;
  int last = 0;
  bool used = (t < r && stage > 0) ? st->used[t] != 0 : false;
  // (the last stage the launcher runs takes every pivot still owed)
  const CholStops stops{steps, theta, tol * tol, theta > 0.0 ? gap : 0.0};
  const int j = lazy_chol<true>(G, ldg, L, ldl, X, ldx, r, kq, steps - kq, stops, d00, last, used, cs);
  if (kq + j >= steps) last = 1;
  // W1(i, bq) = X(pos(i), bq) for the pivots i placed at or before bq
  double* w = wbuf + std::int64_t(blockIdx.x) * wsz;
  for (int e = t; e < r * j; e += kCholThreads) {
    const int bq = e / r, i = e - bq * r;
    const int pi = cs.pos[i];
    w[e] = (pi >= 0 && pi <= bq) ? X[bq * ldx + pi] : 0.0;
  }
  if (t < r) st->used[t] = used ? 1 : 0;
  if (t == 0) {
    st->kq = kq;
    st->j = j;
    st->last = last;
    st->d00 = d00;
    if (last) st->keep = kq + j;
  }
}

// Second pass: G2 = G1 - H^T H from the block's (summed) MODE-1 Gram matrix
// ([H; G1], (kq + j) x j), its Cholesky factor L2 and
// W2 = [-H X; X], X = L2^-T, ((kq + j) x j, ld kq + j).
__global__ void __launch_bounds__(kCholThreads, 2)
gqr_chol2_kernel(const GqrBlock* __restrict__ blocks, const GqrState* __restrict__ state, const double* part,
                 double* wbuf, int kmax, std::int64_t psz, std::int64_t wsz) {
  extern __shared__ __align__(16) double sm[];
  __shared__ CholShared cs;
  const GqrBlock b = blocks[blockIdx.x];
  const GqrState* st = state + blockIdx.x;
  if (st->done) return;
  const int kq = st->kq, j = st->j;
  if (j == 0) return;
  const int n = kq + j, lds = j | 1, ldh = kq | 1;
  double* S = sm;            // j x j, overwritten by L2
  double* X = S + j * lds;   // j x j (upper)
  double* H = X + j * lds;   // kq x j, H[c * ldh + q]
  const int t = threadIdx.x;
  const double* hg = part + std::int64_t(b.task0) * psz;
  for (int e = t; e < n * j; e += kCholThreads) {
    const int c = e / n, i = e - c * n;
    const double v = hg[e];
    if (i < kq)
      H[c * ldh + i] = v;
    else
      S[c * lds + (i - kq)] = v;
  }
  __syncthreads();
  if (kq > 0) {
    for (int e = t; e < j * j; e += kCholThreads) {
      const int c = e / j, i = e - c * j;
      double v = S[c * lds + i];
      for (int q = 0; q < kq; ++q) v = fma(-H[i * ldh + q], H[c * ldh + q], v);
      S[c * lds + i] = v;
    }
    __syncthreads();
  }
  double d00 = 0.0;
  int last = 0;
  bool used = false;
  const CholStops stops{0, 0.0, 0.0, 0.0};
  lazy_chol<false>(S, lds, S, lds, X, lds, j, 0, j, stops, d00, last, used, cs);
  double* w = wbuf + std::int64_t(blockIdx.x) * wsz;
  for (int e = t; e < n * j; e += kCholThreads) {
    const int c = e / n, i = e - c * n;
    double v;
    if (i >= kq) {
      v = i - kq <= c ? X[c * lds + (i - kq)] : 0.0;
    } else {
      v = 0.0;
      for (int q = 0; q <= c; ++q) v = fma(-H[q * ldh + i], X[c * lds + q], v);
    }
    w[e] = v;
  }
}

// Columns [keep, kmax) of Q zeroed; the kept rank to its slot.
__global__ void gqr_finish_kernel(const GqrBlock* __restrict__ blocks, const GqrTask* __restrict__ tasks,
                                  const GqrState* __restrict__ state, double* q, int* ranks, int kmax) {
  const GqrTask tk = tasks[blockIdx.x];
  const GqrBlock b = blocks[tk.block];
  const GqrState* st = state + tk.block;
  const bool nonfinite = st->amax >= kGqrNonFinite;
  const int keep = nonfinite ? 0 : (st->last ? st->keep : st->kq + st->j);
  if (nonfinite && tk.row0 == 0 && threadIdx.x == 0 && b.rank_slot >= 0) ranks[b.rank_slot] = -1;
  if (!nonfinite && tk.row0 == 0 && threadIdx.x == 0 && b.rank_slot >= 0) ranks[b.rank_slot] = keep;
  double* o = q + b.out + tk.row0;
  const int ncol = kmax - keep;
  for (int e = threadIdx.x; e < ncol * tk.rows; e += blockDim.x) {
    const int c = e / tk.rows, i = e - c * tk.rows;
    o[std::int64_t(keep + c) * b.ldo + i] = 0.0;
  }
}

// The Gram matrix squares the block's scale: blocks whose largest entry lies
// outside [2^-300, 2^300] are rescaled by an exact power of two first (Q and
// the kept rank do not depend on the scale; the Householder form has no such
// limit, so this keeps the same domain). Pass 1: largest |entry| per block.
__global__ void gqr_absmax_kernel(const GqrBlock* __restrict__ blocks, const GqrTask* __restrict__ tasks,
                                  GqrState* state, const double* data, int r) {
  const GqrTask tk = tasks[blockIdx.x];
  const GqrBlock b = blocks[tk.block];
  const double* y = data + b.a + tk.row0;
  double m = 0.0;
  bool bad = false;  // NaN / Inf: qr_orthonormal throws "non-finite matrix in qr" (linalg.cpp:59)
  for (int c = 0; c < r; ++c)
    for (int i = threadIdx.x; i < tk.rows; i += blockDim.x) {
      const double v = y[std::int64_t(c) * b.lda + i];
      bad |= !isfinite(v);
      m = fmax(m, fabs(v));
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (bad)
      atomicMax(&state[tk.block].amax, kGqrNonFinite);
    else if (m > 0.0)
      atomicMax(&state[tk.block].amax, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// Blocks with a non-finite entry report rank -1 (the driver raises the
// reference's exception): for the blocks the Householder kernels factor.
__global__ void gqr_flag_kernel(const GqrBlock* __restrict__ blocks, const GqrState* __restrict__ state, int* ranks,
                                int nb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb && state[i].amax >= kGqrNonFinite && blocks[i].rank_slot >= 0) ranks[blocks[i].rank_slot] = -1;
}

// Pass 2: out-of-range blocks scaled to a largest entry in [1, 2).
__global__ void gqr_rescale_kernel(const GqrBlock* __restrict__ blocks, const GqrTask* __restrict__ tasks,
                                   const GqrState* __restrict__ state, double* data, int r) {
  const GqrTask tk = tasks[blockIdx.x];
  const double m = __longlong_as_double(static_cast<long long>(state[tk.block].amax));
  if (!(m > 0.0) || (m >= 0x1p-300 && m <= 0x1p300) || !isfinite(m)) return;
  const GqrBlock b = blocks[tk.block];
  int e;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  double* y = data + b.a + tk.row0;
  for (int c = 0; c < r; ++c)
    for (int i = threadIdx.x; i < tk.rows; i += blockDim.x) {
      double& v = y[std::int64_t(c) * b.lda + i];
      v = scalbn(v, 1 - e);
    }
}

__global__ void gqr_init_kernel(GqrState* state, int nb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) {
    GqrState s{};
    state[i] = s;
  }
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  HP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

}  // namespace

bool gqr_supported(int r, int kmax) { return r >= 1 && r <= 96 && kmax >= 1 && kmax <= r; }

std::int64_t gqr_part_doubles(int r, int kmax) { return std::int64_t(r) * r; }
std::int64_t gqr_w_doubles(int r, int kmax) { return std::int64_t(r) * kmax; }

namespace {

// W: width class (tiles sized for r <= 8 W)
template <int W>
void launch_gqr_w(const GqrBlock* blocks, int nb, const GqrTask* tasks, int nt, GqrState* state, double* data,
                  double* q, double* part, double* wbuf, int* ranks, int r, int kmax, double tol,
                  cudaStream_t s) {
  static const double kTheta = std::getenv("HP_GQR_THETA") ? std::atof(std::getenv("HP_GQR_THETA")) : 1e-12;
  static const int kStages = std::getenv("HP_GQR_STAGES") ? std::atoi(std::getenv("HP_GQR_STAGES")) : 5;
  constexpr int NV = (W + 1) / 2, NU = (W + 3) / 4, NT = (W + 1) / 2;
  const std::int64_t psz = gqr_part_doubles(r, kmax), wsz = gqr_w_doubles(r, kmax);
  const int r8 = up(r, 8), k8 = up(kmax, 8);
  // shared-memory sizes (bytes) at the widest shapes
  const size_t sm_g0 = size_t(r8) * kLds * 8;
  const size_t sm_g1 = size_t(k8 + 8) * kLds * 8;
  const size_t sm_g2 = size_t(k8 + r8) * kLds * 8;
  const size_t w0 = size_t(k8) * ld4(up(r, 4)) * 8, w1 = size_t(k8) * ld4(up(kmax, 4)) * 8,
               w2 = size_t(r8) * ld4(up(kmax, 4)) * 8;
  const size_t sl_a0 = size_t(up(r, 4)) * kLds * 8, sl_a1 = size_t(up(kmax, 4)) * kLds * 8, sl_a2 = sl_a1;
  const size_t sm_pc0 = (size_t(kmax) * (r | 1) + size_t(kmax) * (kmax | 1)) * 8;
  // the Gram matrix joins L and X in shared memory while three CTAs per SM fit
  static const int g_force = std::getenv("HP_GQR_GSHARED") ? std::atoi(std::getenv("HP_GQR_GSHARED")) : -1;
  const int g_shared = g_force >= 0 ? g_force : ((sm_pc0 + size_t(r) * (r | 1) * 8) * 3 <= 216 * 1024 ? 1 : 0);
  const size_t sm_pc = sm_pc0 + (g_shared ? size_t(r) * (r | 1) * 8 : 0);
  // S and X (j x j each) + H ((kq + j <= kmax) : kq x j): j (j|1) 2 + j (kq|1) <= 2 kmax (kmax|1) + 2 kmax
  const size_t sm_c2 = (size_t(2) * kmax * (kmax | 1) + size_t(2) * kmax) * 8;
  // two slice buffers where the CTAs per SM the registers allow still fit
  auto two = [&](size_t fixed, size_t slice, int ctas) { return (fixed + 2 * slice) * ctas <= 208 * 1024 ? 2 : 1; };
  constexpr int cg = NV * NU <= 8 ? 3 : 2, ca = NT <= 4 ? 3 : 2;
  const int nb_g0 = two(0, sm_g0, cg), nb_g1 = two(0, sm_g1, cg), nb_g2 = two(0, sm_g2, cg);
  const int nb_a0 = two(w0, sl_a0, ca), nb_a1 = two(w1, sl_a1, ca), nb_a2 = two(w2, sl_a2, ca);
  // (function attributes are per device: a process may drive several)
  static bool attr_set[64] = {};
  int dev = 0;
  HP_CUDA(cudaGetDevice(&dev));
  bool& attr = attr_set[dev & 63];
  if (!attr) {
    set_smem(gqr_gram_kernel<0, NV, NU>, 200 * 1024);
    set_smem(gqr_gram_kernel<1, NV, NU>, 200 * 1024);
    set_smem(gqr_gram_kernel<2, NV, NU>, 200 * 1024);
    set_smem(gqr_apply_kernel<0, NT>, 200 * 1024);
    set_smem(gqr_apply_kernel<1, NT>, 200 * 1024);
    set_smem(gqr_apply_kernel<2, NT>, 200 * 1024);
    set_smem(gqr_pchol_kernel, 200 * 1024);
    set_smem(gqr_chol2_kernel, 200 * 1024);
    attr = true;
  }
  gqr_init_kernel<<<cdiv(nb, 256), 256, 0, s>>>(state, nb);
  HP_LAUNCHED();
  gqr_absmax_kernel<<<nt, 256, 0, s>>>(blocks, tasks, state, data, r);
  HP_LAUNCHED();
  gqr_rescale_kernel<<<nt, 256, 0, s>>>(blocks, tasks, state, data, r);
  HP_LAUNCHED();
  for (int stage = 0; stage < kStages; ++stage) {
    gqr_gram_kernel<0, NV, NU><<<nt, kGqrThreads, sm_g0 * nb_g0, s>>>(blocks, tasks, state, data, q, part, r, psz,
                                                                        nb_g0, int(sm_g0 / 8));
    HP_LAUNCHED();
    gqr_sum_kernel<0><<<nb, 256, 0, s>>>(blocks, state, part, r, psz);
    HP_LAUNCHED();
    gqr_pchol_kernel<<<nb, kCholThreads, sm_pc, s>>>(blocks, state, part, wbuf, r, kmax, stage + 1 < kStages ? kTheta : 0.0, tol, stage,
                                                      psz, wsz, g_shared, kGqrGapHost);
    HP_LAUNCHED();
    gqr_apply_kernel<0, NT><<<nt, kGqrThreads, w0 + sl_a0 * nb_a0, s>>>(blocks, tasks, state, data, q, wbuf, part,
                                                                         r, wsz, psz, nb_a0, int(sl_a0 / 8));
    HP_LAUNCHED();
    gqr_gram_kernel<1, NV, NU><<<nt, kGqrThreads, sm_g1 * nb_g1, s>>>(blocks, tasks, state, data, q, part, r, psz,
                                                                        nb_g1, int(sm_g1 / 8));
    HP_LAUNCHED();
    gqr_sum_kernel<1><<<nb, 256, 0, s>>>(blocks, state, part, r, psz);
    HP_LAUNCHED();
    gqr_chol2_kernel<<<nb, kCholThreads, sm_c2, s>>>(blocks, state, part, wbuf, kmax, psz, wsz);
    HP_LAUNCHED();
    gqr_apply_kernel<1, NT><<<nt, kGqrThreads, w1 + sl_a1 * nb_a1, s>>>(blocks, tasks, state, data, q, wbuf, part,
                                                                         r, wsz, psz, nb_a1, int(sl_a1 / 8));
    HP_LAUNCHED();
    if (stage + 1 < kStages) {
      gqr_gram_kernel<2, NV, NU><<<nt, kGqrThreads, sm_g2 * nb_g2, s>>>(blocks, tasks, state, data, q, part, r,
                                                                          psz, nb_g2, int(sm_g2 / 8));
      HP_LAUNCHED();
      gqr_sum_kernel<2><<<nb, 256, 0, s>>>(blocks, state, part, r, psz);
      HP_LAUNCHED();
      gqr_apply_kernel<2, NT><<<nt, kGqrThreads, w2 + sl_a2 * nb_a2, s>>>(blocks, tasks, state, data, q, wbuf,
                                                                           part, r, wsz, psz, nb_a2, int(sl_a2 / 8));
      HP_LAUNCHED();
    }
  }
  gqr_finish_kernel<<<nt, 128, 0, s>>>(blocks, tasks, state, q, ranks, kmax);
  HP_LAUNCHED();
}

}  // namespace

void launch_qr_rescale(const GqrBlock* blocks, int nb, const GqrTask* tasks, int nt, GqrState* state,
                       double* data, int r, cudaStream_t s) {
  if (nb == 0) return;
  gqr_init_kernel<<<cdiv(nb, 256), 256, 0, s>>>(state, nb);
  HP_LAUNCHED();
  gqr_absmax_kernel<<<nt, 256, 0, s>>>(blocks, tasks, state, data, r);
  HP_LAUNCHED();
  gqr_rescale_kernel<<<nt, 256, 0, s>>>(blocks, tasks, state, data, r);
  HP_LAUNCHED();
}

void launch_qr_flag(const GqrBlock* blocks, int nb, const GqrState* state, int* ranks, cudaStream_t s) {
  if (nb == 0) return;
  gqr_flag_kernel<<<cdiv(nb, 256), 256, 0, s>>>(blocks, state, ranks, nb);
  HP_LAUNCHED();
}

void launch_gqr(const GqrBlock* blocks, int nb, const GqrTask* tasks, int nt, GqrState* state, double* data,
                double* q, double* part, double* wbuf, int* ranks, int r, int kmax, double tol,
                cudaStream_t s) {
  if (nb == 0) return;
  if (!gqr_supported(r, kmax)) throw std::invalid_argument("gqr: unsupported widths");
  const int w = (r + 7) / 8;
#define HP_GQR(W) launch_gqr_w<W>(blocks, nb, tasks, nt, state, data, q, part, wbuf, ranks, r, kmax, tol, s)
  if (w <= 6)
    HP_GQR(6);
  else if (w <= 8)
    HP_GQR(8);
  else if (w <= 10)
    HP_GQR(10);
  else
    HP_GQR(12);
#undef HP_GQR
}

}  // namespace hpeel
