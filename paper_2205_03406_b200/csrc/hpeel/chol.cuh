// Small dense factorizations shared by K4 (k_gqr.cu) and K5 (k_bsolve2.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hpeel {

// Left-looking (lazy) Cholesky with the triangular inverse built alongside:
// step j needs only column p_j of G, the rows of L built so far and the
// downdated diagonal, so a step is one dot product per row (length j) and
// ONE block barrier. Threads [0, 96) own the rows of L (and the diagonal
// entry of their column); threads [96, 192) own the rows of
// X = (L restricted to the pivots)^-T, X(:, j) = (e_j - sum_b L(p_j, b) X(:, b)) / L_jj,
// the coefficients of Q1's column j over the pivot columns of Y.
// L and X are column-major in shared memory (a thread walks its row with
// stride ld: consecutive threads hit consecutive banks; the pivot row is a
// broadcast). G (column-major, ld ldg) may live in global memory: column p is
// read once, at its step. With PIVOT = false (natural order) L may alias G.
// smallest ld >= n with ld == 4 (mod 16) doubles: DMMA m8n8k4 fragment reads
// (8 x 4 elements per half-warp, either orientation) hit 16 distinct banks
__host__ __device__ constexpr int ld4(int n) { return (n + 11) / 16 * 16 + 4; }

constexpr int kCholThreads = 192;
constexpr int kCholRows = 96;

struct CholShared {
  double wbest[2][4];
  double wsecond[2][4];  // runner-up of the warp (PIVOT)
  int widx[2][4];
  int piv[96];
  int pos[96];  // pivot position of a column chosen in this call, else -1
};

struct CholStops {  // PIVOT only
  int steps;        // total pivots allowed (kq + j < steps)
  double theta, tol2;
  // The Schur diagonal carries ~1e-15 of the stage's first pivot in rounding
  // noise. A pivot is taken only when it beats the runner-up by more than
  // gap * (first pivot of the stage); otherwise the stage ends and the choice
  // is made on the Gram matrix of the deflated block, where it is resolved
  // to ~1e-15 relative (the exact-arithmetic greedy order, ties at the
  // accuracy of dgeqp3's own norm downdating).
  double gap;
};

template <bool PIVOT>
__device__ __forceinline__ int lazy_chol(const double* G, int ldg, double* L, int ldl, double* X, int ldx,
                                         int n, int kq, int jmax, const CholStops& stops, double& d00,
                                         int& last, bool& used, CholShared& cs, int* status = nullptr) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool is_a = t < kCholRows;
  const int i = t, bp = t - kCholRows;
  const bool row = is_a && i < n;
  double d = row ? G[std::int64_t(i) * ldg + i] : -1.0;
  int mypos = -1;
  // Warp argmax through two integer redux steps: a positive double orders
  // like its bit pattern; the low 7 mantissa bits (2^-45 relative, far under
  // the diagonal's own accuracy) carry 127 - column so that equal values go
  // to the lowest column and the winner is unique. Non-positive or used
  // diagonals take key 0; the winner publishes its unmodified value.
  auto publish = [&](int buf) {
    const bool cand = row && !used && d > 0.0;
    const unsigned hi = cand ? unsigned(__double2hiint(d)) : 0u;
    const unsigned lo = cand ? ((unsigned(__double2loint(d)) & ~127u) | unsigned(127 - (i & 127))) : 0u;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    if (mh == 0u && ml == 0u) {
      // nothing positive left in this warp: report its largest (non-positive) diagonal
      double key = (row && !used) ? d : -INFINITY;
      int idx = i;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, key, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ok > key || (ok == key && oi < idx)) {
          key = ok;
          idx = oi;
        }
      }
      if (lane == 0) {
        cs.wbest[buf][warp] = key;
        cs.widx[buf][warp] = idx;
      }
      if (lane == 0) cs.wsecond[buf][warp] = -INFINITY;
    } else {
      const bool win = cand && hi == mh && lo == ml;
      const unsigned mh2 = __reduce_max_sync(0xffffffffu, win ? 0u : hi);
      const unsigned ml2 = __reduce_max_sync(0xffffffffu, (!win && hi == mh2) ? lo : 0u);
      if (win) {
        cs.wbest[buf][warp] = d;
        cs.widx[buf][warp] = i;
        cs.wsecond[buf][warp] =
            (mh2 | ml2) ? __hiloint2double(int(mh2), int(ml2 & ~127u)) : -INFINITY;
      }
    }
  };
  if (PIVOT && is_a) publish(0);
  // natural order: the owner of the next pivot row publishes its downdated
  // diagonal before the step's barrier (a zero pivot marks a null column --
  // zero row and column of X, as the pseudo-inverse gives -- a negative one a
  // failed factorization)
  auto publish_next = [&](int jn) {
    cs.wbest[jn & 1][0] = d;
    if (status) status[jn] = d == 0.0 ? 1 : (d < 0.0 ? 2 : 0);
  };
  if (!PIVOT && row && i == 0) publish_next(0);
  if (is_a && i < 96) cs.pos[i] = -1;
  __syncthreads();
  double dstage = 0.0;
  int j = 0;
  while (j < jmax) {
    double dp;
    int p;
    if (PIVOT) {
      dp = cs.wbest[j & 1][0];
      p = cs.widx[j & 1][0];
      double d2 = cs.wsecond[j & 1][0];  // runner-up over all warps
#pragma unroll
      for (int w = 1; w < kCholRows / 32; ++w) {
        const double bw = cs.wbest[j & 1][w];
        if (bw > dp) {
          d2 = fmax(dp, cs.wsecond[j & 1][w]);
          dp = bw;
          p = cs.widx[j & 1][w];
        } else {
          d2 = fmax(d2, bw);
        }
      }
      if (kq + j == 0) {
        if (!(dp > 0.0)) {  // zero block
          last = 1;
          break;
        }
        d00 = dp;
      }
      if (j == 0) dstage = dp;
      if (!(dp > stops.tol2 * d00)) {  // |R_jj| <= tol |R_00|: numerical rank reached
        last = 1;
        break;
      }
      if (dp < stops.theta * dstage) break;  // next stage, on the deflated block
      if (j > 0 && dp - d2 < stops.gap * dstage) break;  // too close to call on this Gram matrix
    } else {
      p = j;
      dp = cs.wbest[j & 1][0];
    }
    const double rsq = dp > 0.0 ? rsqrt(dp) : 0.0;
    if (is_a) {
      if (row && !used) {
        if (i == p) {
          L[j * ldl + i] = dp * rsq;
          used = true;
          mypos = j;
          cs.piv[j] = p;
        } else {
          const double g = G[std::int64_t(p) * ldg + i];
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int q = 0;
          for (; q + 4 <= j; q += 4) {
            s0 = fma(L[q * ldl + i], L[q * ldl + p], s0);
            s1 = fma(L[(q + 1) * ldl + i], L[(q + 1) * ldl + p], s1);
            s2 = fma(L[(q + 2) * ldl + i], L[(q + 2) * ldl + p], s2);
            s3 = fma(L[(q + 3) * ldl + i], L[(q + 3) * ldl + p], s3);
          }
          for (; q < j; ++q) s0 = fma(L[q * ldl + i], L[q * ldl + p], s0);
          const double l = (g - ((s0 + s1) + (s2 + s3))) * rsq;
          L[j * ldl + i] = l;
          d = fma(-l, l, d);
          if (!PIVOT && i == j + 1) publish_next(j + 1);
        }
      }
      if (PIVOT) publish((j + 1) & 1);
    } else if (bp <= j || (status && bp < n)) {
      if (bp > j) {
        X[j * ldx + bp] = 0.0;  // X is upper triangular; K5 multiplies by all of it
      } else if (bp == j) {
        X[j * ldx + bp] = rsq;
      } else {
        double s0 = 0.0, s1 = 0.0;
        int q = bp;
        for (; q + 2 <= j; q += 2) {
          s0 = fma(X[q * ldx + bp], L[q * ldl + p], s0);
          s1 = fma(X[(q + 1) * ldx + bp], L[(q + 1) * ldl + p], s1);
        }
        if (q < j) s0 = fma(X[q * ldx + bp], L[q * ldl + p], s0);
        X[j * ldx + bp] = -(s0 + s1) * rsq;
      }
    }
    __syncthreads();
    ++j;
  }
  if (row) cs.pos[i] = mypos;
  __syncthreads();
  return j;
}

}  // namespace hpeel
