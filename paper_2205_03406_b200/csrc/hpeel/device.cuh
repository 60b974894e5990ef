// Device-side primitives shared by the sm_100a kernels: error checking, the
// on-the-fly black-box kernel evaluator and the FP64 DMMA (m8n8k4) wrapper.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace hpeel {

#define HP_CUDA(call)                                                                \
  do {                                                                               \
    cudaError_t err__ = (call);                                                      \
    if (err__ != cudaSuccess)                                                        \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(err__) + \
                               " at " + __FILE__ + ":" + std::to_string(__LINE__));  \
  } while (0)

/// Black-box kinds behind the LinearOperator boundary
/// (proj/include/hpeel/linear_operator.hpp:12-24). kDense is the reference's
/// DenseOperator (proj/include/hpeel/operators.hpp:56-69) held in HBM; the
/// kernel kinds are the on-the-fly operators named in BASELINE.json.
enum OpKind : int {
  kOpDense = 0,      // explicit N x N matrix
  kOpLog = 1,        // log|x - y|, A_ii = 0
  kOpInvDist4Pi = 2, // 1 / (4 pi |x - y|), A_ii = 0
  kOpExp = 3,        // exp(-|x - y| / ell), A_ii = 1
};

struct DevOp {
  int kind = kOpDense;
  int dim = 1;
  std::int64_t n = 0;
  const double* x = nullptr;   // dim x n, tree order, SoA (x[d * n + pos])
  const double* a = nullptr;   // kOpDense: n x n col-major, tree order
  double param = 1.0;          // kOpExp length scale
  int symmetric = 1;           // A == A^T: forward and adjoint share K(i, j)
};

/// K(x_i, x_j) for the on-the-fly kinds, from coordinates already in
/// registers. `same` is true iff i == j (tree positions).
template <int KIND, int DIM>
__device__ __forceinline__ double kernel_value(const double* xi, const double* xj, bool same,
                                               double param) {
  double r2 = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const double t = xi[d] - xj[d];
    r2 = fma(t, t, r2);
  }
  if (KIND == kOpLog) {
    if (same) return 0.0;
    if (DIM == 1) return log(fabs(xi[0] - xj[0]));
    return 0.5 * log(r2);
  } else if (KIND == kOpInvDist4Pi) {
    if (same) return 0.0;
    return rsqrt(r2) * 0.07957747154594767;  // 1 / (4 pi)
  } else {
    return exp(-sqrt(r2) / param);
  }
}

/// D = A(8x4, row) * B(4x8, col) + C; fragments per PTX m8n8k4 f64:
/// a: (lane/4, lane%4); b: (k = lane%4, n = lane/4); c: (lane/4, 2*(lane%4)+i).
__device__ __forceinline__ void dmma8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

inline unsigned cdiv(std::int64_t a, std::int64_t b) { return unsigned((a + b - 1) / b); }

}  // namespace hpeel
