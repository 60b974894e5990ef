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

/// Count of kernel launches issued by this library (reported by bench.py as
/// gpu_launches; read through hp_launch_count).
std::int64_t& launch_counter();
#define HP_LAUNCHED()                     \
  do {                                    \
    HP_CUDA(cudaGetLastError());          \
    ++::hpeel::launch_counter();          \
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

/// 1/d to ~1 ulp: MUFU.RCP64H seed + two Newton steps (FP64 pipe only).
__device__ __forceinline__ double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

/// Natural log for positive normal x, |error| <= ~2 ulp (checked against
/// glibc in tests/test_gpu_kernels.py). x = 2^e m with m in [sqrt2/2, sqrt2),
/// log m = 2 atanh(s), s = (m-1)/(m+1), |s| <= 0.1716: series to z^8
/// (truncation < 3e-17 relative). ~21 FP64 ops vs ~56 for the libdevice log.
__device__ __forceinline__ double fast_log(double x) {
  int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  int e = (hi >> 20) - 1023;
  int mhi = (hi & 0x000fffff) | 0x3ff00000;
  if (mhi > 0x3ff6a09e) {  // m > sqrt(2): use m / 2
    mhi -= 0x00100000;
    e += 1;
  }
  const double m = __hiloint2double(mhi, lo);
  const double f = m - 1.0;
  const double s = f * fast_rcp(2.0 + f);
  const double z = s * s;
  double p = 1.0 / 19.0;
  p = fma(p, z, 1.0 / 17.0);
  p = fma(p, z, 1.0 / 15.0);
  p = fma(p, z, 1.0 / 13.0);
  p = fma(p, z, 1.0 / 11.0);
  p = fma(p, z, 1.0 / 9.0);
  p = fma(p, z, 1.0 / 7.0);
  p = fma(p, z, 1.0 / 5.0);
  p = fma(p, z, 1.0 / 3.0);
  const double s2 = s + s;
  const double lm = fma(s2 * z, p, s2);
  const double de = double(e);
  return fma(de, 6.93147180369123816490e-01, fma(de, 1.90821492927058770002e-10, lm));
}

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
    // subnormal / zero distances (coincident points) take the libdevice path
    if (DIM == 1) {
      const double d = fabs(xi[0] - xj[0]);
      return d >= 2.2250738585072014e-308 ? fast_log(d) : log(d);
    }
    return r2 >= 2.2250738585072014e-308 ? 0.5 * fast_log(r2) : 0.5 * log(r2);
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
