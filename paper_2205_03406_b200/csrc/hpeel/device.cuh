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
  kOpCallback = 4,   // caller-supplied apply / apply_adjoint (no device kernel evaluates it)
};

struct DevOp {
  int kind = kOpDense;
  int dim = 1;
  std::int64_t n = 0;
  const double* x = nullptr;   // dim x n, tree order, SoA (x[d * n + pos])
  const double* a = nullptr;   // kOpDense: n x n col-major, tree order
  double param = 1.0;          // kOpExp length scale
  int symmetric = 1;           // A == A^T: forward and adjoint share K(i, j)
  const double* ltab = nullptr;  // half_log table (2 x kLogTab doubles, device)
};

/// fast_log table on `device` (built once per device, never freed).
const double* log_table_device(int device);

/// 1/d to ~1 ulp: MUFU.RCP64H seed + two Newton steps (FP64 pipe only).
__device__ __forceinline__ double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

/// 1/sqrt(x) for positive normal x to ~1 ulp: MUFU.RSQ64H seed (2^-22) and
/// two Newton steps on the FP64 pipe (9 instructions; rsqrt() adds the
/// special-case paths the unchecked K2 tiles never take).
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double t = x * y;
  double e = fma(-t, y, 1.0);
  y = fma(0.5 * y, e, y);
  t = x * y;
  e = fma(-t, y, 1.0);
  return fma(0.5 * y, e, y);
}

/// Table for half_log (built on the host in extended precision, see
/// log_table_device): kLogTab pairs {1/(2 T_k), 0.5 log(T_k')}, 16-byte aligned.
constexpr int kLogBits = 10;                      // T_k = 1 + k / 1024
constexpr int kLogTab = (1 << kLogBits) + 1;
constexpr int kLogSplit = 425;                    // first k with T_k >= sqrt 2: reduce m / 2 against T_k / 2

/// 0.5 * log(x) for positive normal x, <= 2 ulp of 0.5 log x
/// (tests/test_gpu_kernels.py checks 2 * half_log against glibc log).
/// x = 2^e m, m in [1, 2); the top 11 mantissa bits round to the nearest
/// T_k = 1 + k/1024 (k in 0..1024; T = 1 is hit exactly from either side of
/// x = 1, where the table value is 0) and v = (m / T_k - 1) / 2, |v| <= 2^-12,
/// so 0.5 log1p(2v) is a degree-5 series (remainder < 5e-18 relative). The 1/2
/// is folded into the table and the coefficients; the exponent converts
/// exactly through the 2^52 bias: 11 FP64 ops and one 16-byte table read.
__device__ __forceinline__ double half_log(double x, const double* __restrict__ tab) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  // k = round(4096 (m - 1)); e' + 1023 = biased exponent, plus one when the
  // mantissa reaches the split (k >= kLogSplit): a carry into the exponent
  constexpr int kHalf = 1 << (19 - kLogBits);
  const int k = ((hi & 0x000fffff) + kHalf) >> (20 - kLogBits);
  const int eb = (hi + (0x100000 - ((kLogSplit << (20 - kLogBits)) - kHalf))) >> 20;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double2 t = reinterpret_cast<const double2*>(tab)[k];
  const double v = fma(m, t.x, -0.5);
  // 0.5 log1p(2v) = v - v^2 + 4/3 v^3 - 2 v^4 + 16/5 v^5 - ...
  double q = fma(16.0 / 5.0, v, -2.0);
  q = fma(q, v, 4.0 / 3.0);
  q = fma(q, v, -1.0);
  const double lp = fma(v * v, q, v);
  const double de = __hiloint2double(0x43300000, eb) - 4503599627371519.0;  // - (2^52 + 1023)
  return fma(de, 3.46573590279972654709e-01, t.y) + lp;
}

/// K(x_i, x_j) for the on-the-fly kinds, from coordinates already in
/// registers. `same` is true iff i == j (tree positions); `ltab` is the
/// half_log table (log kernels only). CHECK = false drops the i == j and
/// coincident-point cases, for callers that know neither occurs (K2 tiles
/// whose row box is not in the payload, on clouds without duplicate points).
template <int KIND, int DIM, bool CHECK = true>
__device__ __forceinline__ double kernel_value(const double* xi, const double* xj, bool same,
                                               double param, const double* ltab) {
  double r2 = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const double t = xi[d] - xj[d];
    r2 = fma(t, t, r2);
  }
  if (KIND == kOpLog) {
    // log|x - y| = 0.5 log r^2; coincident distinct points give -inf as the
    // dense assembly would (integer test: r2 >= 0); sub-normal r^2
    // (< 2.2e-308) is outside the supported range
    const double v = half_log(r2, ltab);
    if (!CHECK) return v;
    const bool zero = (__double2hiint(r2) | __double2loint(r2)) == 0;  // same => zero
    return zero ? (same ? 0.0 : -INFINITY) : v;
  } else if (KIND == kOpInvDist4Pi) {
    if (CHECK && same) return 0.0;
    // unchecked tiles: r2 > 0 (no coincident points, i != j)
    return (CHECK ? rsqrt(r2) : fast_rsqrt(r2)) * 0.07957747154594767;  // 1 / (4 pi)
  } else {
    // sqrt(r2) = r2 / sqrt(r2), r2 > 0; 1 / param is loop-invariant (hoisted): one multiply
    // instead of a division per entry (the argument moves by <= 1 ulp: <= 2e-15 of the value)
    if (!CHECK) return exp(-(r2 * fast_rsqrt(r2)) * (1.0 / param));
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
