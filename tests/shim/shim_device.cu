// Device-pointer variant of the callback boundary (hp_op_callback with
// device_pointers = 1): the black box runs on the device on the stream the
// driver hands it (cuBLAS DGEMM on the operator's explicit matrix), as a
// GPU-resident application operator (an FMM, a sparse solve) would. Compared
// with the same operator through the host-pointer variant. Built by
// tests/test_shim.py with nvcc ... -lcublas.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "hpeel_b200.h"

namespace {
struct DevDense {
  int64_t n;
  double* d_a;
  std::vector<double> h_a;
  cublasHandle_t blas;
  int calls = 0;
};

int apply_device(void* ctx, int adjoint, const double* x, int64_t w, double* y, void* stream) {
  auto* op = static_cast<DevDense*>(ctx);
  const double one = 1.0, zero = 0.0;
  if (cublasSetStream(op->blas, static_cast<cudaStream_t>(stream)) != CUBLAS_STATUS_SUCCESS) return 1;
  const int n = int(op->n);
  if (cublasDgemm(op->blas, adjoint ? CUBLAS_OP_T : CUBLAS_OP_N, CUBLAS_OP_N, n, int(w), n, &one, op->d_a, n, x, n,
                  &zero, y, n) != CUBLAS_STATUS_SUCCESS)
    return 2;
  ++op->calls;
  return 0;
}

int apply_host(void* ctx, int adjoint, const double* x, int64_t w, double* y, void*) {
  auto* op = static_cast<DevDense*>(ctx);
  const int64_t n = op->n;
  for (int64_t c = 0; c < w; ++c)
    for (int64_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < n; ++j) acc += (adjoint ? op->h_a[j + i * n] : op->h_a[i + j * n]) * x[j + c * n];
      y[i + c * n] = acc;
    }
  ++op->calls;
  return 0;
}

void check(int rc) {
  if (rc != HP_OK) {
    std::fprintf(stderr, "hpeel error: %s\n", hp_last_error());
    std::exit(1);
  }
}
}  // namespace

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atol(argv[1]) : 1024;
  std::vector<double> pts(n);
  for (int64_t i = 0; i < n; ++i) pts[i] = (double(i) + 0.5) / double(n);
  DevDense op{n, nullptr, std::vector<double>(size_t(n * n)), nullptr};
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) op.h_a[size_t(i + j * n)] = i == j ? 0.0 : std::log(std::fabs(pts[i] - pts[j]));
  cudaMalloc(&op.d_a, size_t(n * n) * 8);
  cudaMemcpy(op.d_a, op.h_a.data(), size_t(n * n) * 8, cudaMemcpyHostToDevice);
  cublasCreate(&op.blas);
  hp_tree* tree = nullptr;
  check(hp_tree_build(pts.data(), n, 1, 64, &tree));
  hp_op *dev = nullptr, *host = nullptr, *builtin = nullptr;
  check(hp_op_callback(n, 1, 1, &apply_device, &op, 0, &dev));
  check(hp_op_callback(n, 1, 0, &apply_host, &op, 0, &host));
  check(hp_op_dense(op.h_a.data(), n, 0, &builtin));
  hp_rep *rd = nullptr, *rh = nullptr, *rb = nullptr;
  check(hp_compress(dev, tree, 20, 10, 7, HP_FORMAT_H1, HP_STRATEGY_GRAPH, 0, &rd));
  const int dev_calls = op.calls;
  check(hp_compress(host, tree, 20, 10, 7, HP_FORMAT_H1, HP_STRATEGY_GRAPH, 0, &rh));
  check(hp_compress(builtin, tree, 20, 10, 7, HP_FORMAT_H1, HP_STRATEGY_GRAPH, 0, &rb));
  std::vector<double> x(size_t(n) * 2), yd(x.size()), yh(x.size()), yb(x.size()), ya(x.size());
  for (size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.37 * double(i) + 1.0);
  check(hp_rep_apply(rd, 0, x.data(), 2, yd.data()));
  check(hp_rep_apply(rh, 0, x.data(), 2, yh.data()));
  check(hp_rep_apply(rb, 0, x.data(), 2, yb.data()));
  check(hp_op_apply(builtin, 0, x.data(), 2, ya.data()));
  auto rel = [&](const std::vector<double>& p, const std::vector<double>& q) {
    double a = 0, b = 0;
    for (size_t i = 0; i < p.size(); ++i) {
      a += (p[i] - q[i]) * (p[i] - q[i]);
      b += q[i] * q[i];
    }
    return std::sqrt(a / b);
  };
  double pm = 0.0;
  check(hp_rel_error_power_method(rd, dev, 20, 11, &pm));
  std::printf(
      "{\"n\": %ld, \"device_calls\": %d, \"dev_vs_host\": %.3e, \"dev_vs_builtin\": %.3e, "
      "\"dev_vs_operator\": %.3e, \"power_method_error\": %.3e}\n",
      long(n), dev_calls, rel(yd, yh), rel(yd, yb), rel(yd, ya), pm);
  hp_rep_free(rd);
  hp_rep_free(rh);
  hp_rep_free(rb);
  hp_op_free(dev);
  hp_op_free(host);
  hp_op_free(builtin);
  hp_tree_free(tree);
  cublasDestroy(op.blas);
  cudaFree(op.d_a);
  return 0;
}
