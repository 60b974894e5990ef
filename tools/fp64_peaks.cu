// FP64 roofline microbenchmark for B200 (sm_100a): DFMA, DMMA.8x8x4, mixed,
// and the cost of the kernel evaluations used by the black-box apply.
// Prints one JSON line. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double s) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], s, 0.5);
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) t += acc[c];
  if (t == 1.2345) out[threadIdx.x] = t;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) t += c[i][0] + c[i][1];
  if (t == 1.2345) out[threadIdx.x] = t;
}

// half the warps do DMMA, half do DFMA: do they share the FP64 pipe?
__global__ void mixed_kernel(double* out, int iters, double s) {
  const int warp = threadIdx.x / 32;
  if (warp & 1) {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x + c;
    for (int it = 0; it < iters * 2; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], s, 0.5);
    }
    double t = 0;
    for (int c = 0; c < 8; ++c) t += acc[c];
    if (t == 1.2345) out[threadIdx.x] = t;
  } else {
    double c[8][2];
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    double a = 1.0 + threadIdx.x * 1e-3, b = 0.999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double t = 0;
    for (int i = 0; i < 8; ++i) t += c[i][0] + c[i][1];
    if (t == 1.2345) out[threadIdx.x] = t;
  }
}

template <int KIND>
__global__ void eval_kernel(double* out, int iters) {
  double x = 0.1 + threadIdx.x * 1e-4, acc = 0;
  for (int it = 0; it < iters; ++it) {
    double v;
    if (KIND == 0) v = log(x);
    else if (KIND == 1) v = rsqrt(x);
    else if (KIND == 2) v = exp(-x);
    else v = sqrt(x);
    acc += v;
    x += 1e-7;
  }
  if (acc == 1.2345) out[threadIdx.x] = acc;
}

int main() {
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
  };
  const int blocks = sms * 4, threads = 256, iters = 20000;
  float t_dfma = timeit([&] { dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999); });
  double dfma_tf = 2.0 * blocks * threads * 8.0 * iters / (t_dfma * 1e-3) / 1e12;
  float t_dmma = timeit([&] { dmma_kernel<8><<<blocks, threads>>>(out, iters / 4); });
  double dmma_tf = 2.0 * 256 * (blocks * threads / 32) * 8.0 * (iters / 4) / (t_dmma * 1e-3) / 1e12;
  float t_mix = timeit([&] { mixed_kernel<<<blocks, threads>>>(out, iters / 4, 0.999); });
  double mix_flops = 2.0 * 256 * (blocks * threads / 64) * 8.0 * (iters / 4) +
                     2.0 * (blocks * threads / 2) * 8.0 * (iters / 2);
  double mix_tf = mix_flops / (t_mix * 1e-3) / 1e12;
  const int eit = 4000;
  double evals = double(blocks) * threads * eit;
  float t_log = timeit([&] { eval_kernel<0><<<blocks, threads>>>(out, eit); });
  float t_rsq = timeit([&] { eval_kernel<1><<<blocks, threads>>>(out, eit); });
  float t_exp = timeit([&] { eval_kernel<2><<<blocks, threads>>>(out, eit); });
  float t_sqrt = timeit([&] { eval_kernel<3><<<blocks, threads>>>(out, eit); });
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"mixed_tflops\": %.2f, "
         "\"log_gevals\": %.1f, \"rsqrt_gevals\": %.1f, \"exp_gevals\": %.1f, \"sqrt_gevals\": %.1f}\n",
         prop.name, sms, dfma_tf, dmma_tf, mix_tf, evals / (t_log * 1e-3) / 1e9,
         evals / (t_rsq * 1e-3) / 1e9, evals / (t_exp * 1e-3) / 1e9, evals / (t_sqrt * 1e-3) / 1e9);
  return 0;
}
