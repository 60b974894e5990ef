// How do DMMA.8x8x4 and scalar FP64 share the FP64 datapath on B200?
// One CTA per SM, 8 "DMMA" warps (22 independent accumulator pairs, like K2)
// and 8 "scalar" warps issuing DFMA in CHAINS independent dependency chains.
// Prints, per configuration, the time and the datapath occupancy implied by
// 16 clk per DMMA and 2 clk per warp DFMA per SM sub-partition.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CHAINS, int NDMMA_WARPS, int NSCALAR_WARPS>
__global__ void mix_kernel(double* out, int iters, int dfma_per_iter, double s) {
  const int warp = threadIdx.x / 32;
  if (warp < NDMMA_WARPS) {
    double c[22][2];
#pragma unroll
    for (int i = 0; i < 22; ++i) c[i][0] = c[i][1] = 0;
    double a = 1.0 + threadIdx.x * 1e-3, b = 0.999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 22; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 22; ++i) t += c[i][0] + c[i][1];
    if (t == 1.2345) out[threadIdx.x] = t;
  } else if (warp < NDMMA_WARPS + NSCALAR_WARPS) {
    double acc[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x + c;
    const int n = iters * dfma_per_iter / CHAINS;
    for (int it = 0; it < n; ++it) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], s, 0.5);
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) t += acc[c];
    if (t == 1.2345) out[threadIdx.x] = t;
  }
}

// fused-K2 shape: each warp alternates a burst of 22 DMMAs with 2 chains of
// CH dependent DFMAs (the next k-step's kernel evaluations)
template <int CH, int WARPS>
__global__ void alt_kernel(double* out, int iters, int, double s) {
  double c[22][2];
#pragma unroll
  for (int i = 0; i < 22; ++i) c[i][0] = c[i][1] = 0;
  double a0 = 1.0 + threadIdx.x * 1e-3, a1 = a0 * 0.5, b = 0.999;
  for (int it = 0; it < iters; ++it) {
    double n0 = a0, n1 = a1;
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      n0 = fma(n0, s, 0.5);
      n1 = fma(n1, s, 0.25);
    }
#pragma unroll
    for (int i = 0; i < 11; ++i) {
      dmma(c[2 * i][0], c[2 * i][1], a0, b);
      dmma(c[2 * i + 1][0], c[2 * i + 1][1], a1, b);
    }
    a0 = n0;
    a1 = n1;
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 22; ++i) t += c[i][0] + c[i][1];
  if (t == 1.2345) out[threadIdx.x] = t;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  const double clk = prop.clockRate * 1e3;  // Hz (max boost)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  auto run = [&](const char* name, auto kern, int threads, int ndmma, int nscal, int dfma_per_iter) {
    kern<<<sms, threads>>>(out, iters, dfma_per_iter, 0.999);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<sms, threads>>>(out, iters, dfma_per_iter, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per SMSP pipe clocks demanded: DMMA 16 clk, DFMA (warp) 2 clk
    const double dmma_clk = double(ndmma) / 4 * iters * 22 * 16;
    const double dfma_clk = double(nscal) / 4 * iters * dfma_per_iter * 2;
    const double cyc = ms * 1e-3 * clk;
    printf("{\"case\": \"%s\", \"ms\": %.3f, \"pipe_busy\": %.3f, \"dmma_share\": %.3f}\n", name, ms,
           (dmma_clk + dfma_clk) / cyc, dmma_clk / cyc);
  };
  run("dmma 2/smsp", mix_kernel<1, 8, 0>, 256, 8, 0, 0);
  run("dmma 1/smsp", mix_kernel<1, 4, 0>, 128, 4, 0, 0);
  run("dmma 4/smsp", mix_kernel<1, 16, 0>, 512, 16, 0, 0);
  // K2's ratio: ~26 scalar FP64 per 22 DMMA per warp-pair
  run("mix chains=1", mix_kernel<1, 8, 8>, 512, 8, 8, 26);
  run("mix chains=2", mix_kernel<2, 8, 8>, 512, 8, 8, 26);
  run("mix chains=4", mix_kernel<4, 8, 8>, 512, 8, 8, 26);
  run("mix chains=8", mix_kernel<8, 8, 8>, 512, 8, 8, 26);
  run("mix chains=8 x2", mix_kernel<8, 8, 8>, 512, 8, 8, 52);
  run("dfma only chains=8", mix_kernel<8, 0, 8>, 256, 0, 8, 26);
  run("dfma only chains=1", mix_kernel<1, 0, 8>, 256, 0, 8, 26);
  auto run_alt = [&](const char* name, auto kern, int threads, int ch) {
    kern<<<sms, threads>>>(out, iters, 0, 0.999);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<sms, threads>>>(out, iters, 0, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double w = threads / 32 / 4.0;
    const double dmma_clk = w * iters * 22 * 16, dfma_clk = w * iters * 2 * ch * 2;
    const double cyc = ms * 1e-3 * clk;
    printf("{\"case\": \"%s\", \"ms\": %.3f, \"pipe_busy\": %.3f, \"dmma_share\": %.3f}\n", name, ms,
           (dmma_clk + dfma_clk) / cyc, dmma_clk / cyc);
  };
  run_alt("alt ch=13 4/smsp", alt_kernel<13, 16>, 512, 13);
  run_alt("alt ch=13 2/smsp", alt_kernel<13, 8>, 256, 13);
  run_alt("alt ch=26 4/smsp", alt_kernel<26, 16>, 512, 26);
  return 0;
}
