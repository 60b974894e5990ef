// Microbenchmark: tcgen05.mma kind::i8 (M = 128, K = 32) issue rate per SM for
// several N, with G accumulator groups rotated like the int8 K2 kernel, A/B
// from shared memory (SWIZZLE_NONE or SWIZZLE_32B descriptors).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_bench tools/umma_i8_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ std::uint64_t desc(unsigned addr, int layout, unsigned lbo, unsigned sbo) {
  return std::uint64_t((addr >> 4) & 0x3FFFu) | (std::uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (std::uint64_t((sbo >> 4) & 0x3FFF) << 32) | (std::uint64_t(1) << 46) | (std::uint64_t(layout) << 61);
}
// pattern 0: per group g, its g + 1 MMAs back to back (groups accumulators);
// pattern 1: 28 MMAs spread over `groups` slots, round-robin (slot = m % groups)
template <int N, int PAT>
__global__ void bench(int iters, int groups, int layout, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ std::uint64_t bar, bar2;
  __shared__ unsigned tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 7 * 4096 + 7 * 256 * 32; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(sa(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | (unsigned(N >> 3) << 17) | (8u << 24);
  const unsigned lbo = layout == 0 ? 128 : 16, sbo = layout == 0 ? 256 : 256;
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    int n = 0;
    if (PAT == 5 || PAT == 6) {
      // the K2 kernel's 28 digit-pair MMAs per K-step (SS): PAT 5 group-major
      // (A plane changes every MMA), PAT 6 plane-major (7 - a MMAs per A plane)
      for (int it = 0; it < iters; ++it) {
        if (PAT == 5) {
#pragma unroll
          for (int g = 0; g < 7; ++g)
#pragma unroll
            for (int a = 0; a <= g; ++a) {
              const unsigned ad = sa(sm) + a * 4096, bd = sa(sm) + 7 * 4096 + (g - a) * N * 32;
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase + unsigned(g * N)),
                           "l"(desc(ad, layout, lbo, sbo)), "l"(desc(bd, layout, lbo, sbo)), "r"(idesc), "r"(1u));
              ++n;
            }
        } else {
#pragma unroll
          for (int a = 0; a < 7; ++a)
#pragma unroll
            for (int b = 0; a + b < 7; ++b) {
              const unsigned ad = sa(sm) + a * 4096, bd = sa(sm) + 7 * 4096 + b * N * 32;
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase + unsigned((a + b) * N)),
                           "l"(desc(ad, layout, lbo, sbo)), "l"(desc(bd, layout, lbo, sbo)), "r"(idesc), "r"(1u));
              ++n;
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar2)));
      }
    } else
    if (PAT == 3 || PAT == 4) {
      for (int it = 0; it < iters; ++it) {
        const unsigned abuf = tbase + 448 + (it & 1) * 0;  // one A buffer at columns 448..503
#pragma unroll
        for (int a = 0; a < 7; ++a)
          if (PAT == 3)
          asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(abuf + a * 8),
                       "l"(desc(sa(sm) + a * 4096, layout, lbo, sbo)));
#pragma unroll
        for (int m = 0; m < 28; ++m) {
          const unsigned bd = sa(sm) + 7 * 4096 + ((m / 7) % 7) * N * 32;
          const unsigned d = tbase + unsigned(((m % groups) * N) % 448);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(abuf + (m % 7) * 8), "l"(desc(bd, layout, lbo, sbo)), "r"(idesc), "r"(1u));
          ++n;
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar2)));
      }
    } else
    if (PAT == 1 || PAT == 2) {
      for (int it = 0; it < iters; ++it) {
        if (PAT == 2 && it > 0)  // commit after every 28 MMAs (as the K2 kernel does per K-step)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar2)));
#pragma unroll
        for (int m = 0; m < 28; ++m) {
          const unsigned ad = sa(sm) + (m % 7) * 4096, bd = sa(sm) + 7 * 4096 + ((m / 7) % 7) * N * 32;
          const unsigned d = tbase + unsigned(((m % groups) * N) % 512);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(desc(ad, layout, lbo, sbo)), "l"(desc(bd, layout, lbo, sbo)), "r"(idesc), "r"(1u));
          ++n;
        }
      }
    } else
    for (int it = 0; it < iters; ++it) {
      for (int g = 0; g < groups; ++g)
        for (int a = 0; a <= g && a < 7; ++a) {
          const unsigned ad = sa(sm) + a * 4096, bd = sa(sm) + 7 * 4096 + (g - a) * N * 32;
          const unsigned d = tbase + unsigned((g * N) % 512);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(desc(ad, layout, lbo, sbo)), "l"(desc(bd, layout, lbo, sbo)), "r"(idesc), "r"(1u));
          ++n;
        }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(sa(&bar)));
    const long long t1 = clock64();
    cyc[blockIdx.x * 2] = t1 - t0;
    cyc[blockIdx.x * 2 + 1] = n;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int N, int PAT = 0>
void run(int groups, int layout) {
  long long* d;
  cudaMalloc(&d, 148 * 2 * 8);
  const int smem = 7 * 4096 + 7 * 256 * 32 + 1024;
  cudaFuncSetAttribute(bench<N, PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<N, PAT><<<148, 128, smem>>>(200, groups, layout, d);
  cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double clk = double(h[0]) / double(h[1]);
  const double macs = 128.0 * N * 32;
  std::printf("pat=%d N=%3d groups=%d layout=%d: %.1f clk/MMA, %.0f MAC/clk/SM (%.0f%% of 7737)  err=%s\n", PAT, N, groups,
              layout, clk, macs / clk, 100.0 * macs / clk / 7737.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<48, 5>(7, 0);
  run<48, 6>(7, 0);
  run<64, 5>(7, 0);
  run<64, 6>(7, 0);
  return 0;
}
