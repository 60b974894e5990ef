// K2 black-box apply on the INT8 tensor cores (tcgen05.mma.kind::i8, TMEM
// accumulators): the FP64 contraction Y = K(rows, payload) * Omega is
// computed exactly in fixed point and rounded once.
//
// Each operand entry is split into a fixed-point integer relative to a
// power-of-two scale -- kernel entries: 62 bits against a per-row bound from
// the payload boxes' bounding boxes, written as 8 balanced int8 digits
// (weights 2^56 .. 2^0); payload: 54 bits against 16 >= the Box-Muller
// maximum 8.6, 7 digits (2^48 .. 2^0). Digit products with a + b <= 7
// (group split; a + b <= 6 in the column-split layout) are accumulated per
// group g = a + b in int32 TMEM columns (exact), and the epilogue forms
// Y = sum_g 2^(w_g) P_g in FP64. The kernel entries' rounding (2^-63 of the
// row bound: entries far below the bound keep ~60 bits, where 54 bits had
// left the log kernel's near-zero values with ~1e-14 relative error), the
// payload's (2^-55 of 16) and the dropped groups give errors ~1e-16 of the
// unpeeled product, so after peeling has cancelled most of it (post-peel
// blocks are up to ~100x smaller at the deep levels of config 3) the samples
// stay well inside 1e-12 of the FP64 apply (tests/test_gpu_fullsize.py).
//
// One CTA = 128 packed output rows (the K2Task/K2Row tiles of k2_ws.cuh) x one
// half of the sample columns (forward or adjoint, N = r padded to 16), so the
// 7 accumulator groups fit the 512 TMEM columns. Warps 0-7 evaluate the
// kernel tile (thread = one row x 16 payload rows per 32-row K-step), split it
// into digit planes and store them in the UMMA K-major no-swizzle layout;
// warp 8 lane 0 streams the precomputed payload digit planes with
// cp.async.bulk and issues the 28 MMAs per K-step. int32 accumulators are
// drained to FP64 every 512 K-steps (16384 payload rows), before any can
// overflow (7 * 128 * 128 * 16384 < 2^31).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "device.cuh"
#include "kernels.hpp"

namespace hpeel {
namespace k2i8 {

constexpr int kPlanes = 7;   // payload (B) digit planes: 54-bit fixed point
constexpr int kPlanesA = 8;  // kernel-entry (A) digit planes: 62-bit fixed point
constexpr int kGroups = 7;
constexpr int kStepK = 32;
constexpr int kWindow = 512;
constexpr int kEvalWarps = 16;
constexpr int kThreads = (kEvalWarps + 3) * 32;  // + MMA warp + peer-copy warp + load warp
constexpr int kRows = 128;
#ifndef HP_K2I8_TS
#define HP_K2I8_TS 1
#endif
constexpr bool kTSEnabled = HP_K2I8_TS != 0;
constexpr int kAPlane = kRows * kStepK;  // bytes of one A digit plane per K-step
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52

__host__ __device__ constexpr int padded_width(int r) { return (r + 15) / 16 * 16; }
/// Group split (NP <= 48): the CTA pair divides the digit-pair groups
/// g = a + b <= 7 between its CTAs, each for all 2 NP sample columns (one MMA
/// of N = 2 NP per digit pair): CTA 0 holds groups {0, 1, 2, 4, 7} and CTA 1
/// {3, 5, 6}, 17 + 17 MMAs per K-step. Otherwise (NP = 64) CTA h owns column
/// half h for the groups 0..6.
constexpr int kGroupsGS = 8;
__host__ __device__ constexpr unsigned gs_groups(int half) { return half == 0 ? 0x97u : 0x68u; }
__host__ __device__ constexpr int gs_slots(int half) { return half == 0 ? 5 : 3; }
__host__ __device__ constexpr bool group_split(int np) { return gs_slots(0) * 2 * np <= 512 && gs_slots(1) * 2 * np <= 512; }
__host__ __device__ constexpr int mma_n(int np) { return group_split(np) ? 2 * np : np; }
__host__ __device__ constexpr int b_step_bytes(int np) { return kPlanes * np * kStepK; }
/// Pipeline depth: 4 digit-tile (A) stages and 4 payload digit + coordinate
/// (B) stages (a deeper B ring measured slower: 1.44 s vs 1.26 s on c3).
constexpr int kAStages = 4;
constexpr int kStaticSmem = 9216 + 1024;
__host__ __device__ constexpr int b_ring_bytes(int np) { return b_step_bytes(np) + 3 * kStepK * 8; }
__host__ __device__ constexpr int bstages_for(int np, bool tab) { return (void)np, (void)tab, 3; }
__host__ __device__ constexpr size_t smem_bytes(int np, bool tab) {
  return size_t(kAStages) * kPlanesA * kAPlane + size_t(bstages_for(np, tab)) * b_ring_bytes(mma_n(np)) +
         (tab ? 2 * kLogTab * 8 : 0) + 1024;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// UMMA shared-memory descriptor: K-major, no swizzle; core matrices of 8 rows
// x 16 bytes, K-halves LBO = 128 bytes apart, 8-row groups SBO = 256 bytes.
__device__ __forceinline__ std::uint64_t umma_desc(unsigned addr) {
  return std::uint64_t((addr >> 4) & 0x3FFFu) | (std::uint64_t(128 >> 4) << 16) |
         (std::uint64_t(256 >> 4) << 32) | (std::uint64_t(1) << 46);
}
// instruction descriptor: s8 x s8 -> s32, both K-major, M = 128, N = np
__host__ __device__ constexpr unsigned umma_idesc(int np) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (unsigned(np >> 3) << 17) | (unsigned(kRows >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(unsigned d, std::uint64_t a, std::uint64_t b, unsigned idesc,
                                        unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// A operand from TMEM (128 lanes x 32 bytes of K in 8 columns)
__device__ __forceinline__ void umma_i8_ts(unsigned d, unsigned a_tmem, std::uint64_t b, unsigned idesc,
                                           unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// smem (UMMA descriptor, 128 rows x 32 bytes) -> TMEM 128 lanes x 8 columns
__device__ __forceinline__ void tmem_cp_128x256b(unsigned taddr, std::uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}
__device__ __forceinline__ void umma_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(unsigned taddr, int (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld4(unsigned taddr, int (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------ digit split
// v * c (|v * c| <= 2^30, c a power of two) -> X = hi * 2^24 + lo rounded
// to an integer, returned biased: uh = hi + 0x808080, ul = lo + 0x8080, so
// digit planes are bytes of uh / ul (planes 1-3, 5, 6 xor 0x80; planes 0
// and 4 are the arithmetic tops).
__device__ __forceinline__ void split_digits(double v, double c, unsigned& uh, unsigned& ul) {
  const double t = fma(v, c, kMagic);
  int hi = __double2loint(t);
  const double hf = t - kMagic;
  const double rem = fma(v, c, -hf);
  int lo = __double2loint(fma(rem, 16777216.0, kMagic));
  const bool fix = lo + 0x8080 >= (128 << 16);
  hi += fix ? 1 : 0;
  lo -= fix ? (1 << 24) : 0;
  uh = unsigned(hi + 0x808080);
  ul = unsigned(lo + 0x8080);
}
// Kernel entry v * c (|v * c| < 2^62, c = 2^(62 - e) a power of two, so the
// product is exact) -> X = round(v c) in one conversion (values >= 2^52 are
// already integers), biased by 0x80 in the seven low bytes: X + B returned as
// (low word, high word). Bytes 0..6 xor 0x80 are balanced digits, byte 7
// (arithmetic) the signed top digit.
__device__ __forceinline__ void split62(double v, double c, unsigned& xl, unsigned& xh) {
  const long long x = __double2ll_rn(v * c) + 0x0080808080808080ll;
  xl = unsigned(x);
  xh = unsigned(x >> 32);
}
// byte `i` of four words, packed a..d into bytes 0..3
__device__ __forceinline__ unsigned gather4(unsigned a, unsigned b, unsigned c, unsigned d, unsigned i) {
  const unsigned sel = i | ((i + 4) << 4);
  return __byte_perm(__byte_perm(a, b, sel), __byte_perm(c, d, sel), 0x5410);
}
// the 7 digit-plane words of 4 consecutive entries
__device__ __forceinline__ void pack_planes(const unsigned (&uh)[4], const unsigned (&ul)[4], unsigned (&w)[kPlanes]) {
  w[0] = gather4(uh[0], uh[1], uh[2], uh[3], 3);
  w[1] = gather4(uh[0], uh[1], uh[2], uh[3], 2) ^ 0x80808080u;
  w[2] = gather4(uh[0], uh[1], uh[2], uh[3], 1) ^ 0x80808080u;
  w[3] = gather4(uh[0], uh[1], uh[2], uh[3], 0) ^ 0x80808080u;
  w[4] = gather4(ul[0], ul[1], ul[2], ul[3], 2);
  w[5] = gather4(ul[0], ul[1], ul[2], ul[3], 1) ^ 0x80808080u;
  w[6] = gather4(ul[0], ul[1], ul[2], ul[3], 0) ^ 0x80808080u;
}

// the 8 kernel-entry digit-plane words of 4 consecutive entries (plane 0 =
// byte 7, most significant)
__device__ __forceinline__ void pack_planes8(const unsigned (&xl)[4], const unsigned (&xh)[4],
                                             unsigned (&w)[kPlanesA]) {
  w[0] = gather4(xh[0], xh[1], xh[2], xh[3], 3);
#pragma unroll
  for (int b = 2; b >= 0; --b) w[3 - b] = gather4(xh[0], xh[1], xh[2], xh[3], unsigned(b)) ^ 0x80808080u;
#pragma unroll
  for (int b = 3; b >= 0; --b) w[7 - b] = gather4(xl[0], xl[1], xl[2], xl[3], unsigned(b)) ^ 0x80808080u;
}

/// Bound on |K(x, y)| for y in a box with bounding box [lo, hi]: per row,
/// from the nearest and farthest corner distances.
template <int KIND>
__device__ __forceinline__ double kernel_bound(double dmin, double dmax, double param) {
  if (KIND == kOpLog) return fmax(fabs(log(dmin)), fabs(log(dmax)));
  if (KIND == kOpInvDist4Pi) return 0.07957747154594767 / dmin;
  return exp(-dmin / param);
}

// ------------------------------------------------------------ the kernel
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned mapa(unsigned addr, unsigned cta) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(std::uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(unsigned cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void st_cluster_v2(unsigned cluster_addr, unsigned a, unsigned b) {
  asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" ::"r"(cluster_addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void bulk_s2peer(unsigned dst_cluster, const void* src, unsigned bytes,
                                            unsigned bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(smem_addr(src)), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void umma_commit_both(std::uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_addr(bar)),
      "h"(std::uint16_t(3))
      : "memory");
}

// Cluster of two CTAs per K2 task: CTA h computes sample columns [h r, h r +
// r) (forward / adjoint) for all 128 rows, evaluates rows [64 h, 64 h + 64)
// of every kernel tile and stores their digit planes into both CTAs' shared
// memory, so each kernel entry is evaluated once.
template <int KIND, int DIM, int NP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
sample_apply_i8_kernel(DevOp op, const K2Task* __restrict__ tasks, const K2Row* __restrict__ rowtab,
                       const std::int64_t* __restrict__ pay_off, const std::int64_t* __restrict__ step_off,
                       const double* __restrict__ xstep, const std::int64_t* __restrict__ pb_off,
                       const int* __restrict__ pb_box, const double* __restrict__ box_bbox,
                       const unsigned char* __restrict__ bdig, std::int64_t half_stride, int r,
                       double* __restrict__ out, int dbg) {
  constexpr bool kTab = KIND == kOpLog;
  constexpr int kStages = kAStages;
  constexpr int kBS = bstages_for(NP, kTab);
  // A digit planes staged in TMEM (two buffers of 7 x 8 columns after the
  // 7 accumulator groups) where they fit the 512 columns
  constexpr bool kGS = group_split(NP);
  constexpr int kN = mma_n(NP);  // MMA N (and TMEM columns per accumulator group)
  constexpr int kAcol = kGroups * NP;
  constexpr bool kTS = !kGS && kAcol + 2 * kPlanesA * 8 <= 512 && kTSEnabled;
  constexpr int kBStep = b_step_bytes(kN);
  constexpr int kXStep = DIM * kStepK * 8;  // coordinates of one K-step (dim-major)
  constexpr unsigned kIdesc = umma_idesc(kN);
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sa = smem;                                   // [kStages][kPlanesA][kAPlane]
  unsigned char* sb = smem + kStages * kPlanesA * kAPlane;    // [kBS][kBStep]
  double* sx = reinterpret_cast<double*>(sb + kBS * kBStep);  // [kBS][DIM][32]
  double* lts = sx + kBS * DIM * kStepK;
  // full_a: the peer's half of the digit tile landed (1 expect_tx arrival + bytes);
  // done_a: this CTA's evaluation warps stored their half; full_b: payload
  // digits + coordinates; empty: both CTAs' MMAs of the stage completed
  __shared__ __align__(8) std::uint64_t full_a[kAStages], done_a[kAStages], empty[kAStages];
  __shared__ __align__(8) std::uint64_t full_b[8], empty_b[8];
  __shared__ __align__(8) std::uint64_t acc_full, acc_empty;
  __shared__ unsigned tmem_base;
  __shared__ double row_part[4][kRows][2];  // per (part, row): dmin^2, dmax^2
  __shared__ int row_exp[kRows];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = int(cluster_rank());
  const unsigned peer = unsigned(half ^ 1);
  const K2Task task = tasks[blockIdx.x >> 1];
  const std::int64_t p0 = pay_off[task.color], p1 = pay_off[task.color + 1];
  const int nsteps = int((p1 - p0 + kStepK - 1) / kStepK);
  const std::int64_t step0 = step_off[task.color];
  const unsigned char* bsrc = bdig + (kGS ? 0 : half * half_stride) + step0 * kBStep;
  // accumulator groups of this CTA (group split: the gs_groups(half) mask,
  // slot = rank of the group in the mask; column split: groups 0..6)
  const unsigned gmask = kGS ? gs_groups(half) : (1u << kGroups) - 1u;
  const double* xsrc = xstep + step0 * (DIM * kStepK);
  const double* tab = kTab ? lts : op.ltab;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&done_a[s], kEvalWarps);
      mbar_init(&empty[s], 2);
    }
    for (int s = 0; s < kBS; ++s) {
      mbar_init(&full_b[s], 1);
      mbar_init(&empty_b[s], 1);
    }
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, kEvalWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kEvalWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_addr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if constexpr (kTab) {
    for (int e = tid; e < 2 * kLogTab; e += kThreads) lts[e] = op.ltab[e];
  }
  // per-row scale: bound |K(x_i, y)| over the color's payload box bounding boxes
  if (warp < kEvalWarps) {
    const int row = tid & (kRows - 1), part = tid >> 7;  // 4 parts of the payload box list
    const int ipos = k2_row(task, rowtab, row < task.rows ? row : task.rows - 1).pos;
    double xi[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) xi[d] = op.x[d * op.n + ipos];
    double dmin2 = 1e300, dmax2 = 0.0;
    for (std::int64_t q = pb_off[task.color] + part; q < pb_off[task.color + 1]; q += 4) {
      const double* bb = box_bbox + std::int64_t(pb_box[q]) * 2 * DIM;
      double a2 = 0.0, b2 = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const double lo = bb[d], hi = bb[DIM + d];
        const double gap = fmax(fmax(lo - xi[d], xi[d] - hi), 0.0);
        const double far = fmax(fabs(xi[d] - lo), fabs(hi - xi[d]));
        a2 = fma(gap, gap, a2);
        b2 = fma(far, far, b2);
      }
      dmin2 = fmin(dmin2, a2);
      dmax2 = fmax(dmax2, b2);
    }
    row_part[part][row][0] = dmin2;
    row_part[part][row][1] = dmax2;
  }
  __syncthreads();
  if (tid < kRows) {
    const double dmin = sqrt(fmin(fmin(row_part[0][tid][0], row_part[1][tid][0]),
                                  fmin(row_part[2][tid][0], row_part[3][tid][0])));
    const double dmax = sqrt(fmax(fmax(row_part[0][tid][1], row_part[1][tid][1]),
                                  fmax(row_part[2][tid][1], row_part[3][tid][1])));
    const double bound = kernel_bound<KIND>(fmax(dmin, 1e-300), fmax(dmax, 1e-300), op.param);
    int e = 0;
    frexp(bound, &e);  // bound < 2^e
    row_exp[tid] = (bound > 0.0 && isfinite(bound)) ? max(min(e, 1000), -1000) : -1000;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  // the only 512-column allocation of an SM starts at lane 0, column 0, so
  // accumulator addresses are compile-time constants (no per-MMA uniform
  // register moves); checked
  constexpr unsigned tmem = 0;
  if (tmem_base != 0) __trap();

  if (warp == kEvalWarps) {
    // ------------------------------------------ B / coordinate loader + MMA issuer
    if (lane == 0 && nsteps > 0) {
      for (int step = 0; step < nsteps; ++step) {
        const int st = step % kStages;
        const unsigned ph = (step / kStages) & 1;
        const int bs = step % kBS;
        if (step > 0 && step % kWindow == 0) mbar_wait(&acc_empty, ((step / kWindow) - 1) & 1);
        mbar_wait(&full_b[bs], (step / kBS) & 1);
        mbar_wait(&done_a[st], ph);
        mbar_wait(&full_a[st], ph);
        tc_fence_after();
        const bool fresh = step % kWindow == 0;
        if (!(dbg & 1)) {
          // descriptors of plane 0 of this stage; planes are constant
          // offsets (16-byte units in the start-address field)
          const std::uint64_t ad0 = umma_desc(smem_addr(sa + st * kPlanesA * kAPlane));
          const std::uint64_t bd0 = umma_desc(smem_addr(sb + bs * kBStep));
          if constexpr (kTS) {
            // digit planes -> TMEM once per K-step (the MMAs then read A
            // from TMEM instead of re-reading each plane from shared memory
            // for every digit pair); tcgen05.cp and tcgen05.mma execute in
            // issue order, and the two A buffers alternate by step
            const unsigned abuf = tmem + unsigned(kAcol + (step & 1) * kPlanesA * 8);
#pragma unroll
            for (int a = 0; a < kPlanesA; ++a) tmem_cp_128x256b(abuf + unsigned(a * 8), ad0 + std::uint64_t((a * kAPlane) >> 4));
#pragma unroll
            for (int g = 0; g < kGroups; ++g) {
#pragma unroll
              for (int a = 0; a <= g; ++a) {
                umma_i8_ts(tmem + unsigned(g * NP), abuf + unsigned(a * 8),
                           bd0 + std::uint64_t(((g - a) * NP * kStepK) >> 4), kIdesc, (fresh && a == 0) ? 0u : 1u);
              }
            }
            if (dbg & 4) {  // probe: every MMA issued twice (results invalid)
#pragma unroll
              for (int g = 0; g < kGroups; ++g) {
#pragma unroll
                for (int a = 0; a <= g; ++a) {
                  umma_i8_ts(tmem + unsigned(g * NP), abuf + unsigned(a * 8),
                             bd0 + std::uint64_t(((g - a) * NP * kStepK) >> 4), kIdesc, 1u);
                }
              }
            }
          } else if constexpr (kGS) {
            // constant accumulator addresses per CTA half
            auto issue = [&](auto mask_c) {
              constexpr unsigned kMask = decltype(mask_c)::value;
#pragma unroll
              for (int g = 0; g < kGroupsGS; ++g) {
                if (!((kMask >> g) & 1u)) continue;
                const int slot = __popc(kMask & ((1u << g) - 1u));
                const int a0 = g > kPlanes - 1 ? g - (kPlanes - 1) : 0;    // payload plane g - a <= 6
                const int a1 = g < kPlanesA - 1 ? g : kPlanesA - 1;        // kernel plane a <= 7
#pragma unroll
                for (int a = a0; a <= a1; ++a) {
                  umma_i8(tmem + unsigned(slot * kN), ad0 + std::uint64_t((a * kAPlane) >> 4),
                          bd0 + std::uint64_t(((g - a) * kN * kStepK) >> 4), kIdesc, (fresh && a == a0) ? 0u : 1u);
                }
              }
            };
            if (half == 0)
              issue(std::integral_constant<unsigned, gs_groups(0)>{});
            else
              issue(std::integral_constant<unsigned, gs_groups(1)>{});
          } else {
#pragma unroll
            for (int g = 0; g < kGroups; ++g) {
#pragma unroll
              for (int a = 0; a <= g; ++a) {
                umma_i8(tmem + unsigned(g * kN), ad0 + std::uint64_t((a * kAPlane) >> 4),
                        bd0 + std::uint64_t(((g - a) * kN * kStepK) >> 4), kIdesc, (fresh && a == 0) ? 0u : 1u);
              }
            }
          }
        }
        umma_commit_both(&empty[st]);  // A stage st is free once both CTAs' MMAs are done
        umma_commit(&empty_b[bs]);     // B / coordinate stage (read by this CTA only)
        if ((step + 1) % kWindow == 0 || step + 1 == nsteps) umma_commit(&acc_full);
      }
    }
    __syncwarp();
  } else if (warp == kEvalWarps + 1) {
    // ------------------------------------------ peer copier: this CTA's 64 rows
    // of every digit plane into the peer's stage, completing its full_a
    if (lane == 0) {
      const unsigned sa_peer = mapa(smem_addr(sa), peer);
      for (int step = 0; step < nsteps; ++step) {
        const int st = step % kStages;
        const unsigned ph = (step / kStages) & 1;
        if (step >= kStages) mbar_wait(&full_a[st], ph ^ 1);  // previous round of this stage is complete
        mbar_expect_tx(&full_a[st], kPlanesA * kAPlane / 2);  // the peer's half, inbound
        mbar_wait(&done_a[st], ph);                           // our half is stored (and the peer's stage is free)
        const unsigned bar_peer = mapa(smem_addr(&full_a[st]), peer);
        const unsigned off = unsigned(st * kPlanesA * kAPlane + half * (kAPlane / 2));
#pragma unroll
        for (int a = 0; a < kPlanesA; ++a)
          bulk_s2peer(sa_peer + off + unsigned(a * kAPlane), sa + off + a * kAPlane, kAPlane / 2, bar_peer);
      }
    }
    __syncwarp();
  } else if (warp == kEvalWarps + 2) {
    // ------------------------------------------ loader: payload digits + coordinates,
    // as far ahead as the stages free up
    if (lane == 0) {
      for (int step = 0; step < nsteps; ++step) {
        const int bs = step % kBS;
        if (step >= kBS) mbar_wait(&empty_b[bs], ((step / kBS) - 1) & 1);
        mbar_expect_tx(&full_b[bs], kBStep + kXStep);
        bulk_g2s(sb + bs * kBStep, bsrc + std::int64_t(step) * kBStep, kBStep, &full_b[bs]);
        bulk_g2s(sx + bs * DIM * kStepK, xsrc + std::int64_t(step) * DIM * kStepK, kXStep, &full_b[bs]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------ evaluation + epilogue warps
    // evaluation: rows 64 half + 8 (warp & 7) + (lane & 7), payload rows
    // 16 (warp >> 3) + 4 ((lane >> 3) & 3) .. + 3 of each K-step: a warp
    // writes one whole 8 x 16-byte core matrix of every digit plane
    const int erow = 64 * half + 8 * (warp & 7) + (lane & 7);
    const int kh = warp >> 3, k4 = (lane >> 3) & 3;
    const int epos = k2_row(task, rowtab, erow < task.rows ? erow : task.rows - 1).pos;
    double xi[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) xi[d] = op.x[d * op.n + epos];
    const double cK = ldexp(1.0, 62 - row_exp[erow]);
    unsigned char* a_dst = sa + (erow >> 3) * 256 + kh * 128 + (erow & 7) * 16 + k4 * 4;
    // epilogue: TMEM lanes (warp & 3) * 32 + lane = tile rows, column quarter (warp >> 2)
    const int orow = (warp & 3) * 32 + lane;
    constexpr int kCq = kN / 4;  // columns per epilogue warp (multiple of 4)
    const int cq = warp >> 2;

    double y[kCq];
#pragma unroll
    for (int c = 0; c < kCq; ++c) y[c] = 0.0;
    for (int step = 0; step < nsteps; ++step) {
      const int st = step % kStages;
      const unsigned ph = (step / kStages) & 1;
      if (step >= kStages) mbar_wait(&empty[st], ph ^ 1);
      mbar_wait(&full_b[step % kBS], (step / kBS) & 1);  // coordinates of this step
      const double* xs = sx + (step % kBS) * DIM * kStepK + kh * 16 + k4 * 4;
      unsigned w[kPlanesA];
      {
        unsigned xl[4], xh[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double xj[DIM];
#pragma unroll
          for (int d = 0; d < DIM; ++d) xj[d] = xs[d * kStepK + u];
          const double v = (dbg & 2) ? xj[0] : kernel_value<KIND, DIM, false>(xi, xj, false, op.param, tab);
          split62(v, cK, xl[u], xh[u]);
        }
        pack_planes8(xl, xh, w);
      }
      unsigned char* dst = a_dst + st * kPlanesA * kAPlane;
#pragma unroll
      for (int a = 0; a < kPlanesA; ++a) *reinterpret_cast<unsigned*>(dst + a * kAPlane) = w[a];
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&done_a[st]);

      if ((step + 1) % kWindow == 0 || step + 1 == nsteps) {
        // drain this CTA's int32 groups of the window into FP64
        const int win = step / kWindow;
        mbar_wait(&acc_full, win & 1);
        tc_fence_after();
        const int e = row_exp[orow];
        const unsigned lane_base = tmem + (unsigned((warp & 3) * 32) << 16) + unsigned(cq * kCq);
#pragma unroll
        for (int q = 0; q < kGroupsGS; ++q) {
          if (!((gmask >> q) & 1u)) continue;
          const int slot = __popc(gmask & ((1u << q) - 1u));
          const double wg = ldexp(1.0, e - 8 - 8 * q);
#pragma unroll
          for (int c0 = 0; c0 < kCq; c0 += 4) {
            int v[4];
            tmem_ld4(lane_base + unsigned(slot * kN + c0), v);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 4; ++c) y[c0 + c] = fma(double(v[c]), wg, y[c0 + c]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty);
      }
    }
    if (orow < task.rows) {
      const K2Row dst = k2_row(task, rowtab, orow);
#pragma unroll
      for (int c = 0; c < kCq; ++c) {
        const int col = cq * kCq + c;
        if constexpr (kGS) {
          // both CTAs add their groups' partial sums into the zeroed sample
          // block: two addends per element, so the result is order-independent
          const int hh = col / NP, cc = col - hh * NP;
          if (cc < r) atomicAdd(out + dst.out + std::int64_t(hh * r + cc) * dst.ld, y[c]);
        } else {
          if (col < r) out[dst.out + std::int64_t(half * r + col) * dst.ld] = y[c];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still write into it
  tc_fence_after();
  if (warp == kEvalWarps) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, int DIM, int NP>
void launch_i8(const DevOp& op, const K2Task* tasks, const K2Row* rowtab, int ntasks, const std::int64_t* pay_off,
               const std::int64_t* step_off, const double* xstep, const std::int64_t* pb_off,
               const int* pb_box, const double* box_bbox, const unsigned char* bdig, std::int64_t half_stride,
               int r, double* out, cudaStream_t s) {
  constexpr size_t smem = smem_bytes(NP, KIND == kOpLog);
  auto* fn = sample_apply_i8_kernel<KIND, DIM, NP>;
  HP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  fn<<<2 * ntasks, kThreads, smem, s>>>(op, tasks, rowtab, pay_off, step_off, xstep, pb_off, pb_box, box_bbox,
                                        bdig, half_stride, r, out, k2_int8_debug());
}

#define HP_K2I8_ARGS                                                                                  \
  const DevOp &op, const K2Task *tasks, const K2Row *rowtab, int ntasks, const std::int64_t *pay_off, \
      const std::int64_t *step_off, const double *xstep, const std::int64_t *pb_off,                   \
      const int *pb_box, const double *box_bbox, const unsigned char *bdig, std::int64_t half_stride, \
      int r, double *out, cudaStream_t s

template <int KIND>
void launch_kind(HP_K2I8_ARGS) {
  const int np = (r + 15) / 16 * 16;
#define HP_K2I8_NP(D, N) \
  if (op.dim == D && np == N) return launch_i8<KIND, D, N>(op, tasks, rowtab, ntasks, pay_off, step_off, xstep, pb_off, pb_box, box_bbox, bdig, half_stride, r, out, s);
#define HP_K2I8_D(D) HP_K2I8_NP(D, 16) HP_K2I8_NP(D, 32) HP_K2I8_NP(D, 48) HP_K2I8_NP(D, 64)
  HP_K2I8_D(1) HP_K2I8_D(2) HP_K2I8_D(3)
#undef HP_K2I8_D
#undef HP_K2I8_NP
  throw std::invalid_argument("k2 int8: unsupported dim / width");
}

/// Payload digit planes of one level for every color's K-steps (step_off,
/// step_color). Group split (group_split(np)): one N = 2 np tile per plane,
/// rows [0, np) forward and [np, 2 np) adjoint columns, at bdig[gstep *
/// b_step_bytes(2 np)]; otherwise per column half at bdig[half * half_stride
/// + gstep * b_step_bytes(np)] (np = padded_width(r)).
void launch_payload_digits(const double* gc, int gld, int r, const std::int64_t* pay_off,
                           const std::int64_t* step_off, const int* step_color, std::int64_t tsteps,
                           unsigned char* bdig, std::int64_t half_stride, cudaStream_t s);
/// Step-ordered payload coordinates: xstep[gstep][d][32] (dim-major per
/// K-step), rows past a color's payload padded with far-away points.
void launch_step_coords(const double* xc, std::int64_t nnz, int dim, const std::int64_t* pay_off,
                        const std::int64_t* step_off, const int* step_color, std::int64_t tsteps,
                        double* xstep, cudaStream_t s);
/// Raw-coordinate bounding box of every box (tree-order contiguous ranges).
void launch_box_bbox(const double* x, std::int64_t n, int dim, const std::int64_t* start,
                     const std::int64_t* count, int nboxes, double* bbox, cudaStream_t s);
/// The apply itself: 2 CTAs (forward / adjoint columns) per K2Task.
void launch_sample_apply_i8(HP_K2I8_ARGS);

void launch_log(HP_K2I8_ARGS);
void launch_invdist(HP_K2I8_ARGS);
void launch_exp(HP_K2I8_ARGS);

}  // namespace k2i8
}  // namespace hpeel
