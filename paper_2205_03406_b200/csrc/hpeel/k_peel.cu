// K3 peeling subtraction (sm_100a): the level-truncated H1 apply
// A^(l-1) Omega_c of H1Rep::apply_truncated(_adjoint)
// (proj/src/hmatrix.cpp:86-116), restricted to the sample rows the driver
// reads and to the nonzero rows of Omega_c.
//
// For a coarse pair q = (x, y) and a color c the reference computes
// U_q (B_q (V_q^T Omega_c(I_y))) for every color over all N rows. Here
// coefficient tasks form T_{q,c} = B_q * sum_{v in P_c, v in y} V_q[v]^T G_v
// once (k x r), and apply tasks subtract U_q[rows of a] T_{q,c} from each
// level-l sample block whose box a lies under x. Both contractions run on
// FP64 DMMA (m8n8k4) with shared-memory operand tiles in conflict-free
// strides (== 4 mod 16 doubles) and cp.async double buffering.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"

namespace hpeel {

namespace {

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__host__ __device__ constexpr int stride4(int n) { return ((n + 11) / 16) * 16 + 4; }

constexpr int kThreads = 128;       // coefficient kernel
constexpr int kApplyThreads = 256;  // apply: 4 row groups x 2 column halves
constexpr int kRows = 64;  // apply tile rows (4 warps x 16)
constexpr int kFS = kRows + 4;

// ------------------------------------------------------------------ apply
// out[rows, c0 + c] += alpha * sum_terms F[rows, :k] T[:k, c0 + c]
// Staged in units of (term, 32-wide slice of k): F slice column-major (ld
// kFS), T slice column-major (ld stride4(32)), double-buffered -- 80 KB at
// w = 80, so two CTAs (16 warps) share an SM. Eight warps: warp & 3 picks the
// 16-row group, warp >> 2 the half of the NT column tiles. (Whole-k stages
// took ~150 KB at k = 64, w = 80: one CTA of four warps per SM left the DMMA
// pipe mostly idle, ncu: 6% occupancy, 90% of cycles without an eligible warp.)
constexpr int kKC = 32;
template <int NT>
__global__ void __launch_bounds__(kApplyThreads)
peel_apply_kernel(const PeelTask* __restrict__ tasks, const PeelRef* __restrict__ refs,
                  const PeelTerm* __restrict__ terms, const double* __restrict__ factors,
                  const double* __restrict__ tbuf, int k, int w, double* __restrict__ out, int ocol0,
                  double alpha) {
  extern __shared__ __align__(16) double sm[];
  constexpr int ts = stride4(kKC);
  constexpr int fsz = kKC * kFS, tsz = NT * 8 * ts;
  const int kp = (k + 3) & ~3;
  const int nkc = (kp + kKC - 1) / kKC;
  auto fs = [&](int b) { return sm + b * (fsz + tsz); };
  auto tsm = [&](int b) { return sm + b * (fsz + tsz) + fsz; };
  const PeelTask task = tasks[blockIdx.x];
  const int c0 = blockIdx.y * NT * 8;
  const int ncol = min(NT * 8, min(task.cols, w) - c0);
  if (ncol <= 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rg = warp & 3;                  // 16-row group
  constexpr int NH = (NT + 1) / 2;          // column tiles per half
  const int t0 = (warp >> 2) * NH;          // first column tile of this warp
  for (int e = tid; e < 2 * (fsz + tsz); e += kApplyThreads) sm[e] = 0.0;
  __syncthreads();

  // slice kc of term q: columns / rows [kc * 32, kc * 32 + 32) of F / T; the
  // padding k .. kp (k % 4 != 0) is stored as zeros
  auto issue = [&](int buf, int q, std::int64_t roff, int kc) {
    const PeelTerm term = terms[q];
    const int l0 = kc * kKC;
    const int lend = min(kp, l0 + kKC) - l0;
    const double* f0 = factors + term.f + roff;
    for (int e = tid; e < kRows * lend; e += kApplyThreads) {
      const int i = e % kRows, l = e / kRows;
      if (i < task.rows) {
        if (l0 + l < k)
          cp_async8(fs(buf) + l * kFS + i, f0 + i + std::int64_t(l0 + l) * term.fld);
        else
          fs(buf)[l * kFS + i] = 0.0;
      }
    }
    // one warp per T column, lanes along the slice (coalesced, no runtime division)
    for (int c = warp; c < ncol; c += kApplyThreads / 32)
      if (lane < lend) {
        if (l0 + lane < k)
          cp_async8(tsm(buf) + c * ts + lane, tbuf + term.t + l0 + lane + std::int64_t(c0 + c) * k);
        else
          tsm(buf)[c * ts + lane] = 0.0;
      }
    cp_async_commit();
  };

  double acc[2][NH][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < NH; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;

  // cursor over (ref, term, slice): the unit after (ri, q, kc)
  auto next = [&](int& ri, int& q, int& kc) {
    if (++kc < nkc) return;
    kc = 0;
    ++q;
    while (ri < task.ref_end && q >= refs[ri].term_end) {
      ++ri;
      if (ri < task.ref_end) q = refs[ri].term_begin;
    }
  };
  int ri = task.ref_begin, q = ri < task.ref_end ? refs[ri].term_begin - 1 : 0, kc = nkc - 1;
  next(ri, q, kc);
  if (ri < task.ref_end) issue(0, q, refs[ri].roff, kc);
  int buf = 0;
  for (; ri < task.ref_end; buf ^= 1) {
    int nri = ri, nq = q, nkc_ = kc;
    next(nri, nq, nkc_);
    cp_async_wait_all();
    __syncthreads();
    if (nri < task.ref_end) issue(buf ^ 1, nq, refs[nri].roff, nkc_);
    const int kn = min(kKC, kp - kc * kKC);
    const double* a0p = fs(buf) + (lane & 3) * kFS + rg * 16 + (lane >> 2);
    const double* bp = tsm(buf) + (t0 * 8 + (lane >> 2)) * ts + (lane & 3);
    for (int kk = 0; kk < kn; kk += 4) {
      const double a0 = a0p[kk * kFS], a1 = a0p[kk * kFS + 8];
#pragma unroll
      for (int nt = 0; nt < NH; ++nt) {
        if (t0 + nt >= NT) break;  // odd NT: the second half has one tile less
        const double b = bp[nt * 8 * ts + kk];
        dmma8x8x4(acc[0][nt][0], acc[0][nt][1], a0, b);
        dmma8x8x4(acc[1][nt][0], acc[1][nt][1], a1, b);
      }
    }
    ri = nri;
    q = nq;
    kc = nkc_;
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int rr = rg * 16 + m * 8 + (lane >> 2);
    if (rr >= task.rows) continue;
#pragma unroll
    for (int nt = 0; nt < NH; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = (t0 + nt) * 8 + (lane & 3) * 2 + h;
        if (c < ncol) out[task.out + rr + std::int64_t(ocol0 + c0 + c) * task.ld] += alpha * acc[m][nt][h];
      }
  }
}

// T (k x w, col-major, ld k) = op(B) M from shared B (k x k) and M (k x w),
// both with leading dimension ms_ld. With k % 4 == 0 on DMMA: 8 x 8 output
// tiles over the warps (rows >= k / columns >= w of a tile read stale shared
// memory -- callers allocate 8 spare rows -- and are not stored); otherwise
// one scalar FMA chain per output.
__device__ __forceinline__ void coeff_epilogue(const double* bs, const double* ms, int ms_ld, int k, int w,
                                               bool btrans, double* __restrict__ t_out, int nthreads) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if ((k & 3) == 0) {
    const int mt = (k + 7) / 8, ntl = (w + 7) / 8;
    for (int tt = warp; tt < mt * ntl; tt += nthreads / 32) {
      const int mtile = tt / ntl, nt = tt - mtile * ntl;
      const int am = mtile * 8 + (lane >> 2), bn = nt * 8 + (lane >> 2);
      double c0 = 0.0, c1 = 0.0;
      for (int kk = 0; kk < k; kk += 4) {
        const int l = kk + (lane & 3);
        const double a = btrans ? bs[l + am * ms_ld] : bs[am + l * ms_ld];
        dmma8x8x4(c0, c1, a, ms[l + bn * ms_ld]);
      }
      const int c = nt * 8 + (lane & 3) * 2;
      if (am < k) {
        if (c < w) t_out[am + std::int64_t(c) * k] = c0;
        if (c + 1 < w) t_out[am + std::int64_t(c + 1) * k] = c1;
      }
    }
  } else {
    for (int e = tid; e < k * w; e += nthreads) {
      const int i = e % k, c = e / k;
      double t = 0.0;
      if (btrans) {
        for (int l = 0; l < k; ++l) t = fma(bs[l + i * ms_ld], ms[l + c * ms_ld], t);
      } else {
        for (int l = 0; l < k; ++l) t = fma(bs[i + l * ms_ld], ms[l + c * ms_ld], t);
      }
      t_out[e] = t;
    }
  }
}

// ------------------------------------------------------------------ coeff
// Gaussian payloads: M (k x w) = sum_v F[v rows]^T G[v rows, gcol0 : gcol0 + w]
// on DMMA (A = F^T staged [m][t], B = G staged [t][c]), then T = op(B) M.
constexpr int kCK = 32;  // payload rows per stage

template <int NT>
__global__ void __launch_bounds__(kThreads)
peel_coeff_dmma_kernel(const CoeffTask* __restrict__ tasks, const double* __restrict__ factors,
                       const double* __restrict__ bmat, const std::int64_t* __restrict__ seg_start,
                       const std::int64_t* __restrict__ seg_count, const double* __restrict__ g,
                       int gld, int gcol0, int k, int w, double* __restrict__ tbuf) {
  extern __shared__ __align__(16) double sm[];
  constexpr int S = stride4(NT * 8);
  constexpr int FS = stride4(kCK);  // F^T rows (one per factor column m), kCK payload rows each
  const int mt = (k + 7) / 8;       // m-tiles (<= 8)
  auto fs = [&](int b) { return sm + b * mt * 8 * FS; };
  auto gs = [&](int b) { return sm + 2 * mt * 8 * FS + b * kCK * S; };
  // after the loop, aliasing the drained stages: M (k x w, ld MS) and B (k x k, ld MS)
  const int MS = stride4(k);
  double* ms = sm;
  double* bs = ms + MS * w;
  const CoeffTask task = tasks[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 2 * (mt * 8 * FS + kCK * S); e += kThreads) sm[e] = 0.0;
  __syncthreads();

  auto issue = [&](int buf, int sg, std::int64_t r0) {
    const std::int64_t left = seg_count[sg] - r0;
    const int cnt = left < kCK ? int(left) : kCK;
    const std::int64_t frow = seg_start[sg] - task.f_row0 + r0;
    const std::int64_t gpos = seg_start[sg] + r0;
    // F: one warp per factor column, lanes along the (<= 32) payload rows;
    // G: one warp per payload row, lanes along its columns (no runtime division)
    static_assert(kCK == 32, "one lane per payload row");
    if (lane < cnt)
      for (int m = warp; m < k; m += kThreads / 32)
        cp_async8(fs(buf) + m * FS + lane, factors + task.f + frow + lane + std::int64_t(m) * task.frows);
    for (int t = warp; t < cnt; t += kThreads / 32)
      for (int c = lane; c < w; c += 32) cp_async8(gs(buf) + t * S + c, g + (gpos + t) * gld + gcol0 + c);
    cp_async_commit();
    return cnt;
  };

  double acc[2][NT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;

  int sg = task.seg_begin;
  std::int64_t r0 = 0;
  int buf = 0;
  int cnt_cur = 0;
  if (sg < task.seg_end) cnt_cur = issue(0, sg, 0);
  while (sg < task.seg_end) {
    int nsg = sg;
    std::int64_t nr0 = r0 + kCK;
    if (nr0 >= seg_count[nsg]) {
      ++nsg;
      nr0 = 0;
    }
    cp_async_wait_all();
    __syncthreads();
    int cnt_next = 0;
    if (nsg < task.seg_end) cnt_next = issue(buf ^ 1, nsg, nr0);
    // rows past the chunk end hold stale rows of earlier chunks: zero G there
    if (cnt_cur < kCK) {
      for (int e = tid; e < (kCK - cnt_cur) * S; e += kThreads) gs(buf)[cnt_cur * S + e] = 0.0;
      __syncthreads();
    }
#pragma unroll
    for (int mm = 0; mm < 2; ++mm) {
      const int mtile = warp + 4 * mm;
      if (mtile >= mt) continue;
      const double* ap = fs(buf) + (mtile * 8 + (lane >> 2)) * FS + (lane & 3);
      const double* bp = gs(buf) + (lane & 3) * S + (lane >> 2);
#pragma unroll
      for (int kk = 0; kk < kCK; kk += 4) {
        const double a = ap[kk];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma8x8x4(acc[mm][nt][0], acc[mm][nt][1], a, bp[kk * S + nt * 8]);
      }
    }
    sg = nsg;
    r0 = nr0;
    cnt_cur = cnt_next;
    buf ^= 1;
  }
  __syncthreads();
  // M -> shared (col-major k x w), B -> shared
#pragma unroll
  for (int mm = 0; mm < 2; ++mm) {
    const int mtile = warp + 4 * mm;
    if (mtile >= mt) continue;
    const int m = mtile * 8 + (lane >> 2);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = nt * 8 + (lane & 3) * 2 + h;
        if (m < k && c < w) ms[m + c * MS] = acc[mm][nt][h];
      }
  }
  for (int l = warp; l < k; l += kThreads / 32)
    for (int i = lane; i < k; i += 32) bs[i + l * MS] = bmat[task.b + i + l * k];
  __syncthreads();
  coeff_epilogue(bs, ms, MS, k, w, task.btrans, tbuf + task.t_out, kThreads);
}

// Identity payloads [I | 0] (leaf phase): M[:, t] = sum_v F[row v_t, :]^T for
// t < |v|, a gather; then T = op(B) M.
__global__ void __launch_bounds__(256)
peel_coeff_identity_kernel(const CoeffTask* __restrict__ tasks, const double* __restrict__ factors,
                           const double* __restrict__ bmat, const std::int64_t* __restrict__ seg_start,
                           const std::int64_t* __restrict__ seg_count, int k, int w,
                           double* __restrict__ tbuf) {
  extern __shared__ __align__(16) double sm[];
  const int MS = stride4(k);
  double* ms = sm;
  double* bs = sm + MS * w;
  const CoeffTask task = tasks[blockIdx.x];
  const double* f = factors + task.f;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // M[i, c] = sum over segments of F[row c of the segment, i]: one warp per
  // factor column i, lanes along c (coalesced rows of the column-major F)
  for (int i = warp; i < k; i += nw)
    for (int c = lane; c < w; c += 32) {
      double acc = 0.0;
      for (int sg = task.seg_begin; sg < task.seg_end; ++sg)
        if (c < seg_count[sg]) acc += f[seg_start[sg] - task.f_row0 + c + std::int64_t(i) * task.frows];
      ms[i + c * MS] = acc;
    }
  for (int l = warp; l < k; l += nw)
    for (int i = lane; i < k; i += 32) bs[i + l * MS] = bmat[task.b + i + l * k];
  __syncthreads();
  coeff_epilogue(bs, ms, MS, k, w, task.btrans, tbuf + task.t_out, blockDim.x);
}

template <int NT>
void coeff_nt(const CoeffTask* tasks, int ntasks, const double* factors, const double* bmat,
              const std::int64_t* ss, const std::int64_t* sc, const double* g, int gld, int gcol0,
              int k, int w, double* tbuf, cudaStream_t s) {
  constexpr int S = stride4(NT * 8);
  constexpr int FS = stride4(kCK);
  const int mt = (k + 7) / 8;
  // the epilogue's M and B reuse the pipeline stages (80 KB instead of 154 KB
  // at k = 64, w = 80: two CTAs per SM)
  const size_t smem = size_t(std::max(2 * mt * 8 * FS + 2 * kCK * S, stride4(k) * (w + k + 8))) * sizeof(double);  // + 8: rows >= k of a DMMA tile
  HP_CUDA(cudaFuncSetAttribute(peel_coeff_dmma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  peel_coeff_dmma_kernel<NT><<<ntasks, kThreads, smem, s>>>(tasks, factors, bmat, ss, sc, g, gld, gcol0, k, w, tbuf);
  HP_LAUNCHED();
}

template <int NT>
void apply_nt(const PeelTask* tasks, int ntasks, const PeelRef* refs, const PeelTerm* terms,
              const double* factors, const double* tbuf, int k, int w, double* out, int ocol0, double alpha,
              cudaStream_t s) {
  const size_t smem = size_t(2 * (kKC * kFS + NT * 8 * stride4(kKC))) * sizeof(double);
  HP_CUDA(cudaFuncSetAttribute(peel_apply_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const dim3 grid(unsigned(ntasks), unsigned((w + NT * 8 - 1) / (NT * 8)));
  peel_apply_kernel<NT><<<grid, kApplyThreads, smem, s>>>(tasks, refs, terms, factors, tbuf, k, w, out, ocol0, alpha);
  HP_LAUNCHED();
}

}  // namespace

void launch_peel_coeff(const CoeffTask* tasks, int ntasks, const double* factors,
                       const double* bmat, const std::int64_t* seg_start,
                       const std::int64_t* seg_count, const double* g, int gld, int gcol0, int k,
                       int w, double* tbuf, cudaStream_t s) {
  if (ntasks == 0) return;
  if (k > 64) throw std::invalid_argument("peel: rank k > 64 is not supported");
  if (gcol0 < 0) {
    const size_t smem = size_t(stride4(k) * (w + k + 8)) * sizeof(double);  // + 8: rows >= k of a DMMA tile
    HP_CUDA(cudaFuncSetAttribute(peel_coeff_identity_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    peel_coeff_identity_kernel<<<ntasks, 256, smem, s>>>(tasks, factors, bmat, seg_start, seg_count, k, w, tbuf);
    HP_LAUNCHED();
    return;
  }
  const int nt = (w + 7) / 8;
#define HP_C(N) \
  case N: return coeff_nt<N>(tasks, ntasks, factors, bmat, seg_start, seg_count, g, gld, gcol0, k, w, tbuf, s);
  switch (nt) {
    HP_C(1) HP_C(2) HP_C(3) HP_C(4) HP_C(5) HP_C(6) HP_C(7) HP_C(8) HP_C(9) HP_C(10)
    default: throw std::invalid_argument("peel coefficient width > 80 is not supported");
  }
#undef HP_C
}

void launch_peel_apply(const PeelTask* tasks, int ntasks, const PeelRef* refs, const PeelTerm* terms,
                       const double* factors, const double* tbuf, int k, int w, double* out,
                       int ocol0, double alpha, cudaStream_t s) {
  if (ntasks == 0) return;
  if (k > 64) throw std::invalid_argument("peel: rank k > 64 is not supported");
  const int nt = (w + 7) / 8;
#define HP_A(N) \
  case N: return apply_nt<N>(tasks, ntasks, refs, terms, factors, tbuf, k, w, out, ocol0, alpha, s);
  switch (nt) {
    HP_A(1) HP_A(2) HP_A(3) HP_A(4) HP_A(5) HP_A(6) HP_A(7) HP_A(8) HP_A(9) HP_A(10)
    default: return apply_nt<8>(tasks, ntasks, refs, terms, factors, tbuf, k, w, out, ocol0, alpha, s);
  }
#undef HP_A
}

}  // namespace hpeel
