// K2 on the INT8 tensor cores: payload digit planes, box bounding boxes and
// the launch dispatch (kernel template in k2_i8.cuh; per-kind instantiation
// units k2i8_<kind>.cu).
#include "k2_i8.cuh"

#include <stdexcept>

namespace hpeel {
namespace k2i8 {
namespace {

// One thread per (half, K-step, payload column n < np, K-half): 16 payload
// rows of one column -> 7 digit planes in the UMMA K-major no-swizzle layout.
__global__ void payload_digits_kernel(const double* __restrict__ gc, int gld, int r, int np,
                                      const std::int64_t* __restrict__ pay_off,
                                      const std::int64_t* __restrict__ step_off,
                                      const int* __restrict__ step_color, std::int64_t tsteps,
                                      unsigned char* __restrict__ bdig, std::int64_t half_stride) {
  const std::int64_t t = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const std::int64_t per_half = tsteps * np * 2;
  if (t >= 2 * per_half) return;
  const int half = int(t / per_half);
  std::int64_t u = t - half * per_half;
  const std::int64_t gstep = u / (np * 2);
  u -= gstep * np * 2;
  const int n = int(u >> 1), kh = int(u & 1);
  const int color = step_color[gstep];
  const std::int64_t k0 = pay_off[color] + (gstep - step_off[color]) * kStepK + kh * 16;
  const std::int64_t p1 = pay_off[color + 1];
  const int col = half * r + n;
  const double c = 67108864.0;  // 2^30 / 16
  unsigned w[4][kPlanes];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned uh[4], ul[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const std::int64_t k = k0 + q * 4 + e;
      const double v = (k < p1 && n < r) ? gc[k * gld + col] : 0.0;
      split_digits(v, c, uh[e], ul[e]);
    }
    pack_planes(uh, ul, w[q]);
  }
  unsigned char* dst;
  std::int64_t plane;
  if (group_split(np)) {  // [gstep][plane][2 np rows]: row half * np + n
    const int n2 = half * np + n;
    dst = bdig + gstep * b_step_bytes(2 * np) + (n2 >> 3) * 256 + kh * 128 + (n2 & 7) * 16;
    plane = std::int64_t(2) * np * kStepK;
  } else {
    dst = bdig + half * half_stride + gstep * b_step_bytes(np) + (n >> 3) * 256 + kh * 128 + (n & 7) * 16;
    plane = std::int64_t(np) * kStepK;
  }
#pragma unroll
  for (int a = 0; a < kPlanes; ++a)
    *reinterpret_cast<uint4*>(dst + std::int64_t(a) * plane) = make_uint4(w[0][a], w[1][a], w[2][a], w[3][a]);
}

__global__ void step_coords_kernel(const double* __restrict__ xc, std::int64_t nnz, int dim,
                                   const std::int64_t* __restrict__ pay_off, const std::int64_t* __restrict__ step_off,
                                   const int* __restrict__ step_color, std::int64_t tsteps, double* __restrict__ xstep) {
  const std::int64_t t = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= tsteps * kStepK) return;
  const std::int64_t gstep = t / kStepK;
  const int j = int(t - gstep * kStepK);
  const int color = step_color[gstep];
  const std::int64_t k = pay_off[color] + (gstep - step_off[color]) * kStepK + j;
  const bool in = k < pay_off[color + 1];
  for (int d = 0; d < dim; ++d) xstep[(gstep * dim + d) * kStepK + j] = in ? xc[d * nnz + k] : 1e150;
}

// One warp per box: bounding box of its points (tree order, dim x n SoA),
// stored [lo_0 .. lo_{dim-1}, hi_0 .. hi_{dim-1}].
__global__ void box_bbox_kernel(const double* __restrict__ x, std::int64_t n, int dim,
                                const std::int64_t* __restrict__ start, const std::int64_t* __restrict__ count,
                                int nboxes, double* __restrict__ bbox) {
  const int box = int((std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (box >= nboxes) return;
  for (int d = 0; d < dim; ++d) {
    double lo = 1e308, hi = -1e308;
    for (std::int64_t i = lane; i < count[box]; i += 32) {
      const double v = x[d * n + start[box] + i];
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      bbox[std::int64_t(box) * 2 * dim + d] = lo;
      bbox[std::int64_t(box) * 2 * dim + dim + d] = hi;
    }
  }
}

}  // namespace

void launch_payload_digits(const double* gc, int gld, int r, const std::int64_t* pay_off,
                           const std::int64_t* step_off, const int* step_color, std::int64_t tsteps,
                           unsigned char* bdig, std::int64_t half_stride, cudaStream_t s) {
  const int np = padded_width(r);
  const std::int64_t threads = 2 * tsteps * np * 2;
  if (threads == 0) return;
  payload_digits_kernel<<<cdiv(threads, 256), 256, 0, s>>>(gc, gld, r, np, pay_off, step_off, step_color, tsteps,
                                                            bdig, half_stride);
  HP_LAUNCHED();
}

void launch_step_coords(const double* xc, std::int64_t nnz, int dim, const std::int64_t* pay_off,
                        const std::int64_t* step_off, const int* step_color, std::int64_t tsteps,
                        double* xstep, cudaStream_t s) {
  if (tsteps == 0) return;
  step_coords_kernel<<<cdiv(tsteps * kStepK, 256), 256, 0, s>>>(xc, nnz, dim, pay_off, step_off, step_color, tsteps,
                                                                 xstep);
  HP_LAUNCHED();
}

void launch_box_bbox(const double* x, std::int64_t n, int dim, const std::int64_t* start,
                     const std::int64_t* count, int nboxes, double* bbox, cudaStream_t s) {
  if (nboxes == 0) return;
  box_bbox_kernel<<<cdiv(std::int64_t(nboxes) * 32, 256), 256, 0, s>>>(x, n, dim, start, count, nboxes, bbox);
  HP_LAUNCHED();
}

void launch_sample_apply_i8(HP_K2I8_ARGS) {
  if (ntasks == 0) return;
  switch (op.kind) {
    case kOpLog: launch_log(op, tasks, rowtab, ntasks, pay_off, step_off, xstep, pb_off, pb_box, box_bbox, bdig, half_stride, r, out, s); break;
    case kOpInvDist4Pi: launch_invdist(op, tasks, rowtab, ntasks, pay_off, step_off, xstep, pb_off, pb_box, box_bbox, bdig, half_stride, r, out, s); break;
    case kOpExp: launch_exp(op, tasks, rowtab, ntasks, pay_off, step_off, xstep, pb_off, pb_box, box_bbox, bdig, half_stride, r, out, s); break;
    default: throw std::invalid_argument("k2 int8: dense operators use the FP64 path");
  }
  HP_LAUNCHED();
}

}  // namespace k2i8
}  // namespace hpeel
