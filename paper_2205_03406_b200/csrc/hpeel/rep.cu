// Device-resident black boxes, the H1 representation's device apply and
// host export, the power-method verifier, and parity probes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <stdexcept>

#include "engine.cuh"
#include "rng.hpp"

namespace hpeel {

using namespace detail;

// ---------------------------------------------------------------- operator

std::shared_ptr<DeviceOperator> DeviceOperator::dense(const Matrix& a, int device) {
  if (a.rows() != a.cols()) throw std::invalid_argument("dense operator must be square");
  DeviceGuard g(device);
  std::shared_ptr<DeviceOperator> op(new DeviceOperator());
  op->kind_ = kOpDense;
  op->n_ = a.rows();
  op->device_ = device;
  bool sym = true;
  for (Index j = 0; j < a.cols() && sym; ++j)
    for (Index i = j + 1; i < a.rows(); ++i)
      if (a(i, j) != a(j, i)) {
        sym = false;
        break;
      }
  op->symmetric_ = sym;
  HP_CUDA(cudaMalloc(&op->d_a_, size_t(a.size()) * sizeof(double)));
  HP_CUDA(cudaMemcpy(op->d_a_, a.data(), size_t(a.size()) * sizeof(double), cudaMemcpyHostToDevice));
  return op;
}

std::shared_ptr<DeviceOperator> DeviceOperator::kernel(int kind, const Matrix& pts, double param,
                                                       int device) {
  if (kind != kOpLog && kind != kOpInvDist4Pi && kind != kOpExp)
    throw std::invalid_argument("unknown kernel operator kind");
  if (pts.cols() < 1 || pts.cols() > 3) throw std::invalid_argument("kernel operators need 1..3 dims");
  if (pts.rows() < 1) throw std::invalid_argument("empty point set");
  if (kind == kOpExp && !(param > 0.0)) throw std::invalid_argument("length scale must be > 0");
  DeviceGuard g(device);
  std::shared_ptr<DeviceOperator> op(new DeviceOperator());
  op->kind_ = kind;
  op->dim_ = int(pts.cols());
  op->n_ = pts.rows();
  op->param_ = param;
  op->device_ = device;
  // col-major n x d is exactly SoA dim x n
  HP_CUDA(cudaMalloc(&op->d_x_, size_t(pts.size()) * sizeof(double)));
  HP_CUDA(cudaMemcpy(op->d_x_, pts.data(), size_t(pts.size()) * sizeof(double), cudaMemcpyHostToDevice));
  return op;
}

std::shared_ptr<DeviceOperator> DeviceOperator::callback(Index n, bool symmetric, bool device_pointers,
                                                         ApplyFn fn, void* ctx, int device) {
  if (n < 1) throw std::invalid_argument("callback operator needs n >= 1");
  if (!fn) throw std::invalid_argument("callback operator needs an apply function");
  DeviceGuard g(device);
  std::shared_ptr<DeviceOperator> op(new DeviceOperator());
  op->kind_ = kOpCallback;
  op->n_ = n;
  op->symmetric_ = symmetric;
  op->device_ = device;
  op->fn_ = fn;
  op->ctx_ = ctx;
  op->device_pointers_ = device_pointers;
  return op;
}

void DeviceOperator::call(bool adjoint, const double* d_x, std::int64_t w, double* d_y, cudaStream_t s) const {
  if (!fn_) throw std::logic_error("not a callback operator");
  int rc = 0;
  if (device_pointers_) {
    rc = fn_(ctx_, adjoint ? 1 : 0, d_x, w, d_y, s);
  } else {
    // the reference's call: host matrices in, host matrix out
    const size_t bytes = size_t(n_) * size_t(w) * sizeof(double);
    double* hx = static_cast<double*>(detail::persistent_pinned(bytes, 2));
    double* hy = static_cast<double*>(detail::persistent_pinned(bytes, 3));
    HP_CUDA(cudaMemcpyAsync(hx, d_x, bytes, cudaMemcpyDeviceToHost, s));
    HP_CUDA(cudaStreamSynchronize(s));
    rc = fn_(ctx_, adjoint ? 1 : 0, hx, w, hy, nullptr);
    if (rc == 0) {
      HP_CUDA(cudaMemcpyAsync(d_y, hy, bytes, cudaMemcpyHostToDevice, s));
      HP_CUDA(cudaStreamSynchronize(s));  // hy is reused by the next call
    }
  }
  if (rc != 0)
    throw std::runtime_error("black-box apply" + std::string(adjoint ? "_adjoint" : "") + " failed (status " +
                             std::to_string(rc) + ")");
}

DeviceOperator::~DeviceOperator() {
  if (d_x_) cudaFree(d_x_);
  if (d_a_) cudaFree(d_a_);
}

Matrix DeviceOperator::apply(const Matrix& x, bool adjoint) const {
  if (x.rows() != n_) throw std::invalid_argument("operator apply: row mismatch");
  DeviceGuard g(device_);
  DevOp d;
  d.kind = kind_;
  d.dim = dim_;
  d.n = n_;
  d.x = d_x_;
  d.a = d_a_;
  d.param = param_;
  d.symmetric = symmetric_;
  d.ltab = log_table_device(device_);
  cudaStream_t s;
  HP_CUDA(cudaStreamCreate(&s));
  Matrix y(x.rows(), x.cols());
  if (fn_ && !device_pointers_) {
    cudaStreamDestroy(s);
    if (x.cols() > 0 && fn_(ctx_, adjoint ? 1 : 0, x.data(), x.cols(), y.data(), nullptr) != 0)
      throw std::runtime_error("black-box apply failed");
    return y;
  }
  {
    DevBuf<double> dx(size_t(x.size()), s), dy(size_t(x.size()), s);
    HP_CUDA(cudaMemcpyAsync(dx.get(), x.data(), size_t(x.size()) * 8, cudaMemcpyHostToDevice, s));
    if (x.cols() > 0 && fn_) call(adjoint, dx.get(), x.cols(), dy.get(), s);
    else if (x.cols() > 0) launch_full_apply(d, adjoint, dx.get(), int(x.cols()), dy.get(), s);
    HP_CUDA(cudaMemcpyAsync(y.data(), dy.get(), size_t(x.size()) * 8, cudaMemcpyDeviceToHost, s));
    HP_CUDA(cudaStreamSynchronize(s));
  }
  cudaStreamDestroy(s);
  return y;
}

// ---------------------------------------------------------------- rep

H1Rep::~H1Rep() {
  // pool allocations (cudaMallocAsync): return them to the retained pool
  if (d_factors || d_dense) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (d_factors) cudaFreeAsync(d_factors, nullptr);
    if (d_dense) cudaFreeAsync(d_dense, nullptr);
    cudaStreamSynchronize(nullptr);
    cudaSetDevice(prev);
  }
}

std::int64_t H1Rep::storage_total() const {
  std::int64_t t = 0;
  for (size_t l = 0; l < levels.size(); ++l) {
    const auto& ld = levels[l];
    for (size_t p = 0; p < ld.pairs.size(); ++p) {
      if (!counts_pair(int(l), int(p))) continue;
      t += std::int64_t(tree->box(ld.pairs[p].first).points.size()) * ld.ku[p];
      t += std::int64_t(tree->box(ld.pairs[p].second).points.size()) * ld.kv[p];
      t += std::int64_t(ld.ku[p]) * ld.kv[p];
    }
  }
  for (size_t p = 0; p < dense.pairs.size(); ++p)
    if (dense.off[p] >= 0)
      t += std::int64_t(tree->box(dense.pairs[p].first).points.size()) *
           std::int64_t(tree->box(dense.pairs[p].second).points.size());
  return t;
}

LowRankBlockHost H1Rep::block(int level, int p) const {
  DeviceGuard g(device);
  const auto& ld = levels.at(size_t(level));
  if (ld.uoff.at(size_t(p)) < 0)
    throw std::invalid_argument("block (" + std::to_string(level) + ", " + std::to_string(p) +
                                ") is not held by this rank of a sharded representation");
  const auto [a, b] = ld.pairs.at(size_t(p));
  const int ma = int(layout->count[size_t(a)]), mb = int(layout->count[size_t(b)]);
  std::vector<double> u(size_t(ma) * rank), v(size_t(mb) * rank), bb(size_t(rank) * rank);
  HP_CUDA(cudaMemcpy(u.data(), d_factors + ld.uoff[size_t(p)], u.size() * 8, cudaMemcpyDeviceToHost));
  HP_CUDA(cudaMemcpy(v.data(), d_factors + ld.voff[size_t(p)], v.size() * 8, cudaMemcpyDeviceToHost));
  HP_CUDA(cudaMemcpy(bb.data(), d_factors + ld.boff[size_t(p)], bb.size() * 8, cudaMemcpyDeviceToHost));
  const int ku = ld.ku[size_t(p)], kv = ld.kv[size_t(p)];
  LowRankBlockHost out{Matrix(ma, ku), Matrix(ku, kv), Matrix(mb, kv)};
  // rows back to box.points order
  const auto& pa = tree->box(a).points;
  const auto& pb = tree->box(b).points;
  for (int s = 0; s < ma; ++s) {
    const std::int64_t tr = layout->inv[size_t(pa[size_t(s)])] - layout->start[size_t(a)];
    for (int j = 0; j < ku; ++j) out.u(s, j) = u[size_t(tr + std::int64_t(j) * ma)];
  }
  for (int s = 0; s < mb; ++s) {
    const std::int64_t tr = layout->inv[size_t(pb[size_t(s)])] - layout->start[size_t(b)];
    for (int j = 0; j < kv; ++j) out.v(s, j) = v[size_t(tr + std::int64_t(j) * mb)];
  }
  for (int i = 0; i < ku; ++i)
    for (int j = 0; j < kv; ++j) out.b(i, j) = bb[size_t(i + j * rank)];
  return out;
}

Matrix H1Rep::dense_block(int p) const {
  DeviceGuard g(device);
  const auto [lam, mu] = dense.pairs.at(size_t(p));
  if (dense.off.at(size_t(p)) < 0)
    throw std::invalid_argument("dense block " + std::to_string(p) + " is not held by this rank");
  const Index ml = Index(tree->box(lam).points.size()), mm = Index(tree->box(mu).points.size());
  Matrix d(ml, mm);
  HP_CUDA(cudaMemcpy(d.data(), d_dense + dense.off[size_t(p)], size_t(ml * mm) * 8, cudaMemcpyDeviceToHost));
  return d;
}

std::int64_t H1Rep::export_all(double* host_factors, double* host_dense) const {
  DeviceGuard g(device);
  HP_CUDA(cudaMemcpy(host_factors, d_factors, size_t(factor_doubles) * 8, cudaMemcpyDeviceToHost));
  HP_CUDA(cudaMemcpy(host_dense, d_dense, size_t(dense_doubles) * 8, cudaMemcpyDeviceToHost));
  return (factor_doubles + dense_doubles) * 8;
}

void H1Rep::apply_device(const double* x, int w, bool adjoint, double* y, cudaStream_t s) const {
  // x: tree order row-major n x w; y: tree order col-major n x w (accumulated)
  const int k = rank;
  for (size_t l = 2; l < levels.size(); ++l) {
    const auto& ld = levels[l];
    if (ld.pairs.empty()) continue;
    std::vector<CoeffTask> coeff;
    std::vector<std::int64_t> ss, sc;
    std::vector<PeelTask> tasks;
    std::vector<PeelRef> refs;
    std::vector<PeelTerm> terms;
    for (size_t p = 0; p < ld.pairs.size(); ++p) {
      const auto [a, b] = ld.pairs[p];
      const int src = adjoint ? a : b;
      CoeffTask t{};
      t.f = adjoint ? ld.uoff[p] : ld.voff[p];
      t.b = ld.boff[p];
      t.t_out = std::int64_t(p) * k * w;
      t.f_row0 = layout->start[size_t(src)];
      t.frows = int(layout->count[size_t(src)]);
      t.seg_begin = int(ss.size());
      ss.push_back(layout->start[size_t(src)]);
      sc.push_back(layout->count[size_t(src)]);
      t.seg_end = int(ss.size());
      t.btrans = adjoint ? 1 : 0;
      coeff.push_back(t);
    }
    // expansion: group pairs by output box
    std::map<int, std::vector<int>> by_box;
    for (size_t p = 0; p < ld.pairs.size(); ++p)
      by_box[adjoint ? ld.pairs[p].second : ld.pairs[p].first].push_back(int(p));
    for (auto& [box, ps] : by_box) {
      const int rows = int(layout->count[size_t(box)]);
      const int tb = int(terms.size());
      for (int p : ps)
        terms.push_back(PeelTerm{adjoint ? ld.voff[size_t(p)] : ld.uoff[size_t(p)], std::int64_t(p) * k * w,
                                 rows, 0});
      const int te = int(terms.size());
      for (int t0 = 0; t0 < rows; t0 += kTile) {
        tasks.push_back(PeelTask{layout->start[size_t(box)] + t0, std::min(kTile, rows - t0),
                                 int(tree->num_points()), int(refs.size()), int(refs.size()) + 1, w, 0});
        refs.push_back(PeelRef{tb, te, t0});
      }
    }
    DevBuf<CoeffTask> dc;
    dc.upload(coeff, s);
    DevBuf<std::int64_t> dss, dsc;
    dss.upload(ss, s);
    dsc.upload(sc, s);
    DevBuf<double> tbuf(coeff.size() * size_t(k) * size_t(w), s);
    launch_peel_coeff(dc.get(), int(coeff.size()), d_factors, d_factors, dss.get(), dsc.get(), x, w,
                      0, k, w, tbuf.get(), s);
    DevBuf<PeelTask> dt;
    dt.upload(tasks, s);
    DevBuf<PeelRef> dref;
    dref.upload(refs, s);
    DevBuf<PeelTerm> dterm;
    dterm.upload(terms, s);
    launch_peel_apply(dt.get(), int(tasks.size()), dref.get(), dterm.get(), d_factors, tbuf.get(), k, w, y, 0,
                      1.0, s);
    HP_CUDA(cudaStreamSynchronize(s));
  }
  if (dense_ready && !dense.pairs.empty()) {
    std::vector<DenseTask> dt;
    std::vector<int> off(size_t(tree->num_boxes()) + 1, 0);
    std::vector<std::vector<DenseTask>> per_box(size_t(tree->num_boxes()));
    for (size_t p = 0; p < dense.pairs.size(); ++p) {
      const auto [lam, mu] = dense.pairs[p];
      DenseTask t{dense.off[p], layout->start[size_t(lam)], layout->start[size_t(mu)],
                  int(layout->count[size_t(lam)]), int(layout->count[size_t(mu)])};
      per_box[size_t(adjoint ? mu : lam)].push_back(t);
    }
    for (size_t b = 0; b < per_box.size(); ++b) {
      off[b + 1] = off[b] + int(per_box[b].size());
      dt.insert(dt.end(), per_box[b].begin(), per_box[b].end());
    }
    DevBuf<DenseTask> d_dt;
    d_dt.upload(dt, s);
    DevBuf<int> d_off;
    d_off.upload(off, s);
    launch_dense_apply(d_dt.get(), d_off.get(), tree->num_boxes(), d_dense, x, w, adjoint, y,
                       tree->num_points(), s);
    HP_CUDA(cudaStreamSynchronize(s));
  }
}

Matrix H1Rep::apply(const Matrix& x, bool adjoint) const {
  if (!dense_ready) throw std::runtime_error("h1 apply: dense blocks missing");
  if (sharded()) throw std::invalid_argument("h1 apply: this rank holds a shard of the representation");
  const Index n = tree->num_points();
  if (x.rows() != n) throw std::invalid_argument("rep apply: row mismatch");
  DeviceGuard g(device);
  const int w = int(x.cols());
  Matrix y(n, w);
  if (w == 0) return y;
  cudaStream_t s;
  HP_CUDA(cudaStreamCreate(&s));
  {
    DevBuf<int> perm;
    perm.upload(layout->perm, s);
    DevBuf<double> dx(size_t(x.size()), s), xt(size_t(x.size()), s), yt(size_t(x.size()), s),
        dy(size_t(x.size()), s);
    HP_CUDA(cudaMemcpyAsync(dx.get(), x.data(), size_t(x.size()) * 8, cudaMemcpyHostToDevice, s));
    DevBuf<int> inv;
    inv.upload(layout->inv, s);
    constexpr int kCols = 32;  // column block (coefficient tiles are k x kCols)
    for (int c0 = 0; c0 < w; c0 += kCols) {
      const int wc = std::min(kCols, w - c0);
      // xt row-major tree order: xt[s * wc + c] = x[perm[s] + (c0 + c) n]
      launch_permute_rows(dx.get() + std::int64_t(c0) * n, 1, n, perm.get(), n, wc, xt.get(), wc, 1, s);
      HP_CUDA(cudaMemsetAsync(yt.get(), 0, size_t(n) * size_t(wc) * 8, s));
      apply_device(xt.get(), wc, adjoint, yt.get(), s);
      // y[perm[s] + (c0 + c) n] = yt[s + c n]
      launch_permute_rows(yt.get(), 1, n, inv.get(), n, wc, dy.get() + std::int64_t(c0) * n, 1, n, s);
    }
    HP_CUDA(cudaMemcpyAsync(y.data(), dy.get(), size_t(x.size()) * 8, cudaMemcpyDeviceToHost, s));
    HP_CUDA(cudaStreamSynchronize(s));
  }
  cudaStreamDestroy(s);
  return y;
}

// ---------------------------------------------------------------- verifier

double rel_error_power_method(const H1Rep& rep, const DeviceOperator& op, int iters,
                              std::uint64_t seed) {
  if (iters < 1) throw std::invalid_argument("power method needs iters >= 1");
  const Index n = rep.tree->num_points();
  if (op.rows() != n) throw std::invalid_argument("operator dimension mismatch");
  if (!rep.dense_ready) throw std::runtime_error("h1 apply: dense blocks missing");
  if (rep.sharded()) throw std::invalid_argument("power method: this rank holds a shard of the representation");
  DeviceGuard guard(rep.device);
  cudaStream_t s;
  HP_CUDA(cudaStreamCreate(&s));
  double result = 0.0;
  {
    Engine e(*rep.tree, *rep.adj, *rep.layout, op, s);
    DevBuf<double> x(size_t(n), s), y(size_t(n), s), z(size_t(n), s), t(size_t(n), s);
    std::vector<double> hx(static_cast<size_t>(n));
    auto norm = [&](const double* d) {
      HP_CUDA(cudaMemcpyAsync(hx.data(), d, size_t(n) * 8, cudaMemcpyDeviceToHost, s));
      HP_CUDA(cudaStreamSynchronize(s));
      double acc = 0.0;
      for (double v : hx) acc += v * v;
      return std::sqrt(acc);
    };
    auto scale_upload = [&](const std::vector<double>& v, double f) {
      std::vector<double> tmp(v.size());
      for (size_t i = 0; i < v.size(); ++i) tmp[i] = v[i] * f;
      HP_CUDA(cudaMemcpyAsync(x.get(), tmp.data(), tmp.size() * 8, cudaMemcpyHostToDevice, s));
      HP_CUDA(cudaStreamSynchronize(s));
    };
    // power_norm_diff (proj/src/linalg.cpp:179-196), tree order throughout
    auto power = [&](bool with_rep, std::uint64_t sd) {
      const Matrix g0 = gaussian_matrix(n, 1, sd);
      std::vector<double> v(static_cast<size_t>(n));
      double nrm = 0.0;
      for (Index i = 0; i < n; ++i) nrm += g0(i, 0) * g0(i, 0);
      nrm = std::sqrt(nrm);
      for (Index s2 = 0; s2 < n; ++s2) v[size_t(s2)] = g0(rep.layout->perm[size_t(s2)], 0);
      scale_upload(v, 1.0 / nrm);
      double estimate = 0.0;
      for (int it = 0; it < iters; ++it) {
        // y = A_rep x - A x   (or A x)
        e.op_apply(false, x.get(), 1, y.get());
        if (with_rep) {
          HP_CUDA(cudaMemsetAsync(t.get(), 0, size_t(n) * 8, s));
          rep.apply_device(x.get(), 1, false, t.get(), s);
          std::vector<double> a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
          HP_CUDA(cudaMemcpyAsync(a.data(), t.get(), size_t(n) * 8, cudaMemcpyDeviceToHost, s));
          HP_CUDA(cudaMemcpyAsync(b.data(), y.get(), size_t(n) * 8, cudaMemcpyDeviceToHost, s));
          HP_CUDA(cudaStreamSynchronize(s));
          for (size_t i = 0; i < a.size(); ++i) a[i] -= b[i];
          HP_CUDA(cudaMemcpyAsync(y.get(), a.data(), a.size() * 8, cudaMemcpyHostToDevice, s));
        }
        e.op_apply(true, y.get(), 1, z.get());
        if (with_rep) {
          HP_CUDA(cudaMemsetAsync(t.get(), 0, size_t(n) * 8, s));
          rep.apply_device(y.get(), 1, true, t.get(), s);
          std::vector<double> a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
          HP_CUDA(cudaMemcpyAsync(a.data(), t.get(), size_t(n) * 8, cudaMemcpyDeviceToHost, s));
          HP_CUDA(cudaMemcpyAsync(b.data(), z.get(), size_t(n) * 8, cudaMemcpyDeviceToHost, s));
          HP_CUDA(cudaStreamSynchronize(s));
          for (size_t i = 0; i < a.size(); ++i) a[i] -= b[i];
          HP_CUDA(cudaMemcpyAsync(z.get(), a.data(), a.size() * 8, cudaMemcpyHostToDevice, s));
        }
        const double nz = norm(z.get());
        if (nz == 0.0) return 0.0;
        estimate = std::sqrt(nz);
        std::vector<double> zz(hx);
        scale_upload(zz, 1.0 / nz);
      }
      return estimate;
    };
    const double err = power(true, mix_seed(seed, 11));
    const double ref = power(false, mix_seed(seed, 12));
    result = ref == 0.0 ? (err == 0.0 ? 0.0 : std::numeric_limits<double>::infinity()) : err / ref;
  }
  cudaStreamDestroy(s);
  return result;
}

}  // namespace hpeel

namespace hpeel {

// K4 probe (capi hp_debug_qr): the batched range finder on nb blocks stacked
// column-major one after another (block i: rows[i] x cols, ld rows[i]); Q
// (rows[i] x kmax each, stacked the same way) and the kept ranks come back.
// Returns the device milliseconds of run_qr.
double debug_qr(const double* blocks, const int* rows, int nb, int cols, int kmax, int device,
                double* q, int* ranks) {
  DeviceGuard guard(device);
  cudaStream_t s;
  HP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::vector<QrRequest> reqs;
  std::int64_t a = 0, o = 0;
  for (int i = 0; i < nb; ++i) {
    reqs.push_back(QrRequest{a, o, rows[i], rows[i], i});
    a += std::int64_t(rows[i]) * cols;
    o += std::int64_t(rows[i]) * kmax;
  }
  const QrPlan plan = plan_qr(reqs, cols, kmax);
  double ms = 0.0;
  {
    DevBuf<double> d_a(size_t(std::max<std::int64_t>(a, 1)), s), d_q(size_t(std::max<std::int64_t>(o, 1)), s);
    DevBuf<int> d_r(size_t(std::max(nb, 1)), s);
    HP_CUDA(cudaMemcpyAsync(d_a.get(), blocks, size_t(a) * 8, cudaMemcpyHostToDevice, s));
    Events ev;
    HP_CUDA(cudaEventRecord(ev.a, s));
    run_qr(plan, d_a.get(), d_q.get(), d_r.get(), cols, kmax, s);
    HP_CUDA(cudaEventRecord(ev.b, s));
    HP_CUDA(cudaMemcpyAsync(q, d_q.get(), size_t(o) * 8, cudaMemcpyDeviceToHost, s));
    HP_CUDA(cudaMemcpyAsync(ranks, d_r.get(), size_t(nb) * sizeof(int), cudaMemcpyDeviceToHost, s));
    HP_CUDA(cudaStreamSynchronize(s));
    ms = ev.ms();
  }
  HP_CUDA(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
  return ms;
}

// K1 parity probe (capi hp_debug_payload): payload rows of every box at
// `level`, n x 2r col-major in input order.
Matrix debug_payload(const BoxTree& tree, const TreeLayout& lay, int level, int r,
                     std::uint64_t seed, int device) {
  if (level < 0 || level > tree.depth()) throw std::invalid_argument("level out of range");
  if (r < 1) throw std::invalid_argument("width must be >= 1");
  DeviceGuard guard(device);
  const Index n = tree.num_points();
  std::vector<int> pos_box(static_cast<size_t>(n), -1), local(static_cast<size_t>(n), 0);
  for (int b : tree.level_boxes(level)) {
    const int* lr = lay.local_flat.data() + lay.local_off[size_t(b)];
    for (std::int64_t q = 0; q < lay.count[size_t(b)]; ++q) {
      pos_box[size_t(lay.start[size_t(b)] + q)] = b;
      local[size_t(lay.start[size_t(b)] + q)] = lr[q];
    }
  }
  Matrix out(n, 2 * r);
  cudaStream_t s;
  HP_CUDA(cudaStreamCreate(&s));
  {
    DevBuf<int> d_pb, d_loc, d_inv;
    d_pb.upload(pos_box, s);
    d_loc.upload(local, s);
    d_inv.upload(lay.inv, s);
    DevBuf<double> g(size_t(n) * 2 * size_t(r), s), o(size_t(n) * 2 * size_t(r), s);
    HP_CUDA(cudaMemsetAsync(g.get(), 0, size_t(n) * 2 * size_t(r) * 8, s));
    launch_payload_gaussian(g.get(), 2 * r, r, n, d_pb.get(), d_loc.get(), seed, level, s);
    // out[i + c n] = g[inv[i] * 2r + c]
    launch_permute_rows(g.get(), 2 * r, 1, d_inv.get(), n, 2 * r, o.get(), 1, n, s);
    HP_CUDA(cudaMemcpyAsync(out.data(), o.get(), size_t(out.size()) * 8, cudaMemcpyDeviceToHost, s));
    HP_CUDA(cudaStreamSynchronize(s));
  }
  cudaStreamDestroy(s);
  return out;
}

}  // namespace hpeel

namespace hpeel {
namespace {
__global__ void fast_log_probe_kernel(const double* x, std::int64_t n, double* y, const double* tab) {
  const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = 2.0 * half_log(x[i], tab);
}
}  // namespace

// Accuracy probe of the device log used by the log-kernel black box.
void debug_fast_log(const double* x, std::int64_t n, double* y, int device) {
  DeviceGuard guard(device);
  double *dx = nullptr, *dy = nullptr;
  HP_CUDA(cudaMalloc(&dx, size_t(n) * 8));
  HP_CUDA(cudaMalloc(&dy, size_t(n) * 8));
  HP_CUDA(cudaMemcpy(dx, x, size_t(n) * 8, cudaMemcpyHostToDevice));
  fast_log_probe_kernel<<<cdiv(n, 256), 256>>>(dx, n, dy, log_table_device(device));
  HP_LAUNCHED();
  HP_CUDA(cudaMemcpy(y, dy, size_t(n) * 8, cudaMemcpyDeviceToHost));
  cudaFree(dx);
  cudaFree(dy);
}
}  // namespace hpeel
