// H1 peeling driver (Alg. 4.1) on the device.
//
// Host-side control follows compress()/run_h1()/extract_leaf()
// (proj/src/peeling.cpp:211-275, :490-524, :576-639) step for step: the same
// plans (make_plan, :98-154), the same colors and payload seeds, the same
// rank-drop and pseudo-inverse tolerances. What changes is where the work
// runs and how much of it: per level one K1 payload launch, one K2 apply over
// the sample rows that the extraction reads, K3 peeling restricted to nonzero
// payload rows, batched K4 QR and K5 B-solves, all stream-ordered in HBM.
#include "peeling.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <set>
#include <sstream>
#include <stdexcept>
#include <unordered_map>

#include "kernels.hpp"
#include "rng.hpp"

namespace hpeel {

namespace {

using Clock = std::chrono::steady_clock;

constexpr int kForwardPhase = 0;  // proj/src/peeling.cpp:19-20
constexpr int kTile = 64;         // K2/K3 row tile
constexpr int kGramChunk = 512;

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t n, cudaStream_t s) {
    release();
    n_ = n;
    s_ = s;
    if (n) HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(v.size(), s);
    if (!v.empty())
      HP_CUDA(cudaMemcpyAsync(p_, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
};

struct Events {
  cudaEvent_t a = nullptr, b = nullptr;
  Events() {
    HP_CUDA(cudaEventCreate(&a));
    HP_CUDA(cudaEventCreate(&b));
  }
  ~Events() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  float ms() const {
    float t = 0.f;
    HP_CUDA(cudaEventElapsedTime(&t, a, b));
    return t;
  }
};

std::int64_t gemm_flops(std::int64_t m, std::int64_t n, std::int64_t k) { return 2 * m * n * k; }
std::int64_t svd_flops(std::int64_t m, std::int64_t n) {
  return m >= n ? 6 * m * n * n + 11 * n * n * n : 6 * n * m * m + 11 * m * m * m;
}

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    HP_CUDA(cudaGetDevice(&prev_));
    if (prev_ != dev) HP_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev_); }

 private:
  int prev_ = 0;
};

// Everything compress() needs on the device for one tree.
struct Engine {
  const BoxTree& tree;
  const AdjacencyInfo& adj;
  const TreeLayout& lay;
  const DeviceOperator& op;
  cudaStream_t s;
  int r = 0, k = 0;
  std::uint64_t seed = 0;
  Index n = 0;
  DevBuf<double> xt;  // tree-order coordinates
  DevBuf<double> at;  // tree-order dense matrix
  DevOp dop;
  DevBuf<std::int64_t> d_box_start, d_box_count;
  std::vector<std::vector<int>> anc;  // anc[l][box] = ancestor at level l (or -1)

  Engine(const BoxTree& t, const AdjacencyInfo& a, const TreeLayout& l, const DeviceOperator& o,
         cudaStream_t st)
      : tree(t), adj(a), lay(l), op(o), s(st) {
    n = tree.num_points();
    DevBuf<int> perm;
    perm.upload(lay.perm, s);
    dop.kind = op.kind();
    dop.dim = op.dim();
    dop.n = n;
    dop.param = op.param();
    dop.symmetric = op.symmetric() ? 1 : 0;
    if (op.kind() == kOpDense) {
      DevBuf<double> tmp(size_t(n) * size_t(n), s);
      at.alloc(size_t(n) * size_t(n), s);
      // rows then columns: at[s + t n] = a[perm[s] + perm[t] n]
      launch_permute_rows(op.device_matrix(), 1, n, perm.get(), n, int(n), tmp.get(), 1, n, s);
      launch_permute_rows(tmp.get(), n, 1, perm.get(), n, int(n), at.get(), n, 1, s);
      dop.a = at.get();
    } else {
      xt.alloc(size_t(op.dim()) * size_t(n), s);
      launch_permute_rows(op.device_points(), 1, n, perm.get(), n, op.dim(), xt.get(), 1, n, s);
      dop.x = xt.get();
    }
    d_box_start.upload(lay.start, s);
    d_box_count.upload(lay.count, s);
    anc.assign(size_t(tree.depth() + 1), std::vector<int>(size_t(tree.num_boxes()), -1));
    for (const Box& b : tree.boxes()) {
      int cur = b.id;
      for (int l = b.level; l >= 0; --l) {
        anc[size_t(l)][size_t(b.id)] = cur;
        cur = tree.box(cur).parent;
      }
    }
    HP_CUDA(cudaStreamSynchronize(s));
  }
  std::int64_t start(int b) const { return lay.start[size_t(b)]; }
  int count(int b) const { return int(lay.count[size_t(b)]); }
};

// Index of pair (a, b) in a sorted admissible-pairs list, -1 if absent.
int pair_index(const std::vector<std::pair<int, int>>& pairs, int a, int b) {
  auto it = std::lower_bound(pairs.begin(), pairs.end(), std::make_pair(a, b));
  if (it == pairs.end() || *it != std::make_pair(a, b)) return -1;
  return int(it - pairs.begin());
}
std::pair<int, int> first_range(const std::vector<std::pair<int, int>>& pairs, int a) {
  auto lo = std::lower_bound(pairs.begin(), pairs.end(), std::make_pair(a, std::numeric_limits<int>::min()));
  auto hi = std::lower_bound(pairs.begin(), pairs.end(), std::make_pair(a + 1, std::numeric_limits<int>::min()));
  return {int(lo - pairs.begin()), int(hi - pairs.begin())};
}

// Reference flop count of H1Rep::apply_truncated(level) for one width-w
// product (proj/src/hmatrix.cpp:86-100).
std::int64_t truncated_apply_flops(const H1Rep& rep, int level, std::int64_t w,
                                   const Engine& e) {
  std::int64_t f = 0;
  for (int l = 2; l <= std::min<int>(level, int(rep.levels.size()) - 1); ++l) {
    const auto& ld = rep.levels[size_t(l)];
    for (size_t p = 0; p < ld.pairs.size(); ++p) {
      const std::int64_t ma = e.count(ld.pairs[p].first), mb = e.count(ld.pairs[p].second);
      f += gemm_flops(ld.kv[p], w, mb) + gemm_flops(ld.ku[p], w, ld.kv[p]) + gemm_flops(ma, w, ld.ku[p]);
    }
  }
  return f;
}

// Batched qr_orthonormal over sample blocks (see k_qr.cu). Requests are
// col-major blocks in `data` (ld = rows); Q(:, :k) lands in `out`.
struct QrRequest {
  std::int64_t a;
  std::int64_t out;
  int rows;
  int ldo;
  int rank_slot;
};

void batched_qr(const std::vector<QrRequest>& reqs, double* data, double* out, int* d_ranks,
                int r, int kmax, cudaStream_t s) {
  const int rm = qr_rows_max(r);
  std::vector<QrBlock> direct, tops;
  std::vector<std::vector<QrBlock>> chunk_rounds;             // by round: data S (0) / W
  std::vector<std::vector<QrBlock>> back_rounds;              // by round
  std::int64_t wsize = 0, tausize = 0;
  struct Pending {
    std::vector<QrBlock> back;  // per round
  };
  for (const QrRequest& q : reqs) {
    if (q.rows <= rm) {
      direct.push_back(QrBlock{q.a, q.out, 0, 0, q.rows, q.rows, q.ldo, 0, q.rank_slot, 0});
      continue;
    }
    std::int64_t cur_off = q.a;
    int cur_rows = q.rows, cur_ld = q.rows;
    std::int64_t cur_c = -1;  // C offset of the current matrix in W (round >= 1)
    int round = 0;
    while (cur_rows > rm) {
      const int nch = (cur_rows + rm - 1) / rm;
      const int base = cur_rows / nch, extra = cur_rows % nch;
      int next_rows = 0;
      for (int i = 0; i < nch; ++i) next_rows += std::min(base + (i < extra ? 1 : 0), r);
      const std::int64_t stacked = wsize;
      wsize += std::int64_t(next_rows) * r;
      const std::int64_t c_next = wsize;
      wsize += std::int64_t(next_rows) * kmax;
      if (int(chunk_rounds.size()) <= round) chunk_rounds.resize(size_t(round) + 1);
      if (int(back_rounds.size()) <= round) back_rounds.resize(size_t(round) + 1);
      int row = 0, srow = 0;
      for (int i = 0; i < nch; ++i) {
        const int cr = base + (i < extra ? 1 : 0);
        const std::int64_t tau = tausize;
        tausize += r;
        chunk_rounds[size_t(round)].push_back(
            QrBlock{cur_off + row, stacked + srow, tau, 0, cr, cur_ld, next_rows, 0, -1, 0});
        QrBlock bp{};
        bp.a = cur_off + row;
        bp.tau = tau;
        bp.c = c_next + srow;
        bp.ldc = next_rows;
        bp.rows = cr;
        bp.lda = cur_ld;
        if (round == 0) {
          bp.out = q.out + row;
          bp.ldo = q.ldo;
        } else {
          bp.out = cur_c + row;
          bp.ldo = cur_rows;
        }
        bp.rank_slot = -1;
        back_rounds[size_t(round)].push_back(bp);
        row += cr;
        srow += std::min(cr, r);
      }
      cur_off = stacked;
      cur_rows = next_rows;
      cur_ld = next_rows;
      cur_c = c_next;
      ++round;
    }
    tops.push_back(QrBlock{cur_off, cur_c, 0, 0, cur_rows, cur_ld, cur_rows, 0, q.rank_slot, 0});
  }
  DevBuf<double> w(size_t(std::max<std::int64_t>(wsize, 1)), s);
  DevBuf<double> tau(size_t(std::max<std::int64_t>(tausize, 1)), s);
  DevBuf<QrBlock> d_blocks;
  if (!direct.empty()) {
    d_blocks.upload(direct, s);
    launch_qr_top(d_blocks.get(), int(direct.size()), data, out, d_ranks, r, kmax,
                  kQrRankDropTol, s);
  }
  for (size_t rd = 0; rd < chunk_rounds.size(); ++rd) {
    DevBuf<QrBlock> d;
    d.upload(chunk_rounds[rd], s);
    launch_qr_chunk(d.get(), int(chunk_rounds[rd].size()), rd == 0 ? data : w.get(), w.get(),
                    tau.get(), r, s);
  }
  if (!tops.empty()) {
    DevBuf<QrBlock> d;
    d.upload(tops, s);
    launch_qr_top(d.get(), int(tops.size()), w.get(), w.get(), d_ranks, r, kmax, kQrRankDropTol, s);
  }
  for (size_t rd = back_rounds.size(); rd-- > 0;) {
    DevBuf<QrBlock> d;
    d.upload(back_rounds[rd], s);
    launch_qr_backprop(d.get(), int(back_rounds[rd].size()), rd == 0 ? data : w.get(), tau.get(),
                       w.get(), rd == 0 ? out : w.get(), r, kmax, s);
  }
  HP_CUDA(cudaStreamSynchronize(s));  // keep task arrays alive until done
}

// Gram products X^T Y for a list of (x, y, rows, ...) requests, one nx x ny
// result per request, summed over row chunks in fixed order.
struct GramReq {
  std::int64_t x, y;
  int rows, lx, ly, x_rowmajor, y_rowmajor;
};
void batched_gram(const std::vector<GramReq>& reqs, const double* xb, const double* yb, int nx,
                  int ny, double* out, cudaStream_t s) {
  if (reqs.empty()) return;
  std::vector<GramTask> tasks;
  std::vector<std::int64_t> off(reqs.size() + 1, 0);
  for (size_t i = 0; i < reqs.size(); ++i) {
    const GramReq& q = reqs[i];
    for (int r0 = 0; r0 < q.rows; r0 += kGramChunk) {
      GramTask t{};
      t.x = q.x + (q.x_rowmajor ? std::int64_t(r0) * q.lx : r0);
      t.y = q.y + (q.y_rowmajor ? std::int64_t(r0) * q.ly : r0);
      t.out = std::int64_t(tasks.size()) * nx * ny;
      t.rows = std::min(kGramChunk, q.rows - r0);
      t.lx = q.lx;
      t.ly = q.ly;
      t.x_rowmajor = q.x_rowmajor;
      t.y_rowmajor = q.y_rowmajor;
      tasks.push_back(t);
    }
    off[i + 1] = std::int64_t(tasks.size());
  }
  DevBuf<GramTask> d_tasks;
  d_tasks.upload(tasks, s);
  DevBuf<std::int64_t> d_off;
  d_off.upload(off, s);
  DevBuf<double> partial(tasks.size() * size_t(nx) * size_t(ny), s);
  launch_gram(d_tasks.get(), int(tasks.size()), xb, yb, nx, ny, partial.get(), s);
  launch_sum_partials(d_off.get(), int(reqs.size()), partial.get(), nx * ny, out, s);
  HP_CUDA(cudaStreamSynchronize(s));
}

// Peeling task lists for one set of sample blocks (H1 level or leaf phase).
struct PeelPlan {
  std::vector<CoeffTask> coeff_fwd, coeff_adj;
  std::vector<std::int64_t> seg_start, seg_count;
  std::vector<PeelTask> tasks_fwd, tasks_adj;
  std::vector<PeelTerm> terms_fwd, terms_adj;
};

struct SampleBlock {
  int box;          // row box
  int color;
  std::int64_t off; // sample block offset (col-major, ld = |I_box|)
};

// Builds the K3 task lists: for every sample block (box a, color c), the
// terms U_q[rows a] T_{q,c} (forward) / V_q[rows a] T^a_{q,c} (adjoint) of all
// built levels lp < `top` whose row box contains a.
// payload_boxes[c] = payload boxes of color c; identity = leaf phase.
PeelPlan build_peel_plan(const Engine& e, const H1Rep& rep, const std::vector<SampleBlock>& blocks,
                         const std::vector<std::vector<int>>& payload_boxes, int top_level,
                         int w, bool identity, bool with_adjoint) {
  PeelPlan pp;
  const int k = e.k;
  // group[(lp, box, c)] -> segment range of payload boxes under `box`
  struct Key {
    int lp, box, c;
    bool operator==(const Key& o) const { return lp == o.lp && box == o.box && c == o.c; }
  };
  struct KeyHash {
    size_t operator()(const Key& x) const {
      return (size_t(x.lp) * 1000003u + size_t(x.box)) * 1000033u + size_t(x.c);
    }
  };
  std::unordered_map<Key, std::vector<int>, KeyHash> groups;
  for (int c = 0; c < int(payload_boxes.size()); ++c) {
    for (int v : payload_boxes[size_t(c)]) {
      const int lv = e.tree.box(v).level;
      for (int lp = 2; lp <= std::min(lv, top_level); ++lp) groups[Key{lp, e.anc[size_t(lp)][size_t(v)], c}].push_back(v);
    }
  }
  std::unordered_map<std::uint64_t, int> tidx;  // (side, lp, q, c) -> coefficient index or -1
  auto coeff = [&](int side, int lp, int q, int c) -> int {
    const std::uint64_t key = ((std::uint64_t(side) * 64 + std::uint64_t(lp)) * (1ull << 28) +
                               std::uint64_t(q)) * (1ull << 24) + std::uint64_t(c);
    auto it = tidx.find(key);
    if (it != tidx.end()) return it->second;
    const auto& ld = rep.levels[size_t(lp)];
    const auto [x, y] = ld.pairs[size_t(q)];
    const int src_box = side == 0 ? y : x;
    auto g = groups.find(Key{lp, src_box, c});
    if (g == groups.end()) return tidx[key] = -1;
    CoeffTask t{};
    if (side == 0) {
      t.f = ld.voff[size_t(q)];
      t.btrans = 0;
    } else {
      t.f = ld.uoff[size_t(q)];
      t.btrans = 1;
    }
    t.b = ld.boff[size_t(q)];
    t.f_row0 = e.start(src_box);
    t.frows = e.count(src_box);
    t.seg_begin = int(pp.seg_start.size());
    for (int v : g->second) {
      pp.seg_start.push_back(e.start(v));
      pp.seg_count.push_back(e.count(v));
    }
    t.seg_end = int(pp.seg_start.size());
    auto& list = side == 0 ? pp.coeff_fwd : pp.coeff_adj;
    t.t_out = std::int64_t(list.size()) * k * w;
    list.push_back(t);
    return tidx[key] = int(list.size()) - 1;
  };
  for (const SampleBlock& sb : blocks) {
    const int a = sb.box;
    const int la = e.tree.box(a).level;
    const int rows = e.count(a);
    for (int t0 = 0; t0 < rows; t0 += kTile) {
      PeelTask tf{sb.off + t0, std::min(kTile, rows - t0), rows, int(pp.terms_fwd.size()), 0};
      PeelTask ta{sb.off + t0, std::min(kTile, rows - t0), rows, int(pp.terms_adj.size()), 0};
      for (int lp = 2; lp <= std::min(la, top_level); ++lp) {
        const auto& ld = rep.levels[size_t(lp)];
        if (ld.pairs.empty()) continue;
        const int ap = e.anc[size_t(lp)][size_t(a)];
        const std::int64_t roff = e.start(a) - e.start(ap) + t0;
        const auto [q0, q1] = first_range(ld.pairs, ap);
        for (int q = q0; q < q1; ++q) {
          const int ti = coeff(0, lp, q, sb.color);
          if (ti >= 0)
            pp.terms_fwd.push_back(PeelTerm{ld.uoff[size_t(q)] + roff, std::int64_t(ti) * k * w, e.count(ap), 0});
        }
        if (!with_adjoint) continue;
        for (int x : e.adj.interaction[size_t(ap)]) {
          const int q = pair_index(ld.pairs, x, ap);
          if (q < 0) continue;
          const int ti = coeff(1, lp, q, sb.color);
          if (ti >= 0)
            pp.terms_adj.push_back(PeelTerm{ld.voff[size_t(q)] + roff, std::int64_t(ti) * k * w, e.count(ap), 0});
        }
      }
      tf.term_end = int(pp.terms_fwd.size());
      ta.term_end = int(pp.terms_adj.size());
      if (tf.term_end > tf.term_begin) pp.tasks_fwd.push_back(tf);
      if (with_adjoint && ta.term_end > ta.term_begin) pp.tasks_adj.push_back(ta);
    }
  }
  return pp;
}

// Runs a peel plan: coefficient launches then subtraction launches.
void run_peel(const PeelPlan& pp, const Engine& e, const H1Rep& rep, const double* g, int gld,
              int w, bool identity, double* samples, int r_adj_col, cudaStream_t s) {
  const int k = e.k;
  DevBuf<std::int64_t> d_ss, d_sc;
  d_ss.upload(pp.seg_start, s);
  d_sc.upload(pp.seg_count, s);
  for (int side = 0; side < 2; ++side) {
    const auto& coeff = side == 0 ? pp.coeff_fwd : pp.coeff_adj;
    const auto& tasks = side == 0 ? pp.tasks_fwd : pp.tasks_adj;
    const auto& terms = side == 0 ? pp.terms_fwd : pp.terms_adj;
    if (coeff.empty() || tasks.empty()) continue;
    DevBuf<CoeffTask> d_coeff;
    d_coeff.upload(coeff, s);
    DevBuf<double> tbuf(coeff.size() * size_t(k) * size_t(w), s);
    launch_peel_coeff(d_coeff.get(), int(coeff.size()), rep.d_factors, rep.d_factors, d_ss.get(),
                      d_sc.get(), g, gld, identity ? -1 : (side == 0 ? 0 : e.r), k, w, tbuf.get(), s);
    DevBuf<PeelTask> d_tasks;
    d_tasks.upload(tasks, s);
    DevBuf<PeelTerm> d_terms;
    d_terms.upload(terms, s);
    launch_peel_apply(d_tasks.get(), int(tasks.size()), d_terms.get(), rep.d_factors, tbuf.get(), k,
                      w, samples, side == 0 ? 0 : r_adj_col, -1.0, s);
    HP_CUDA(cudaStreamSynchronize(s));
  }
}

}  // namespace

// ---------------------------------------------------------------------------

void PeelConfig::validate() const {
  if (rank < 1) throw std::invalid_argument("fixed rank must be >= 1");
  if (oversample < 0) throw std::invalid_argument("negative oversampling");
}

std::string RunReport::to_csv() const {
  std::ostringstream out;
  out << "phase,level,colors,forward_cols,adjoint_cols,wall_ms_total,wall_ms_net,net_flops\n";
  for (const PhaseReport& p : phases) {
    out << p.phase << ',' << p.level << ',' << p.colors << ',' << p.forward_cols << ','
        << p.adjoint_cols << ',' << p.wall_ms_total << ',' << p.wall_ms_net << ','
        << p.net_flops << '\n';
  }
  return out.str();
}

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
  cudaStream_t s;
  HP_CUDA(cudaStreamCreate(&s));
  Matrix y(x.rows(), x.cols());
  {
    DevBuf<double> dx(size_t(x.size()), s), dy(size_t(x.size()), s);
    HP_CUDA(cudaMemcpyAsync(dx.get(), x.data(), size_t(x.size()) * 8, cudaMemcpyHostToDevice, s));
    if (x.cols() > 0) launch_full_apply(d, adjoint, dx.get(), int(x.cols()), dy.get(), s);
    HP_CUDA(cudaMemcpyAsync(y.data(), dy.get(), size_t(x.size()) * 8, cudaMemcpyDeviceToHost, s));
    HP_CUDA(cudaStreamSynchronize(s));
  }
  cudaStreamDestroy(s);
  return y;
}

// ---------------------------------------------------------------- rep

H1Rep::~H1Rep() {
  if (d_factors) cudaFree(d_factors);
  if (d_dense) cudaFree(d_dense);
}

std::int64_t H1Rep::storage_total() const {
  std::int64_t t = 0;
  for (size_t l = 0; l < levels.size(); ++l) {
    const auto& ld = levels[l];
    for (size_t p = 0; p < ld.pairs.size(); ++p) {
      t += std::int64_t(tree->box(ld.pairs[p].first).points.size()) * ld.ku[p];
      t += std::int64_t(tree->box(ld.pairs[p].second).points.size()) * ld.kv[p];
      t += std::int64_t(ld.ku[p]) * ld.kv[p];
    }
  }
  for (auto [lam, mu] : dense.pairs)
    t += std::int64_t(tree->box(lam).points.size()) * std::int64_t(tree->box(mu).points.size());
  return t;
}

LowRankBlockHost H1Rep::block(int level, int p) const {
  DeviceGuard g(device);
  const auto& ld = levels.at(size_t(level));
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
      for (int t0 = 0; t0 < rows; t0 += kTile) {
        PeelTask t{layout->start[size_t(box)] + t0, std::min(kTile, rows - t0), int(tree->num_points()),
                   int(terms.size()), 0};
        for (int p : ps)
          terms.push_back(PeelTerm{(adjoint ? ld.voff[size_t(p)] : ld.uoff[size_t(p)]) + t0,
                                   std::int64_t(p) * k * w, rows, 0});
        t.term_end = int(terms.size());
        tasks.push_back(t);
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
    DevBuf<PeelTerm> dterm;
    dterm.upload(terms, s);
    launch_peel_apply(dt.get(), int(tasks.size()), dterm.get(), d_factors, tbuf.get(), k, w, y, 0,
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
    // xt row-major tree order: xt[s * w + c] = x[perm[s] + c n]
    launch_permute_rows(dx.get(), 1, n, perm.get(), n, w, xt.get(), w, 1, s);
    HP_CUDA(cudaMemsetAsync(yt.get(), 0, size_t(x.size()) * 8, s));
    apply_device(xt.get(), w, adjoint, yt.get(), s);
    // y[perm[s] + c n] = yt[s + c n]
    DevBuf<int> inv;
    inv.upload(layout->inv, s);
    launch_permute_rows(yt.get(), 1, n, inv.get(), n, w, dy.get(), 1, n, s);
    HP_CUDA(cudaMemcpyAsync(y.data(), dy.get(), size_t(x.size()) * 8, cudaMemcpyDeviceToHost, s));
    HP_CUDA(cudaStreamSynchronize(s));
  }
  cudaStreamDestroy(s);
  return y;
}

// ---------------------------------------------------------------- compress

PeelResult compress(const DeviceOperator& op, std::shared_ptr<const BoxTree> tree,
                    const PeelConfig& config) {
  if (!tree) throw std::invalid_argument("null tree");
  if (op.rows() != tree->num_points() || op.cols() != tree->num_points())
    throw std::invalid_argument("operator and tree dimensions differ");
  config.validate();
  if (config.format != PeelFormat::kH1)
    throw std::invalid_argument("only format h1 is on the device hot path");
  if (config.strategy != ColoringStrategy::kGraph)
    throw std::invalid_argument("only the graph coloring strategy is on the device hot path");
  if (op.kind() != kOpDense && op.dim() != tree->dim())
    throw std::invalid_argument("operator and tree dimensions differ");

  DeviceGuard guard(op.device());
  const auto t_begin = Clock::now();
  auto adj = std::make_shared<const AdjacencyInfo>(adjacency(*tree));
  auto lay = std::make_shared<const TreeLayout>(tree_layout(*tree));
  const int r = config.sample_width();
  const int k = config.rank;
  if (2 * r > 160) throw std::invalid_argument("sample width k + p > 80 is not supported");

  cudaStream_t s;
  HP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  PeelResult result;
  auto rep = std::make_shared<H1Rep>();
  rep->tree = tree;
  rep->adj = adj;
  rep->layout = lay;
  rep->rank = k;
  rep->device = op.device();
  rep->levels.resize(size_t(tree->depth()) + 1);
  RunReport& report = result.report;
  double blackbox_ms = 0.0;

  try {
    Engine e(*tree, *adj, *lay, op, s);
    e.r = r;
    e.k = k;
    e.seed = config.seed;
    const Index n = tree->num_points();

    // Factor arena: U (|I_a| x k), V (|I_b| x k), B (k x k) per pair.
    std::int64_t ftotal = 0;
    for (int l = 2; l <= tree->depth(); ++l) {
      auto& ld = rep->levels[size_t(l)];
      ld.pairs = admissible_pairs(*tree, *adj, l);
      const size_t np = ld.pairs.size();
      ld.uoff.resize(np);
      ld.voff.resize(np);
      ld.boff.resize(np);
      ld.ku.assign(np, 0);
      ld.kv.assign(np, 0);
      for (size_t p = 0; p < np; ++p) {
        ld.uoff[p] = ftotal;
        ftotal += std::int64_t(e.count(ld.pairs[p].first)) * k;
        ld.voff[p] = ftotal;
        ftotal += std::int64_t(e.count(ld.pairs[p].second)) * k;
        ld.boff[p] = ftotal;
        ftotal += std::int64_t(k) * k;
      }
    }
    rep->factor_doubles = ftotal;
    HP_CUDA(cudaMalloc(&rep->d_factors, size_t(std::max<std::int64_t>(ftotal, 1)) * 8));

    // per-level pos -> box / local rank
    std::vector<int> pos_box(static_cast<size_t>(n)), local(static_cast<size_t>(n));
    DevBuf<int> d_pos_box, d_local, d_ranks;
    const int gld = 2 * r;
    DevBuf<double> g(size_t(n) * size_t(gld), s);

    for (int l = 2; l <= tree->depth(); ++l) {
      auto& ld = rep->levels[size_t(l)];
      if (ld.pairs.empty()) continue;  // proj/src/peeling.cpp:221 (built_level not advanced)
      {
        std::set<std::pair<int, int>> all(ld.pairs.begin(), ld.pairs.end());
        for (auto [a, b] : ld.pairs)
          if (!all.count({b, a})) throw std::logic_error("asymmetric admissibility structure");
      }
      if (l - 1 >= 2 && l - 1 > rep->built_level) {
        throw std::runtime_error("h1 apply: representation incomplete for level " + std::to_string(l - 1));
      }
      const auto t0 = Clock::now();
      PhaseReport ph;
      ph.phase = "h1";
      ph.level = l;
      const SamplingPlan plan = make_plan(*tree, *adj, l, SampleMode::kH1, r, config.seed, kForwardPhase);
      ph.colors = plan.colors();
      const int nc = plan.colors();
      std::vector<std::vector<int>> color_boxes(static_cast<size_t>(nc));
      std::vector<std::int64_t> pay_off(size_t(nc) + 1, 0);
      std::vector<int> pay_pos;
      for (int c = 0; c < nc; ++c) {
        for (auto [box, tag] : plan.matrices[size_t(c)].payload) {
          color_boxes[size_t(c)].push_back(box);
          for (std::int64_t q = 0; q < e.count(box); ++q) pay_pos.push_back(int(e.start(box) + q));
        }
        pay_off[size_t(c) + 1] = std::int64_t(pay_pos.size());
        ph.forward_cols += plan.matrices[size_t(c)].payload.empty() ? 0 : r;
      }
      ph.adjoint_cols = ph.forward_cols;
      const size_t np = ld.pairs.size();
      std::vector<int> pcolor(np);
      std::vector<std::int64_t> soff(np + 1, 0);
      for (size_t p = 0; p < np; ++p) {
        pcolor[p] = plan.block_to_matrix.at(ld.pairs[p]);
        soff[p + 1] = soff[p] + std::int64_t(e.count(ld.pairs[p].first)) * 2 * r;
      }
      std::vector<int> swap(np);
      for (size_t p = 0; p < np; ++p) swap[p] = pair_index(ld.pairs, ld.pairs[p].second, ld.pairs[p].first);

      // K1 payload
      std::fill(pos_box.begin(), pos_box.end(), -1);
      for (int b : tree->level_boxes(l)) {
        const int* lr = lay->local_flat.data() + lay->local_off[size_t(b)];
        for (int q = 0; q < e.count(b); ++q) {
          pos_box[size_t(e.start(b) + q)] = b;
          local[size_t(e.start(b) + q)] = lr[q];
        }
      }
      d_pos_box.upload(pos_box, s);
      d_local.upload(local, s);
      launch_payload_gaussian(g.get(), gld, r, n, d_pos_box.get(), d_local.get(), config.seed, l, s);

      // K2 apply
      std::vector<SampleTask> tasks;
      double evals = 0.0;
      for (size_t p = 0; p < np; ++p) {
        const int a = ld.pairs[p].first;
        const int rows = e.count(a);
        for (int t0 = 0; t0 < rows; t0 += kTile)
          tasks.push_back(SampleTask{e.start(a) + t0, soff[p] + t0, std::min(kTile, rows - t0),
                                     pcolor[p], rows, 0});
        evals += double(rows) * double(pay_off[size_t(pcolor[p]) + 1] - pay_off[size_t(pcolor[p])]);
      }
      ph.kernel_evals = evals;
      ph.apply_flops = evals * 2.0 * 2.0 * r;
      DevBuf<SampleTask> d_tasks;
      d_tasks.upload(tasks, s);
      DevBuf<std::int64_t> d_pay_off;
      d_pay_off.upload(pay_off, s);
      DevBuf<int> d_pay_pos;
      d_pay_pos.upload(pay_pos, s);
      DevBuf<double> samples(size_t(soff[np]), s);
      Events ev_apply, ev_peel, ev_qr, ev_b;
      HP_CUDA(cudaEventRecord(ev_apply.a, s));
      if (op.symmetric()) {
        launch_sample_apply(e.dop, false, d_tasks.get(), int(tasks.size()), d_pay_off.get(),
                            d_pay_pos.get(), g.get(), gld, 0, 2 * r, samples.get(), 0, s);
      } else {
        launch_sample_apply(e.dop, false, d_tasks.get(), int(tasks.size()), d_pay_off.get(),
                            d_pay_pos.get(), g.get(), gld, 0, r, samples.get(), 0, s);
        launch_sample_apply(e.dop, true, d_tasks.get(), int(tasks.size()), d_pay_off.get(),
                            d_pay_pos.get(), g.get(), gld, r, r, samples.get(), r, s);
      }
      HP_CUDA(cudaEventRecord(ev_apply.b, s));

      // K3 peel (prev_level = l - 1 >= 2)
      HP_CUDA(cudaEventRecord(ev_peel.a, s));
      if (l - 1 >= 2) {
        std::vector<SampleBlock> blocks(np);
        for (size_t p = 0; p < np; ++p) blocks[p] = SampleBlock{ld.pairs[p].first, pcolor[p], soff[p]};
        const PeelPlan pp = build_peel_plan(e, *rep, blocks, color_boxes, l - 1, r, false, true);
        // adjoint half starts at column r of each block: ocol0 = r
        run_peel(pp, e, *rep, g.get(), gld, r, false, samples.get(), r, s);
        ph.net_flops += 2 * std::int64_t(nc) * truncated_apply_flops(*rep, l - 1, r, e);
      }
      HP_CUDA(cudaEventRecord(ev_peel.b, s));

      if (config.capture_samples) {
        HP_CUDA(cudaStreamSynchronize(s));
        std::vector<Matrix> cap;
        for (size_t p = 0; p < np; ++p) {
          const int rows = e.count(ld.pairs[p].first);
          Matrix m(rows, 2 * r);
          HP_CUDA(cudaMemcpy(m.data(), samples.get() + soff[p], size_t(rows) * 2 * r * 8, cudaMemcpyDeviceToHost));
          cap.push_back(std::move(m));
        }
        rep->captured[l] = std::move(cap);
      }

      // K5a: middle = G'_a^T Y_p before the QR overwrites Y
      HP_CUDA(cudaEventRecord(ev_b.a, s));
      DevBuf<double> middle(np * size_t(r) * size_t(r), s), gpu(np * size_t(r) * size_t(k), s),
          vg(np * size_t(k) * size_t(r), s);
      {
        std::vector<GramReq> reqs(np);
        for (size_t p = 0; p < np; ++p) {
          const int a = ld.pairs[p].first;
          reqs[p] = GramReq{e.start(a) * gld + r, soff[p], e.count(a), gld, e.count(a), 1, 0};
        }
        batched_gram(reqs, g.get(), samples.get(), r, r, middle.get(), s);
      }
      HP_CUDA(cudaEventRecord(ev_b.b, s));
      HP_CUDA(cudaStreamSynchronize(s));
      float gram1_ms = ev_b.ms();

      // K4 QR: U_p from Y_p, V_swap(p) from Z_p
      HP_CUDA(cudaEventRecord(ev_qr.a, s));
      d_ranks.alloc(2 * np, s);
      {
        std::vector<QrRequest> reqs;
        reqs.reserve(2 * np);
        for (size_t p = 0; p < np; ++p) {
          const int rows = e.count(ld.pairs[p].first);
          reqs.push_back(QrRequest{soff[p], ld.uoff[p], rows, rows, int(p)});
          reqs.push_back(QrRequest{soff[p] + std::int64_t(rows) * r, ld.voff[size_t(swap[p])], rows,
                                   rows, int(np + size_t(swap[p]))});
        }
        batched_qr(reqs, samples.get(), rep->d_factors, d_ranks.get(), r, k, s);
      }
      HP_CUDA(cudaEventRecord(ev_qr.b, s));

      // K5b: gpU = G'^T U, VG = V^T G, B
      HP_CUDA(cudaEventRecord(ev_b.a, s));
      {
        std::vector<GramReq> ru(np), rv(np);
        for (size_t p = 0; p < np; ++p) {
          const auto [a, b] = ld.pairs[p];
          ru[p] = GramReq{e.start(a) * gld + r, ld.uoff[p], e.count(a), gld, e.count(a), 1, 0};
          rv[p] = GramReq{ld.voff[p], e.start(b) * gld, e.count(b), e.count(b), gld, 0, 1};
        }
        batched_gram(ru, g.get(), rep->d_factors, r, k, gpu.get(), s);
        batched_gram(rv, rep->d_factors, g.get(), k, r, vg.get(), s);
        DevBuf<std::int64_t> d_boff;
        d_boff.upload(ld.boff, s);
        launch_bsolve(int(np), gpu.get(), middle.get(), vg.get(), r, k, kPinvCutoff, d_boff.get(),
                      rep->d_factors, s);
        HP_CUDA(cudaStreamSynchronize(s));
      }
      HP_CUDA(cudaEventRecord(ev_b.b, s));
      std::vector<int> ranks(2 * np);
      HP_CUDA(cudaMemcpyAsync(ranks.data(), d_ranks.get(), ranks.size() * sizeof(int),
                              cudaMemcpyDeviceToHost, s));
      HP_CUDA(cudaStreamSynchronize(s));
      for (size_t p = 0; p < np; ++p) {
        ld.ku[p] = ranks[p];
        ld.kv[p] = ranks[np + p];
      }
      rep->built_level = l;
      ph.apply_ms = ev_apply.ms();
      ph.peel_ms = ev_peel.ms();
      ph.qr_ms = ev_qr.ms();
      ph.bsolve_ms = ev_b.ms() + gram1_ms;
      blackbox_ms += ph.apply_ms;
      // reference net flops: QR (flops.hpp:18-20) and the B solve (peeling.cpp:262-268)
      for (size_t p = 0; p < np; ++p) {
        const std::int64_t ma = e.count(ld.pairs[p].first), mb = e.count(ld.pairs[p].second);
        const std::int64_t ku = ld.ku[p], kv = ld.kv[p];
        ph.net_flops += 2 * ma * r * r + 2 * mb * r * r;
        ph.net_flops += gemm_flops(r, r, ma) + gemm_flops(r, ku, ma) + gemm_flops(kv, r, mb);
        if (ku > 0) ph.net_flops += svd_flops(r, ku) + gemm_flops(ku, r, r);
        if (kv > 0) ph.net_flops += svd_flops(r, kv) + gemm_flops(kv, ku, r);
      }
      ph.wall_ms_total = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
      ph.wall_ms_net = ph.wall_ms_total - ph.apply_ms;
      report.phases.push_back(ph);
    }
    rep->built_level = tree->depth();

    // ------------------------------------------------------------- leaf phase
    {
      const auto t0 = Clock::now();
      PhaseReport ph;
      ph.phase = "leaf";
      ph.level = tree->depth();
      const int w = tree->max_leaf_size();
      const SamplingPlan plan = make_plan(*tree, *adj, tree->depth(), SampleMode::kLeaf, w,
                                          config.seed, kForwardPhase);
      ph.colors = plan.colors();
      const int nc = plan.colors();
      std::vector<std::vector<int>> color_boxes(static_cast<size_t>(nc));
      std::vector<std::int64_t> pay_off(size_t(nc) + 1, 0);
      std::vector<int> pay_box;
      for (int c = 0; c < nc; ++c) {
        for (auto [box, tag] : plan.matrices[size_t(c)].payload) {
          color_boxes[size_t(c)].push_back(box);
          pay_box.push_back(box);
        }
        pay_off[size_t(c) + 1] = std::int64_t(pay_box.size());
        ph.forward_cols += plan.matrices[size_t(c)].payload.empty() ? 0 : w;
      }
      rep->dense.pairs = dense_pairs(*tree, *adj);
      const size_t nd = rep->dense.pairs.size();
      rep->dense.off.resize(nd);
      std::int64_t dtotal = 0;
      std::vector<SampleTask> tasks;
      std::vector<SampleBlock> blocks(nd);
      double evals = 0.0;
      for (size_t p = 0; p < nd; ++p) {
        const auto [lam, mu] = rep->dense.pairs[p];
        const int c = plan.block_to_matrix.at(rep->dense.pairs[p]);
        const int rows = e.count(lam);
        rep->dense.off[p] = dtotal;
        for (int t0 = 0; t0 < rows; t0 += kTile)
          tasks.push_back(SampleTask{e.start(lam) + t0, dtotal + t0, std::min(kTile, rows - t0), c, rows, 0});
        blocks[p] = SampleBlock{lam, c, dtotal};
        std::int64_t nnz = 0;
        for (std::int64_t q = pay_off[size_t(c)]; q < pay_off[size_t(c) + 1]; ++q) nnz += e.count(pay_box[size_t(q)]);
        evals += double(rows) * double(nnz);
        dtotal += std::int64_t(rows) * w;
      }
      ph.kernel_evals = evals;
      rep->dense_doubles = dtotal;
      HP_CUDA(cudaMalloc(&rep->d_dense, size_t(std::max<std::int64_t>(dtotal, 1)) * 8));
      DevBuf<SampleTask> d_tasks;
      d_tasks.upload(tasks, s);
      DevBuf<std::int64_t> d_pay_off;
      d_pay_off.upload(pay_off, s);
      DevBuf<int> d_pay_box;
      d_pay_box.upload(pay_box, s);
      Events ev_apply, ev_peel;
      HP_CUDA(cudaEventRecord(ev_apply.a, s));
      launch_identity_apply(e.dop, d_tasks.get(), int(tasks.size()), d_pay_off.get(), d_pay_box.get(),
                            e.d_box_start.get(), e.d_box_count.get(), w, rep->d_dense, s);
      HP_CUDA(cudaEventRecord(ev_apply.b, s));
      HP_CUDA(cudaEventRecord(ev_peel.a, s));
      if (tree->depth() >= 2) {
        const PeelPlan pp = build_peel_plan(e, *rep, blocks, color_boxes, tree->depth(), w, true, false);
        run_peel(pp, e, *rep, nullptr, 0, w, true, rep->d_dense, 0, s);
        ph.net_flops += std::int64_t(nc) * truncated_apply_flops(*rep, tree->depth(), w, e);
      }
      HP_CUDA(cudaEventRecord(ev_peel.b, s));
      HP_CUDA(cudaStreamSynchronize(s));
      if (config.capture_samples) {
        for (size_t p = 0; p < nd; ++p) {
          const int rows = e.count(rep->dense.pairs[p].first);
          Matrix m(rows, w);
          HP_CUDA(cudaMemcpy(m.data(), rep->d_dense + rep->dense.off[p], size_t(rows) * w * 8, cudaMemcpyDeviceToHost));
          rep->captured_leaf.push_back(std::move(m));
        }
      }
      rep->dense_ready = true;
      ph.apply_ms = ev_apply.ms();
      ph.peel_ms = ev_peel.ms();
      blackbox_ms += ph.apply_ms;
      ph.wall_ms_total = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
      ph.wall_ms_net = ph.wall_ms_total - ph.apply_ms;
      report.phases.push_back(ph);
    }
  } catch (...) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    throw;
  }
  HP_CUDA(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);

  for (const PhaseReport& p : report.phases) {
    report.forward_cols += p.forward_cols;
    report.adjoint_cols += p.adjoint_cols;
    report.net_flops += p.net_flops;
    if (p.phase != "leaf") report.max_sampling_colors = std::max(report.max_sampling_colors, p.colors);
  }
  report.wall_s_total = std::chrono::duration<double>(Clock::now() - t_begin).count();
  report.wall_s_net = report.wall_s_total - blackbox_ms * 1e-3;
  result.rep = rep;
  return result;
}

// ---------------------------------------------------------------- verifier

double rel_error_power_method(const H1Rep& rep, const DeviceOperator& op, int iters,
                              std::uint64_t seed) {
  if (iters < 1) throw std::invalid_argument("power method needs iters >= 1");
  const Index n = rep.tree->num_points();
  if (op.rows() != n) throw std::invalid_argument("operator dimension mismatch");
  if (!rep.dense_ready) throw std::runtime_error("h1 apply: dense blocks missing");
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
        launch_full_apply(e.dop, false, x.get(), 1, y.get(), s);
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
        launch_full_apply(e.dop, true, y.get(), 1, z.get(), s);
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
