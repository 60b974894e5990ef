// H1 peeling driver (Alg. 4.1) on the device.
//
// Control follows compress()/run_h1()/extract_leaf()
// (proj/src/peeling.cpp:211-275, :490-524, :576-639) step for step: the same
// plans (make_plan, :98-154), colors, payload seeds, rank-drop and
// pseudo-inverse tolerances, and the same error behaviour. What changes is
// where the work runs: every level's host plan (coloring, task lists, QR
// and peeling structure) is built on host threads up front, and the device
// executes the levels with no host round trip: K1 payload and K2 apply on
// the sample rows the extraction reads (apply stream, one level ahead), then
// K3 peeling restricted to nonzero payload rows, batched K4 QR and K5
// B-solves (main stream), so level l + 1's apply overlaps level l's
// factorization.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <future>
#include <memory>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <sstream>
#include <stdexcept>
#include <thread>

#include "engine.cuh"
#include "k2_i8.cuh"
#include "rng.hpp"
#include "shard.hpp"

namespace hpeel {

using namespace detail;

namespace {

using Clock = std::chrono::steady_clock;
constexpr int kForwardPhase = 0;  // proj/src/peeling.cpp:19-20

std::int64_t gemm_flops(std::int64_t m, std::int64_t n, std::int64_t k) { return 2 * m * n * k; }
std::int64_t svd_flops(std::int64_t m, std::int64_t n) {
  return m >= n ? 6 * m * n * n + 11 * n * n * n : 6 * n * m * m + 11 * m * m * m;
}

// Reference flop count of H1Rep::apply_truncated(level) for one width-w
// product (proj/src/hmatrix.cpp:86-100).
std::int64_t truncated_apply_flops(const H1Rep& rep, int level, std::int64_t w, const Engine& e) {
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

// Destroy `obj` on a detached thread (large host plans: their frees would
// otherwise sit on the driver thread between device phases or before return).
template <class T>
void reap_async(T&& obj) {
  auto* p = new std::decay_t<T>(std::forward<T>(obj));
  std::thread([p] { delete p; }).detach();
}

struct LevelWork {
  int level = 0;
  bool empty = true;
  bool symmetric = true;
  int nc = 0;
  std::int64_t fwd_cols = 0;
  size_t np = 0;
  std::vector<int> pcolor, swap;
  std::vector<std::int64_t> soff;
  std::vector<std::int64_t> pay_off;
  std::vector<int> pay_pos;
  std::vector<std::int64_t> step_off;      // int8 K2: 32-row K-steps per color (prefix)
  std::vector<int> step_color;             // color of every K-step
  std::vector<std::int64_t> pb_off;        // payload boxes per color (prefix)
  std::vector<int> pb_box;
  std::vector<int> pos_box, local;
  std::vector<K2Row> rowtab;               // K2 rows, grouped by shard and color
  std::vector<std::vector<K2Task>> k2;     // K2 tiles per shard
  std::vector<std::int64_t> seg;           // shard q owns samples [seg[q], seg[q+1])
  bool k2_checked = false;                 // some row box is in its own color's payload
  double evals = 0;
  bool has_peel = false;
  PeelPlan peel;
  // K4/K5 per shard: shard q owns pairs [fb[q], fb[q+1]) and
  // computes their U, V (QR), grams and B; factor segments are then shared
  struct Shard45 {
    std::int64_t p0 = 0, p1 = 0;
    QrPlan qr;
    GramPlan g_mid, g_gpu, g_vg;
  };
  std::vector<Shard45> s45;
  std::vector<std::int64_t> fb;
};

LevelWork build_level(const Engine& e, const H1Rep& rep, int l, const PeelConfig& cfg) {
  LevelWork w;
  w.level = l;
  const auto& ld = rep.levels[size_t(l)];
  if (ld.pairs.empty()) return w;
  w.empty = false;
  {
    std::set<std::pair<int, int>> all(ld.pairs.begin(), ld.pairs.end());
    for (auto [a, b] : ld.pairs)
      if (!all.count({b, a})) w.symmetric = false;
  }
  if (!w.symmetric) return w;
  const int r = e.r, k = e.k;
  static const bool timing = std::getenv("HP_PLAN_TIMING") != nullptr;
  auto t0 = Clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = Clock::now();
    std::fprintf(stderr, "[build_level %d] %s %.1f ms\n", l, what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const SamplingPlan plan = make_plan(e.tree, e.adj, l, SampleMode::kH1, r, cfg.seed, kForwardPhase);
  lap("make_plan");
  w.nc = plan.colors();
  std::vector<std::vector<int>> color_boxes(size_t(w.nc));
  w.pay_off.assign(size_t(w.nc) + 1, 0);
  for (int c = 0; c < w.nc; ++c) {
    for (auto [box, tag] : plan.matrices[size_t(c)].payload) {
      color_boxes[size_t(c)].push_back(box);
      for (std::int64_t q = 0; q < e.count(box); ++q) w.pay_pos.push_back(int(e.start(box) + q));
    }
    w.pay_off[size_t(c) + 1] = std::int64_t(w.pay_pos.size());
    w.fwd_cols += plan.matrices[size_t(c)].payload.empty() ? 0 : r;
  }
  // int8 K2 layout: per color, ceil(nnz_c / 32) K-steps and the payload boxes
  w.step_off.assign(size_t(w.nc) + 1, 0);
  w.pb_off.assign(size_t(w.nc) + 1, 0);
  for (int c = 0; c < w.nc; ++c) {
    const std::int64_t ns = (w.pay_off[size_t(c) + 1] - w.pay_off[size_t(c)] + 31) / 32;
    w.step_off[size_t(c) + 1] = w.step_off[size_t(c)] + ns;
    for (std::int64_t q = 0; q < ns; ++q) w.step_color.push_back(c);
    for (int b : color_boxes[size_t(c)]) w.pb_box.push_back(b);
    w.pb_off[size_t(c) + 1] = std::int64_t(w.pb_box.size());
  }
  const size_t np = ld.pairs.size();
  w.np = np;
  w.pcolor.resize(np);
  w.soff.assign(np + 1, 0);
  w.swap.resize(np);
  for (size_t p = 0; p < np; ++p) {
    w.pcolor[p] = plan.block_to_matrix.at(ld.pairs[p]);
    w.soff[p + 1] = w.soff[p] + std::int64_t(e.count(ld.pairs[p].first)) * 2 * r;
    w.swap[p] = pair_index(ld.pairs, ld.pairs[p].second, ld.pairs[p].first);
  }
  // K1: pos -> box, local rank
  w.pos_box.assign(size_t(e.n), -1);
  w.local.assign(size_t(e.n), 0);
  for (int b : e.tree.level_boxes(l)) {
    const int* lr = e.lay.local_flat.data() + e.lay.local_off[size_t(b)];
    for (int q = 0; q < e.count(b); ++q) {
      w.pos_box[size_t(e.start(b) + q)] = b;
      w.local[size_t(e.start(b) + q)] = lr[q];
    }
  }
  // K2: split the pairs into work-balanced contiguous ranges, one per shard
  // (DESIGN.md §7); inside a shard, the target rows of all pairs served by
  // one color are packed into full tiles, largest payload lists first.
  const int world = cfg.comm ? cfg.comm->world() : std::max(1, cfg.emulate_shards);
  std::vector<double> pair_work(np);
  for (size_t p = 0; p < np; ++p) {
    const std::int64_t nnz = w.pay_off[size_t(w.pcolor[p]) + 1] - w.pay_off[size_t(w.pcolor[p])];
    pair_work[p] = double(e.count(ld.pairs[p].first)) * double(nnz);
    w.evals += pair_work[p];
  }
  {
    // a valid H1 coloring never puts a row box into the payload serving it;
    // if it did, K2 would have to test i == j
    std::set<std::pair<int, int>> box_color;
    for (int c = 0; c < w.nc; ++c)
      for (int box : color_boxes[size_t(c)]) box_color.insert({box, c});
    for (size_t p = 0; p < np; ++p)
      if (box_color.count({ld.pairs[p].first, w.pcolor[p]})) w.k2_checked = true;
  }
  const auto bounds = partition_ranges(pair_work, world);
  w.seg.resize(size_t(world) + 1);
  for (int q = 0; q <= world; ++q) w.seg[size_t(q)] = w.soff[size_t(bounds[size_t(q)])];
  const int tile = k2_tile_rows(e.dop.symmetric ? 2 * r : r);
  w.k2.resize(size_t(world));
  std::vector<std::vector<int>> by_color(size_t(w.nc));
  for (int q = 0; q < world; ++q) {
    for (auto& v : by_color) v.clear();
    for (std::int64_t p = bounds[size_t(q)]; p < bounds[size_t(q) + 1]; ++p)
      by_color[size_t(w.pcolor[size_t(p)])].push_back(int(p));
    auto& tl = w.k2[size_t(q)];
    for (int c = 0; c < w.nc; ++c) {
      // whole tiles of big boxes run in place; their remainders and the small
      // boxes are packed through the row table
      const std::int64_t first = std::int64_t(w.rowtab.size());
      for (int p : by_color[size_t(c)]) {
        const int a = ld.pairs[size_t(p)].first;
        const int rows = e.count(a);
        const int full = rows / tile * tile;
        for (int t0 = 0; t0 < full; t0 += tile)
          tl.push_back(K2Task{w.soff[size_t(p)] + t0, tile, c, rows, int(e.start(a) + t0)});
        for (int i = full; i < rows; ++i)
          w.rowtab.push_back(K2Row{w.soff[size_t(p)] + i, int(e.start(a) + i), rows});
      }
      const std::int64_t last = std::int64_t(w.rowtab.size());
      for (std::int64_t t0 = first; t0 < last; t0 += tile)
        tl.push_back(K2Task{t0, int(std::min<std::int64_t>(tile, last - t0)), c, 0, 0});
    }
    std::stable_sort(tl.begin(), tl.end(), [&](const K2Task& x, const K2Task& y) {
      return w.pay_off[size_t(x.color) + 1] - w.pay_off[size_t(x.color)] >
             w.pay_off[size_t(y.color) + 1] - w.pay_off[size_t(y.color)];
    });
  }
  // K3 (prev_level = l - 1 >= 2)
  if (l - 1 >= 2) {
    std::vector<SampleBlock> blocks(np);
    for (size_t p = 0; p < np; ++p) blocks[p] = SampleBlock{ld.pairs[p].first, w.pcolor[p], w.soff[p]};
    lap("k2 tasks");
    w.peel = plan_peel(e, rep, blocks, color_boxes, l - 1, r, true);
    lap("plan_peel");
    w.has_peel = true;
  }
  // K5a middle = G'_a^T Y_p; K4 QR; K5b grams -- per shard, on the pairs it
  // owns (outputs by pair: U_p from Y_p, V_p from Z of swap(p))
  const int gld = 2 * r;
  {
    std::vector<double> w45(np);
    for (size_t p = 0; p < np; ++p)
      w45[p] = double(e.count(ld.pairs[p].first) + e.count(ld.pairs[p].second)) * double(r) * double(r);
    w.fb = partition_ranges(w45, world);
  }
  w.s45.resize(size_t(world));
  for (int q = 0; q < world; ++q) {
    LevelWork::Shard45& sh = w.s45[size_t(q)];
    sh.p0 = w.fb[size_t(q)];
    sh.p1 = w.fb[size_t(q) + 1];
    std::vector<GramReq> mid, gu, vg;
    std::vector<QrRequest> qr;
    for (std::int64_t p = sh.p0; p < sh.p1; ++p) {
      const auto [a, b] = ld.pairs[size_t(p)];
      const int rows = e.count(a), rows_b = e.count(b);
      const std::int64_t sp = w.swap[size_t(p)];  // block (b, a): its adjoint columns give V_p
      mid.push_back(GramReq{e.start(a) * gld + r, w.soff[size_t(p)], rows, gld, rows, 1, 0});
      gu.push_back(GramReq{e.start(a) * gld + r, ld.uoff[size_t(p)], rows, gld, rows, 1, 0});
      vg.push_back(GramReq{ld.voff[size_t(p)], e.start(b) * gld, rows_b, rows_b, gld, 0, 1});
      qr.push_back(QrRequest{w.soff[size_t(p)], ld.uoff[size_t(p)], rows, rows, int(p)});
      qr.push_back(QrRequest{w.soff[size_t(sp)] + std::int64_t(rows_b) * r, ld.voff[size_t(p)], rows_b, rows_b,
                             int(np + size_t(p))});
    }
    sh.g_mid = plan_gram(mid, r, r);
    sh.g_gpu = plan_gram(gu, r, k);
    sh.g_vg = plan_gram(vg, k, r);
    sh.qr = plan_qr(qr, r, k);
  }
  lap("plan_qr");
  return w;
}

struct LeafWork {
  int nc = 0;
  int w = 0;
  std::int64_t fwd_cols = 0;
  std::vector<std::int64_t> pay_off;
  std::vector<int> pay_box;
  std::vector<SampleTask> tasks;
  double evals = 0;
  bool has_peel = false;
  PeelPlan peel;
  std::vector<std::pair<int, int>> pairs;
  std::vector<std::int64_t> off;
  std::int64_t total = 0;
};

LeafWork build_leaf(const Engine& e, const H1Rep& rep, const PeelConfig& cfg) {
  LeafWork lw;
  const BoxTree& tree = e.tree;
  lw.w = tree.max_leaf_size();
  static const bool timing = std::getenv("HP_PLAN_TIMING") != nullptr;
  auto t0 = Clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = Clock::now();
    std::fprintf(stderr, "[build_leaf] %s %.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const SamplingPlan plan =
      make_plan(tree, e.adj, tree.depth(), SampleMode::kLeaf, lw.w, cfg.seed, kForwardPhase);
  lap("make_plan");
  lw.nc = plan.colors();
  std::vector<std::vector<int>> color_boxes(size_t(lw.nc));
  lw.pay_off.assign(size_t(lw.nc) + 1, 0);
  for (int c = 0; c < lw.nc; ++c) {
    for (auto [box, tag] : plan.matrices[size_t(c)].payload) {
      color_boxes[size_t(c)].push_back(box);
      lw.pay_box.push_back(box);
    }
    lw.pay_off[size_t(c) + 1] = std::int64_t(lw.pay_box.size());
    lw.fwd_cols += plan.matrices[size_t(c)].payload.empty() ? 0 : lw.w;
  }
  lw.pairs = dense_pairs(tree, e.adj);
  const size_t nd = lw.pairs.size();
  lw.off.resize(nd);
  std::vector<SampleBlock> blocks(nd);
  for (size_t p = 0; p < nd; ++p) {
    const auto [lam, mu] = lw.pairs[p];
    const int c = plan.block_to_matrix.at(lw.pairs[p]);
    const int rows = e.count(lam);
    lw.off[p] = lw.total;
    for (int t0 = 0; t0 < rows; t0 += kTile)
      lw.tasks.push_back(SampleTask{e.start(lam) + t0, lw.total + t0, std::min(kTile, rows - t0), c, rows, 0});
    blocks[p] = SampleBlock{lam, c, lw.total};
    std::int64_t nnz = 0;
    for (std::int64_t q = lw.pay_off[size_t(c)]; q < lw.pay_off[size_t(c) + 1]; ++q)
      nnz += e.count(lw.pay_box[size_t(q)]);
    lw.evals += double(rows) * double(nnz);
    lw.total += std::int64_t(rows) * lw.w;
  }
  lap("tasks");
  if (tree.depth() >= 2) {
    lw.peel = plan_peel(e, rep, blocks, color_boxes, tree.depth(), lw.w, false);
    lw.has_peel = true;
  }
  lap("plan_peel");
  return lw;
}

struct LevelTimers {
  Events apply, peel, mid, qr, bsolve;
};

/// One level's sampling stage (K1 payload + K2 apply), issued on the apply
/// stream one level ahead of the level's peel / QR / B work on the main
/// stream: K2 of level l + 1 depends only on its host plan, so it overlaps
/// the factorization of level l. Every buffer is allocated and freed on the
/// main stream `s`; the apply stream starts after `ready` (recorded on `s`
/// after the uploads) and the frees wait for `done`.
struct ApplyStage {
  cudaStream_t s = nullptr;
  cudaEvent_t ready = nullptr, done = nullptr;
  LevelWork w;
  std::unique_ptr<LevelTimers> tm;
  bool use_i8 = false;
  DevBuf<int> d_pos_box, d_local;
  DevBuf<K2Row> d_rowtab;
  DevBuf<std::int64_t> d_pay_off;
  DevBuf<int> d_pay_pos;
  DevBuf<double> samples, gcol, xcol;
  DevBuf<unsigned char> bdig;
  DevBuf<std::int64_t> d_step_off, d_pb_off;
  DevBuf<double> xstep;
  DevBuf<int> d_step_color, d_pb_box;
  std::vector<DevBuf<K2Task>> d_tasks;

  explicit ApplyStage(cudaStream_t st) : s(st) {
    HP_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    HP_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  }
  ApplyStage(const ApplyStage&) = delete;
  ApplyStage& operator=(const ApplyStage&) = delete;
  ~ApplyStage() {
    cudaStreamWaitEvent(s, done, 0);  // the members' frees (on s) follow the apply stream's use
    cudaEventDestroy(ready);
    cudaEventDestroy(done);
    reap_async(std::move(w));
  }
};

}  // namespace

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

void export_sizes(const BoxTree& tree, int rank, std::int64_t* factor_doubles,
                  std::int64_t* dense_doubles) {
  const AdjacencyInfo adj = adjacency(tree);
  std::int64_t f = 0, d = 0;
  for (int l = 2; l <= tree.depth(); ++l)
    for (auto [a, b] : admissible_pairs(tree, adj, l))
      f += std::int64_t(tree.box(a).points.size() + tree.box(b).points.size()) * rank +
           std::int64_t(rank) * rank;
  const std::int64_t w = tree.max_leaf_size();
  for (auto [lam, mu] : dense_pairs(tree, adj)) d += std::int64_t(tree.box(lam).points.size()) * w;
  if (factor_doubles) *factor_doubles = f;
  if (dense_doubles) *dense_doubles = d;
}

namespace {

// Copies finished parts of the representation to the caller's host arrays on
// a second stream, each after an event on the compute stream. Pinned
// destinations overlap the later levels; pageable ones are copied at the end.
class Exporter {
 public:
  Exporter(double* hf, double* hd, int device) : hf_(hf), hd_(hd) {
    if (!hf_ && !hd_) return;
    pinned_ = is_pinned(hf_) && is_pinned(hd_);
    if (pinned_) HP_CUDA(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking));
    (void)device;
  }
  ~Exporter() {
    if (xs_) {
      cudaStreamSynchronize(xs_);
      cudaStreamDestroy(xs_);
    }
    for (cudaEvent_t ev : events_) cudaEventDestroy(ev);
  }
  bool active() const { return hf_ || hd_; }
  // device [src, src + n) -> host dst once the work queued on s so far is done
  void copy(double* dst, const double* src, std::int64_t n, cudaStream_t s) {
    if (!dst || n <= 0) return;
    if (!pinned_) {
      deferred_.push_back({dst, src, n});
      return;
    }
    cudaEvent_t ev;
    HP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    events_.push_back(ev);
    HP_CUDA(cudaEventRecord(ev, s));
    HP_CUDA(cudaStreamWaitEvent(xs_, ev, 0));
    HP_CUDA(cudaMemcpyAsync(dst, src, size_t(n) * 8, cudaMemcpyDeviceToHost, xs_));
  }
  void finish(cudaStream_t s) {
    if (xs_) HP_CUDA(cudaStreamSynchronize(xs_));
    if (!deferred_.empty()) {
      HP_CUDA(cudaStreamSynchronize(s));
      for (const auto& d : deferred_)
        HP_CUDA(cudaMemcpy(d.dst, d.src, size_t(d.n) * 8, cudaMemcpyDeviceToHost));
      deferred_.clear();
    }
  }
  double* factors() const { return hf_; }
  double* dense() const { return hd_; }

 private:
  static bool is_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeHost;
  }
  struct Deferred {
    double* dst;
    const double* src;
    std::int64_t n;
  };
  double* hf_;
  double* hd_;
  bool pinned_ = false;
  cudaStream_t xs_ = nullptr;
  std::vector<cudaEvent_t> events_;
  std::vector<Deferred> deferred_;
};

}  // namespace

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
  const int r = config.sample_width();
  const int k = config.rank;
  if (2 * r > 160) throw std::invalid_argument("sample width k + p > 80 is not supported");

  DeviceGuard guard(op.device());
  const auto t_begin = Clock::now();
  auto adj = std::make_shared<const AdjacencyInfo>(adjacency(*tree));
  auto lay = std::make_shared<const TreeLayout>(tree_layout(*tree));

  // s: uploads, peel / QR / B and the leaf phase (high priority: it gates the
  // next level's stage); sa: K1 + K2 of the level ahead (ApplyStage)
  cudaStream_t s, sa;
  {
    int least = 0, greatest = 0;
    HP_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    static const int flip = std::getenv("HP_APPLY_PRIORITY") ? std::atoi(std::getenv("HP_APPLY_PRIORITY")) : 0;
    HP_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, flip == 1 ? least : greatest));
    HP_CUDA(cudaStreamCreateWithPriority(&sa, cudaStreamNonBlocking, flip == 1 ? greatest : least));
  }
  PeelResult result;
  auto rep = std::make_shared<H1Rep>();
  rep->tree = tree;
  rep->adj = adj;
  rep->layout = lay;
  rep->rank = k;
  rep->device = op.device();
  rep->levels.resize(size_t(tree->depth()) + 1);
  RunReport& report = result.report;
  int* h_ranks = nullptr;

  try {
    Exporter exporter(config.export_factors, config.export_dense, op.device());
    Events dev_span;  // a: first device work of this compress
    HP_CUDA(cudaEventRecord(dev_span.a, s));
    Engine e(*tree, *adj, *lay, op, s);
    StagingScope staging(s);  // uploads below stay asynchronous
    e.r = r;
    e.k = k;
    const Index n = tree->num_points();

    // Factor arena: U (|I_a| x k), V (|I_b| x k), B (k x k) per pair, all levels.
    std::int64_t ftotal = 0, rank_total = 0;
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
      rank_total += 2 * std::int64_t(np);
    }
    rep->factor_doubles = ftotal;
    // stream-ordered from the retained device pool: repeated compress() calls reuse the memory
    HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rep->d_factors), size_t(std::max<std::int64_t>(ftotal, 1)) * 8, s));
    h_ranks = static_cast<int*>(persistent_pinned(size_t(std::max<std::int64_t>(rank_total, 1)) * sizeof(int), 0));

    // Host plans of every level and of the leaf phase, built concurrently.
    std::vector<std::future<LevelWork>> futs(size_t(tree->depth()) + 1);
    for (int l = 2; l <= tree->depth(); ++l)
      futs[size_t(l)] = std::async(std::launch::async, build_level, std::cref(e), std::cref(*rep), l,
                                   std::cref(config));
    auto leaf_fut = std::async(std::launch::async, build_leaf, std::cref(e), std::cref(*rep),
                               std::cref(config));

    // Sharding: ranks launch K2/K6 for contiguous work-balanced
    // ranges and broadcast their rows; emulate_shards splits the launches the
    // same way inside one process (tests).
    const int world = config.comm ? config.comm->world() : std::max(1, config.emulate_shards);
    const int my_rank = config.comm ? config.comm->rank() : -1;
    auto shard_tasks = [&](const std::vector<SampleTask>& tasks, const std::vector<double>& work,
                           const std::vector<std::int64_t>& item_off, std::vector<std::int64_t>& seg) {
      const auto b = partition_ranges(work, world);
      seg.assign(size_t(world) + 1, 0);
      for (int q = 0; q <= world; ++q) seg[size_t(q)] = item_off[size_t(b[size_t(q)])];
      std::vector<std::vector<SampleTask>> lists(static_cast<size_t>(world));
      for (const SampleTask& t : tasks) {
        const int q = int(std::upper_bound(seg.begin(), seg.end(), t.out) - seg.begin()) - 1;
        lists[size_t(std::min(std::max(q, 0), world - 1))].push_back(t);
      }
      return lists;
    };

    const int gld = 2 * r;
    // payload Gaussians of two levels: K1 of level l + 1 (apply stream) runs
    // while level l's peel and B solve (main stream) still read its payloads
    DevBuf<double> gbuf[2] = {DevBuf<double>(size_t(n) * size_t(gld), s), DevBuf<double>(size_t(n) * size_t(gld), s)};
    std::vector<std::unique_ptr<LevelTimers>> timers(size_t(tree->depth()) + 1);
    std::vector<std::int64_t> rank_off(size_t(tree->depth()) + 1, 0);
    std::vector<double> evals(size_t(tree->depth()) + 1, 0.0), peel_flops(size_t(tree->depth()) + 1, 0.0);
    std::vector<int> colors(size_t(tree->depth()) + 1, 0), apply_path(size_t(tree->depth()) + 1, 0);
    std::vector<std::int64_t> fcols(size_t(tree->depth()) + 1, 0);
    std::int64_t roff = 0;
    int built = 1;

    std::vector<double> wait_ms(size_t(tree->depth()) + 1, 0.0);
    report.setup_ms = std::chrono::duration<double, std::milli>(Clock::now() - t_begin).count();

    // K1 + K2 of level l: uploads on s, launches on sa after `ready`
    auto issue_apply = [&](int l) {
      auto st = std::make_unique<ApplyStage>(s);
      const auto t_wait = Clock::now();
      st->w = futs[size_t(l)].get();
      wait_ms[size_t(l)] = std::chrono::duration<double, std::milli>(Clock::now() - t_wait).count();
      LevelWork& w = st->w;
      if (w.empty) return st;  // proj/src/peeling.cpp:221 (built_level not advanced)
      if (!w.symmetric) throw std::logic_error("asymmetric admissibility structure");
      const size_t np = w.np;
      st->tm = std::make_unique<LevelTimers>();
      LevelTimers* tm = st->tm.get();
      colors[size_t(l)] = w.nc;
      fcols[size_t(l)] = w.fwd_cols;
      evals[size_t(l)] = w.evals;
      peel_flops[size_t(l)] = w.peel.coeff_flops + w.peel.apply_flops;
      double* g = gbuf[l & 1].get();

      st->d_pos_box.upload(w.pos_box, s);
      st->d_local.upload(w.local, s);
      st->d_rowtab.upload(w.rowtab, s);
      st->d_pay_off.upload(w.pay_off, s);
      st->d_pay_pos.upload(w.pay_pos, s);
      st->samples.alloc(size_t(w.soff[np]), s);
      // payload rows and coordinates in color order (contiguous K2 chunks)
      const std::int64_t nnz = std::int64_t(w.pay_pos.size());
      st->gcol.alloc(size_t(nnz) * size_t(gld), s);
      st->xcol.alloc(op.kind() == kOpDense ? 1 : size_t(nnz) * size_t(op.dim()), s);
      const bool checked = w.k2_checked || e.has_dups;
      // int8 tensor-core K2 (k2_i8.cuh): on-the-fly symmetric kernels,
      // unchecked tiles, widths with the group split (r <= 48). At r = 64 the
      // column-split int8 kernel is no faster than DMMA (config 4 scaled:
      // 1.74 s both) and its sample error (5e-13) sits closest to the 1e-12
      // bar, so those widths keep FP64 DMMA.
      const bool use_i8 = op.kind() != kOpDense && op.symmetric() && !checked &&
                          k2i8::group_split(k2i8::padded_width(r)) && k2_mode() == 0 && k2_int8_enabled();
      st->use_i8 = use_i8;
      apply_path[size_t(l)] = use_i8 ? 1 : 0;
      std::int64_t half_stride = 0, tsteps = 0;
      if (use_i8) {
        tsteps = w.step_off.back();
        half_stride = tsteps * k2i8::b_step_bytes(k2i8::padded_width(r));
        st->bdig.alloc(size_t(std::max<std::int64_t>(2 * half_stride, 16)), s);  // same size in both layouts
        st->d_step_off.upload(w.step_off, s);
        st->d_step_color.upload(w.step_color, s);
        st->d_pb_off.upload(w.pb_off, s);
        st->d_pb_box.upload(w.pb_box, s);
        st->xstep.alloc(size_t(std::max<std::int64_t>(tsteps, 1)) * 32 * size_t(op.dim()), s);
        e.ensure_box_bbox();  // on s, before `ready`
      }
      st->d_tasks.reserve(w.k2.size());
      for (int sr = 0; sr < int(w.k2.size()); ++sr) {
        st->d_tasks.emplace_back();
        if (my_rank >= 0 && sr != my_rank) continue;
        st->d_tasks.back().upload(w.k2[size_t(sr)], s);
      }
      HP_CUDA(cudaEventRecord(st->ready, s));
      HP_CUDA(cudaStreamWaitEvent(sa, st->ready, 0));

      // K1 payload
      launch_payload_gaussian(g, gld, r, n, st->d_pos_box.get(), st->d_local.get(), config.seed, l, sa);
      // K2 apply (forward + adjoint samples of every pair's row block); each
      // shard launches its own tiles, then the shards' rows are broadcast
      HP_CUDA(cudaEventRecord(tm->apply.a, sa));
      launch_permute_rows(g, gld, 1, st->d_pay_pos.get(), nnz, gld, st->gcol.get(), gld, 1, sa);
      if (op.kind() != kOpDense)
        launch_permute_rows(e.dop.x, 1, n, st->d_pay_pos.get(), nnz, op.dim(), st->xcol.get(), 1, nnz, sa);
      if (use_i8) {
        // group split: the CTA pair adds two partial sums per sample element
        HP_CUDA(cudaMemsetAsync(st->samples.get(), 0, size_t(w.soff[np]) * sizeof(double), sa));
        k2i8::launch_payload_digits(st->gcol.get(), gld, r, st->d_pay_off.get(), st->d_step_off.get(),
                                    st->d_step_color.get(), tsteps, st->bdig.get(), half_stride, sa);
        k2i8::launch_step_coords(st->xcol.get(), nnz, op.dim(), st->d_pay_off.get(), st->d_step_off.get(),
                                 st->d_step_color.get(), tsteps, st->xstep.get(), sa);
      }
      for (int sr = 0; sr < int(w.k2.size()); ++sr) {
        if (my_rank >= 0 && sr != my_rank) continue;
        const K2Task* tasks = st->d_tasks[size_t(sr)].get();
        const int nt = int(w.k2[size_t(sr)].size());
        if (use_i8) {
          k2i8::launch_sample_apply_i8(e.dop, tasks, st->d_rowtab.get(), nt, st->d_pay_off.get(),
                                       st->d_step_off.get(), st->xstep.get(), st->d_pb_off.get(),
                                       st->d_pb_box.get(), e.d_box_bbox.get(), st->bdig.get(), half_stride, r,
                                       st->samples.get(), sa);
        } else if (op.symmetric()) {
          launch_sample_apply(e.dop, false, tasks, st->d_rowtab.get(), nt, st->d_pay_off.get(),
                              st->d_pay_pos.get(), st->gcol.get(), gld, 0, 2 * r, st->xcol.get(), nnz,
                              st->samples.get(), 0, checked, sa);
        } else {
          launch_sample_apply(e.dop, false, tasks, st->d_rowtab.get(), nt, st->d_pay_off.get(),
                              st->d_pay_pos.get(), st->gcol.get(), gld, 0, r, st->xcol.get(), nnz,
                              st->samples.get(), 0, checked, sa);
          launch_sample_apply(e.dop, true, tasks, st->d_rowtab.get(), nt, st->d_pay_off.get(),
                              st->d_pay_pos.get(), st->gcol.get(), gld, r, r, st->xcol.get(), nnz,
                              st->samples.get(), r, checked, sa);
        }
      }
      HP_CUDA(cudaEventRecord(tm->apply.b, sa));
      HP_CUDA(cudaEventRecord(st->done, sa));
      return st;
    };
    // HP_SERIAL_LEVELS=1: no overlap (each level's apply after the previous
    // level's factorization), so K2 can be timed alone (bench.py)
    // Overlap only pays when K2 runs on the int8 tensor cores: the FP64 DMMA
    // K2 and the peel / QR / B kernels share the FP64 datapath, and there the
    // overlapped order measured slower (config 5 scaled 3.12 s vs 3.02 s
    // serialized; config 4 scaled 3.767 vs 3.757 s).
    const char* serial_env = std::getenv("HP_SERIAL_LEVELS");
    const bool k2_on_int8 = op.kind() != kOpDense && op.symmetric() &&
                            k2i8::group_split(k2i8::padded_width(r)) && k2_mode() == 0 && k2_int8_enabled();
    const bool serial = serial_env ? std::atoi(serial_env) != 0 : !k2_on_int8;
    std::unique_ptr<ApplyStage> next;
    if (tree->depth() >= 2) next = issue_apply(2);
    for (int l = 2; l <= tree->depth(); ++l) {
      std::unique_ptr<ApplyStage> cur = std::move(next);
      // issue the next level's sampling ahead of this level's factorization
      // (waiting for its host plan here is fine: the host runs far ahead of
      // the device, and H1 level plans take <= 1.5 s even at config 4 full)
      if (!serial && l + 1 <= tree->depth()) next = issue_apply(l + 1);
      LevelWork& w = cur->w;
      if (!w.empty) {
        if (l - 1 >= 2 && l - 1 > built)
          throw std::runtime_error("h1 apply: representation incomplete for level " + std::to_string(l - 1));
        auto& ld = rep->levels[size_t(l)];
        const size_t np = w.np;
        LevelTimers* tm = cur->tm.get();
        double* g = gbuf[l & 1].get();
        double* samples = cur->samples.get();
        HP_CUDA(cudaStreamWaitEvent(s, cur->done, 0));
        if (config.comm) config.comm->broadcast_segments(samples, w.seg, s);

        // K3 peel
        HP_CUDA(cudaEventRecord(tm->peel.a, s));
        if (w.has_peel) run_peel(w.peel, e, *rep, g, gld, r, false, samples, r, s);
        HP_CUDA(cudaEventRecord(tm->peel.b, s));

        if (config.capture_samples) {
          HP_CUDA(cudaStreamSynchronize(s));
          std::vector<Matrix> cap;
          for (size_t p = 0; p < np; ++p) {
            const int rows = e.count(ld.pairs[p].first);
            Matrix m(rows, 2 * r);
            HP_CUDA(cudaMemcpy(m.data(), samples + w.soff[p], size_t(rows) * 2 * r * 8,
                               cudaMemcpyDeviceToHost));
            cap.push_back(std::move(m));
          }
          rep->captured[l] = std::move(cap);
        }

        // K5a: middle = G'_a^T Y_p before the QR overwrites Y; K4 QR; K5b grams
        // and B -- each shard on its own pairs, then the shards' factor and
        // rank segments are broadcast
        DevBuf<double> middle(np * size_t(r) * size_t(r), s), gpu(np * size_t(r) * size_t(k), s),
            vg(np * size_t(k) * size_t(r), s);
        DevBuf<int> d_ranks(2 * np, s);
        DevBuf<std::int64_t> d_boff;
        d_boff.upload(ld.boff, s);
        auto mine = [&](int sr) { return my_rank < 0 || sr == my_rank; };
        HP_CUDA(cudaEventRecord(tm->mid.a, s));
        for (int sr = 0; sr < int(w.s45.size()); ++sr)
          if (mine(sr))
            run_gram(w.s45[size_t(sr)].g_mid, g, samples, middle.get() + w.s45[size_t(sr)].p0 * r * r, s);
        HP_CUDA(cudaEventRecord(tm->mid.b, s));
        HP_CUDA(cudaEventRecord(tm->qr.a, s));
        for (int sr = 0; sr < int(w.s45.size()); ++sr)
          if (mine(sr)) run_qr(w.s45[size_t(sr)].qr, samples, rep->d_factors, d_ranks.get(), r, k, s);
        HP_CUDA(cudaEventRecord(tm->qr.b, s));
        HP_CUDA(cudaEventRecord(tm->bsolve.a, s));
        for (int sr = 0; sr < int(w.s45.size()); ++sr) {
          if (!mine(sr)) continue;
          const LevelWork::Shard45& sh = w.s45[size_t(sr)];
          run_gram(sh.g_gpu, g, rep->d_factors, gpu.get() + sh.p0 * r * k, s);
          run_gram(sh.g_vg, rep->d_factors, g, vg.get() + sh.p0 * k * r, s);
          launch_bsolve(int(sh.p1 - sh.p0), gpu.get() + sh.p0 * r * k, middle.get() + sh.p0 * r * r,
                        vg.get() + sh.p0 * k * r, r, k, kPinvCutoff, d_boff.get() + sh.p0, rep->d_factors, s);
        }
        if (config.comm && np > 0) {
          const std::int64_t fend = ld.boff[np - 1] + std::int64_t(k) * k;
          std::vector<std::int64_t> fseg(w.fb.size()), useg(w.fb.size()), vseg(w.fb.size());
          for (size_t q = 0; q < w.fb.size(); ++q) {
            const std::int64_t p = w.fb[q];
            fseg[q] = p < std::int64_t(np) ? ld.uoff[size_t(p)] : fend;
            useg[q] = p;
            vseg[q] = std::int64_t(np) + p;
          }
          config.comm->broadcast_segments(rep->d_factors, fseg, s);
          config.comm->broadcast_segments_i32(d_ranks.get(), useg, s);
          config.comm->broadcast_segments_i32(d_ranks.get(), vseg, s);
        }
        HP_CUDA(cudaEventRecord(tm->bsolve.b, s));
        HP_CUDA(cudaMemcpyAsync(h_ranks + roff, d_ranks.get(), 2 * np * sizeof(int), cudaMemcpyDeviceToHost, s));
        rank_off[size_t(l)] = roff;
        roff += 2 * std::int64_t(np);
        timers[size_t(l)] = std::move(cur->tm);
        if (exporter.active() && np > 0) {  // this level's U, V, B are final
          const std::int64_t f0 = ld.uoff[0], f1 = ld.boff[np - 1] + std::int64_t(k) * k;
          exporter.copy(exporter.factors() ? exporter.factors() + f0 : nullptr, rep->d_factors + f0, f1 - f0, s);
        }
        built = l;
      }
      cur.reset();  // frees (on s) after the apply stream's use of its buffers
      if (serial && l + 1 <= tree->depth()) next = issue_apply(l + 1);  // waits for this level on s
    }
    rep->built_level = tree->depth();

    // ------------------------------------------------------------- leaf phase
    const auto t_leaf_wait = Clock::now();
    LeafWork lw = leaf_fut.get();
    const double leaf_wait_ms = std::chrono::duration<double, std::milli>(Clock::now() - t_leaf_wait).count();
    rep->dense.pairs = lw.pairs;
    rep->dense.off = lw.off;
    rep->dense_doubles = lw.total;
    HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rep->d_dense), size_t(std::max<std::int64_t>(lw.total, 1)) * 8, s));
    Events leaf_apply, leaf_peel;
    {
      std::vector<double> dwork(lw.pairs.size());
      std::vector<std::int64_t> doff(lw.off);
      doff.push_back(lw.total);
      for (size_t p = 0; p < lw.pairs.size(); ++p)
        dwork[p] = double(e.count(lw.pairs[p].first)) * double(lw.w);
      std::vector<std::int64_t> seg;
      const auto lists = shard_tasks(lw.tasks, dwork, doff, seg);
      DevBuf<std::int64_t> d_pay_off;
      d_pay_off.upload(lw.pay_off, s);
      DevBuf<int> d_pay_box;
      d_pay_box.upload(lw.pay_box, s);
      HP_CUDA(cudaEventRecord(leaf_apply.a, s));
      for (int sr = 0; sr < int(lists.size()); ++sr) {
        if (my_rank >= 0 && sr != my_rank) continue;
        DevBuf<SampleTask> d_tasks;
        d_tasks.upload(lists[size_t(sr)], s);
        launch_identity_apply(e.dop, d_tasks.get(), int(lists[size_t(sr)].size()), d_pay_off.get(),
                              d_pay_box.get(), e.d_box_start.get(), e.d_box_count.get(), lw.w,
                              rep->d_dense, s);
      }
      HP_CUDA(cudaEventRecord(leaf_apply.b, s));
      HP_CUDA(cudaEventRecord(leaf_peel.a, s));
      if (lw.has_peel) {
        if (my_rank >= 0) {
          // peel this rank's dense blocks only, then share them
          PeelPlan mine = lw.peel;
          const std::int64_t lo = seg[size_t(my_rank)], hi = seg[size_t(my_rank) + 1];
          mine.tasks_fwd.erase(std::remove_if(mine.tasks_fwd.begin(), mine.tasks_fwd.end(),
                                              [&](const PeelTask& t) { return t.out < lo || t.out >= hi; }),
                               mine.tasks_fwd.end());
          run_peel(mine, e, *rep, nullptr, 0, lw.w, true, rep->d_dense, 0, s);
        } else {
          run_peel(lw.peel, e, *rep, nullptr, 0, lw.w, true, rep->d_dense, 0, s);
        }
      }
      if (config.comm) config.comm->broadcast_segments(rep->d_dense, seg, s);
      HP_CUDA(cudaEventRecord(leaf_peel.b, s));
      if (exporter.active()) exporter.copy(exporter.dense(), rep->d_dense, lw.total, s);
    }
    exporter.finish(s);
    HP_CUDA(cudaStreamSynchronize(s));
    if (config.capture_samples) {
      for (size_t p = 0; p < lw.pairs.size(); ++p) {
        const int rows = e.count(lw.pairs[p].first);
        Matrix m(rows, lw.w);
        HP_CUDA(cudaMemcpy(m.data(), rep->d_dense + lw.off[p], size_t(rows) * lw.w * 8, cudaMemcpyDeviceToHost));
        rep->captured_leaf.push_back(std::move(m));
      }
    }
    rep->dense_ready = true;
    static const bool drv_timing = std::getenv("HP_DRIVER_TIMING") != nullptr;
    const auto t_report = Clock::now();

    // ------------------------------------------------------------- report
    double blackbox_ms = 0.0;
    float fstart = 0.f;
    for (int l = 2; l <= tree->depth(); ++l) {
      auto& ld = rep->levels[size_t(l)];
      if (!timers[size_t(l)]) continue;
      const size_t np = ld.pairs.size();
      for (size_t p = 0; p < np; ++p) {
        ld.ku[p] = h_ranks[rank_off[size_t(l)] + std::int64_t(p)];
        ld.kv[p] = h_ranks[rank_off[size_t(l)] + std::int64_t(np + p)];
      }
    }
    for (int l = 2; l <= tree->depth(); ++l) {
      const auto& tm = timers[size_t(l)];
      if (!tm) continue;
      const auto& ld = rep->levels[size_t(l)];
      PhaseReport ph;
      ph.phase = "h1";
      ph.level = l;
      ph.colors = colors[size_t(l)];
      ph.apply_path = apply_path[size_t(l)];
      ph.forward_cols = fcols[size_t(l)];
      ph.adjoint_cols = fcols[size_t(l)];
      ph.kernel_evals = evals[size_t(l)];
      ph.apply_flops = evals[size_t(l)] * 2.0 * 2.0 * r;
      ph.peel_flops = peel_flops[size_t(l)];
      ph.apply_ms = tm->apply.ms();
      ph.peel_ms = tm->peel.ms();
      ph.qr_ms = tm->qr.ms();
      ph.bsolve_ms = tm->bsolve.ms() + tm->mid.ms();
      ph.wall_ms_total = ph.apply_ms + ph.peel_ms + ph.qr_ms + ph.bsolve_ms;
      ph.wall_ms_net = ph.wall_ms_total - ph.apply_ms;
      ph.host_wait_ms = wait_ms[size_t(l)];
      HP_CUDA(cudaEventElapsedTime(&fstart, dev_span.a, tm->apply.a));
      ph.start_ms = fstart;
      blackbox_ms += ph.apply_ms;
      if (l - 1 >= 2) ph.net_flops += 2 * std::int64_t(ph.colors) * truncated_apply_flops(*rep, l - 1, r, e);
      // QR (flops.hpp:18-20) and the B solve (peeling.cpp:262-268)
      for (size_t p = 0; p < ld.pairs.size(); ++p) {
        const std::int64_t ma = e.count(ld.pairs[p].first), mb = e.count(ld.pairs[p].second);
        const std::int64_t ku = ld.ku[p], kv = ld.kv[p];
        ph.net_flops += 2 * ma * r * r + 2 * mb * r * r;
        ph.qr_flops += 2.0 * double(ma) * r * r + 2.0 * double(mb) * r * r;
        ph.net_flops += gemm_flops(r, r, ma) + gemm_flops(r, ku, ma) + gemm_flops(kv, r, mb);
        if (ku > 0) ph.net_flops += svd_flops(r, ku) + gemm_flops(ku, r, r);
        if (kv > 0) ph.net_flops += svd_flops(r, kv) + gemm_flops(kv, ku, r);
      }
      report.phases.push_back(ph);
    }
    {
      PhaseReport ph;
      ph.phase = "leaf";
      ph.level = tree->depth();
      ph.colors = lw.nc;
      ph.forward_cols = lw.fwd_cols;
      ph.kernel_evals = lw.evals;
      ph.peel_flops = lw.peel.coeff_flops + lw.peel.apply_flops;
      ph.apply_ms = leaf_apply.ms();
      ph.peel_ms = leaf_peel.ms();
      ph.wall_ms_total = ph.apply_ms + ph.peel_ms;
      ph.wall_ms_net = ph.peel_ms;
      ph.host_wait_ms = leaf_wait_ms;
      HP_CUDA(cudaEventElapsedTime(&fstart, dev_span.a, leaf_apply.a));
      ph.start_ms = fstart;
      blackbox_ms += ph.apply_ms;
      if (tree->depth() >= 2) ph.net_flops += std::int64_t(lw.nc) * truncated_apply_flops(*rep, tree->depth(), lw.w, e);
      report.phases.push_back(ph);
    }
    for (const PhaseReport& p : report.phases) {
      report.forward_cols += p.forward_cols;
      report.adjoint_cols += p.adjoint_cols;
      report.net_flops += p.net_flops;
      if (p.phase != "leaf") report.max_sampling_colors = std::max(report.max_sampling_colors, p.colors);
    }
    report.wall_s_total = std::chrono::duration<double>(Clock::now() - t_begin).count();
    if (drv_timing)
      std::fprintf(stderr, "[driver] device drained at %.1f ms, report %.1f ms, total %.1f ms\n",
                   std::chrono::duration<double, std::milli>(t_report - t_begin).count(),
                   std::chrono::duration<double, std::milli>(Clock::now() - t_report).count(),
                   report.wall_s_total * 1e3);
    report.wall_s_net = report.wall_s_total - blackbox_ms * 1e-3;
    // the leaf plan's host vectors (hundreds of MB on adaptive trees) are
    // released on a background thread: freeing them here (munmap across the
    // planning threads' pages) had put 0-0.6 s of host time on the return path
    reap_async(std::move(lw));
  } catch (...) {
    cudaStreamSynchronize(sa);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(sa);
    cudaStreamDestroy(s);
    throw;
  }
  HP_CUDA(cudaStreamSynchronize(s));
  cudaStreamDestroy(sa);
  cudaStreamDestroy(s);
  result.rep = rep;
  return result;
}

}  // namespace hpeel
