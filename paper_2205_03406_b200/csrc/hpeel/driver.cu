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
//
// Multi-GPU (shard.hpp): owner-computes. Each rank computes the
// samples of the pairs whose row box it owns, peels them with the factors it
// holds, and keeps only the factors of pairs touching its boxes; per level two
// point-to-point exchanges ship V (to the row owner) and U, B (to the column
// owner) of the cut-crossing pairs. The levels above the cut are replicated.
// The black box itself may be the caller's callback (the reference's virtual
// LinearOperator::apply): then each color's dense test matrix is realized on
// the device, handed to the callback, and the sample rows read back.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <future>
#include <mutex>
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
// product (proj/src/hmatrix.cpp:86-100), over the pairs this rank counts.
std::int64_t truncated_apply_flops(const H1Rep& rep, int level, std::int64_t w, const Engine& e) {
  std::int64_t f = 0;
  for (int l = 2; l <= std::min<int>(level, int(rep.levels.size()) - 1); ++l) {
    const auto& ld = rep.levels[size_t(l)];
    for (size_t p = 0; p < ld.pairs.size(); ++p) {
      if (!rep.counts_pair(l, int(p))) continue;
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

// ------------------------------------------------------------------ arena

/// Factor-arena and dense-block layout of one rank: offsets of the pairs it
/// holds (-1 elsewhere). Replicated levels come first and are laid out the
/// same on every rank; dense blocks are compact |I_lam| x |I_mu|
/// (D = Y(I_lam, 0:|I_mu|), proj/src/peeling.cpp:513-517).
struct ArenaLayout {
  std::vector<H1Rep::LevelData> levels;
  std::int64_t factors = 0;
  std::vector<std::pair<int, int>> dense_pairs;
  std::vector<std::int64_t> dense_off;
  std::int64_t dense = 0;
};

ArenaLayout arena_layout(const BoxTree& tree, const AdjacencyInfo& adj, const Ownership& o, int k) {
  ArenaLayout L;
  L.levels.resize(size_t(tree.depth()) + 1);
  auto cnt = [&](int b) { return std::int64_t(tree.box(b).points.size()); };
  for (int l = 2; l <= tree.depth(); ++l) {
    auto& ld = L.levels[size_t(l)];
    ld.pairs = admissible_pairs(tree, adj, l);
    const size_t np = ld.pairs.size();
    ld.uoff.assign(np, -1);
    ld.voff.assign(np, -1);
    ld.boff.assign(np, -1);
    ld.ku.assign(np, 0);
    ld.kv.assign(np, 0);
    for (size_t p = 0; p < np; ++p) {
      const auto [a, b] = ld.pairs[p];
      if (!(o.replicated(l) || o.mine(a) || o.mine(b))) continue;
      ld.uoff[p] = L.factors;
      L.factors += cnt(a) * k;
      ld.voff[p] = L.factors;
      L.factors += cnt(b) * k;
      ld.boff[p] = L.factors;
      L.factors += std::int64_t(k) * k;
    }
  }
  L.dense_pairs = dense_pairs(tree, adj);
  L.dense_off.assign(L.dense_pairs.size(), -1);
  for (size_t p = 0; p < L.dense_pairs.size(); ++p) {
    const auto [lam, mu] = L.dense_pairs[p];
    if (!o.mine(lam)) continue;
    L.dense_off[p] = L.dense;
    L.dense += cnt(lam) * cnt(mu);
  }
  return L;
}

// ------------------------------------------------------------------ exchanges

/// One all-to-all-v of factor segments and rank slots between the owners of
/// cut-crossing pairs. Phase 1: V_q (computed by the column owner) to the row
/// owner; phase 2: U_q and B_q (row owner) to the column owner. Message i -> j
/// carries the pairs q in ascending order, so both ends enumerate it alike.
struct Exchange {
  std::vector<CopySeg> pack, unpack;      // arena -> send buffer, recv buffer -> arena
  std::vector<std::int64_t> soff, roff;   // world + 1 (doubles)
  std::vector<int> rs_idx, rr_idx;        // rank slots gathered / scattered
  std::vector<std::int64_t> rsoff, rroff; // world + 1 (ints)
};

Exchange make_exchange(const H1Rep::LevelData& ld, const Ownership& o, const BoxTree& tree, int k, bool phase1) {
  Exchange X;
  const int W = o.world, me = o.rank;
  const size_t np = ld.pairs.size();
  auto cnt = [&](int b) { return std::int64_t(tree.box(b).points.size()); };
  auto ends = [&](size_t q, int& from, int& to) {
    const int oa = o.of(ld.pairs[q].first), ob = o.of(ld.pairs[q].second);
    from = phase1 ? ob : oa;
    to = phase1 ? oa : ob;
  };
  auto parts = [&](size_t q, auto&& fn) {
    if (phase1) {
      fn(ld.voff[q], cnt(ld.pairs[q].second) * k);
    } else {
      fn(ld.uoff[q], cnt(ld.pairs[q].first) * k);
      fn(ld.boff[q], std::int64_t(k) * k);
    }
  };
  auto slot = [&](size_t q) { return int(phase1 ? np + q : q); };
  X.soff.assign(size_t(W) + 1, 0);
  X.roff.assign(size_t(W) + 1, 0);
  X.rsoff.assign(size_t(W) + 1, 0);
  X.rroff.assign(size_t(W) + 1, 0);
  std::int64_t cur = 0, rcur = 0;
  for (int j = 0; j < W; ++j) {
    X.soff[size_t(j)] = cur;
    X.rsoff[size_t(j)] = std::int64_t(X.rs_idx.size());
    X.roff[size_t(j)] = rcur;
    X.rroff[size_t(j)] = std::int64_t(X.rr_idx.size());
    if (j == me) continue;
    for (size_t q = 0; q < np; ++q) {
      int from = 0, to = 0;
      ends(q, from, to);
      if (from == me && to == j) {
        parts(q, [&](std::int64_t off, std::int64_t len) {
          X.pack.push_back(CopySeg{off, cur, len});
          cur += len;
        });
        X.rs_idx.push_back(slot(q));
      } else if (from == j && to == me) {
        parts(q, [&](std::int64_t off, std::int64_t len) {
          X.unpack.push_back(CopySeg{rcur, off, len});
          rcur += len;
        });
        X.rr_idx.push_back(slot(q));
      }
    }
  }
  X.soff[size_t(W)] = cur;
  X.roff[size_t(W)] = rcur;
  X.rsoff[size_t(W)] = std::int64_t(X.rs_idx.size());
  X.rroff[size_t(W)] = std::int64_t(X.rr_idx.size());
  return X;
}

double run_exchange(const Exchange& X, Comm& comm, double* arena, int* d_ranks, cudaStream_t s) {
  DevBuf<double> send(size_t(X.soff.back()), s), recv(size_t(X.roff.back()), s);
  DevBuf<CopySeg> dp, du;
  dp.upload(X.pack, s);
  du.upload(X.unpack, s);
  launch_copy_segments(arena, dp.get(), int(X.pack.size()), send.get(), s);
  comm.exchange(send.get(), X.soff, recv.get(), X.roff, s);
  launch_copy_segments(recv.get(), du.get(), int(X.unpack.size()), arena, s);
  DevBuf<int> si, ri, isend(X.rs_idx.size(), s), irecv(X.rr_idx.size(), s);
  si.upload(X.rs_idx, s);
  ri.upload(X.rr_idx, s);
  launch_move_i32(d_ranks, si.get(), std::int64_t(X.rs_idx.size()), isend.get(), nullptr, s);
  comm.exchange_i32(isend.get(), X.rsoff, irecv.get(), X.rroff, s);
  launch_move_i32(irecv.get(), nullptr, std::int64_t(X.rr_idx.size()), d_ranks, ri.get(), s);
  return double(X.soff.back()) * 8.0 + double(X.rs_idx.size()) * 4.0;
}

// ------------------------------------------------------------------ level plan

struct LevelWork {
  int level = 0;
  bool empty = true;
  bool symmetric = true;
  bool replicated = false;   // above the cut: every rank holds every pair
  int nc = 0;
  std::int64_t fwd_cols = 0;
  size_t np = 0;
  std::vector<int> pcolor, swap;           // per pair
  std::vector<int> own;                    // sample blocks on this rank (pair indices)
  std::vector<int> own_idx;                // per pair: index in `own` or -1
  std::vector<std::int64_t> soff;          // per own block (+ total)
  std::vector<std::int64_t> pay_off;
  std::vector<int> pay_pos;
  std::vector<std::int64_t> step_off;      // int8 K2: 32-row K-steps per color (prefix)
  std::vector<int> step_color;             // color of every K-step
  std::vector<std::int64_t> pb_off;        // payload boxes per color (prefix)
  std::vector<int> pb_box;
  std::vector<int> pos_box, local;
  std::vector<K2Row> rowtab;               // K2 rows of this rank's tiles
  std::vector<K2Task> k2;                  // K2 tiles this rank launches
  std::vector<std::int64_t> seg;           // replicated: rank q computes samples [seg[q], seg[q+1])
  bool k2_checked = false;                 // some row box is in its own color's payload
  double evals = 0;
  bool has_peel = false;
  PeelPlan peel;
  // callback black box: per color, the own sample rows it serves
  std::vector<std::int64_t> cb_off;
  std::vector<GatherRow> cb_rows;
  // K4/K5 on this rank: QR requests (U and V), grams and B solves of `solve`
  QrPlan qr;
  GramPlan g_mid, g_gpu, g_vg;
  std::vector<int> solve;
  std::vector<std::int64_t> solve_boff;
  // replicated: factor / rank broadcast segments (rank q solves pairs [fb[q], fb[q+1]))
  std::vector<std::int64_t> fb, fseg, useg, vseg;
  // owned: crossing-pair exchanges (V to the row owner, then U / B back)
  Exchange x1, x2;
};

LevelWork build_level(const Engine& e, const H1Rep& rep, int l, const PeelConfig& cfg, const Ownership& o) {
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
  w.replicated = o.replicated(l);
  const int world = o.world, me = o.rank;
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
  const SamplingPlan plan = make_plan(e.tree, e.adj, l, SampleMode::kH1, r, cfg.seed, kForwardPhase,
                                      cfg.strategy == ColoringStrategy::kFallbackPattern);
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
  w.swap.resize(np);
  for (size_t p = 0; p < np; ++p) {
    w.pcolor[p] = plan.block_to_matrix.at(ld.pairs[p]);
    w.swap[p] = pair_index(ld.pairs, ld.pairs[p].second, ld.pairs[p].first);
  }
  // sample blocks computed here: every pair on a replicated level, else the
  // pairs whose row box this rank owns
  w.own_idx.assign(np, -1);
  for (size_t p = 0; p < np; ++p)
    if (w.replicated || o.mine(ld.pairs[p].first)) {
      w.own_idx[p] = int(w.own.size());
      w.own.push_back(int(p));
    }
  w.soff.assign(w.own.size() + 1, 0);
  for (size_t i = 0; i < w.own.size(); ++i)
    w.soff[i + 1] = w.soff[i] + std::int64_t(e.count(ld.pairs[size_t(w.own[i])].first)) * 2 * r;
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
  std::vector<double> pair_work(np);
  for (size_t p = 0; p < np; ++p) {
    const std::int64_t nnz = w.pay_off[size_t(w.pcolor[p]) + 1] - w.pay_off[size_t(w.pcolor[p])];
    pair_work[p] = double(e.count(ld.pairs[p].first)) * double(nnz);
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
  // K2 pairs this rank applies: its own blocks, or on a replicated level its
  // work-balanced contiguous range (the rows are then broadcast)
  std::int64_t k2_p0 = 0, k2_p1 = std::int64_t(np);
  if (w.replicated) {
    const auto bounds = partition_ranges(pair_work, world);
    w.seg.resize(size_t(world) + 1);
    for (int q = 0; q <= world; ++q) w.seg[size_t(q)] = w.soff[size_t(bounds[size_t(q)])];
    k2_p0 = bounds[size_t(me)];
    k2_p1 = bounds[size_t(me) + 1];
  }
  for (size_t i = 0; i < w.own.size(); ++i) {
    const int p = w.own[i];
    if (p >= k2_p0 && p < k2_p1) w.evals += pair_work[size_t(p)];
  }
  if (e.op.is_callback()) {
    // rows of the blocks each color serves, read back from the callback's Y
    std::vector<std::vector<int>> by_color(size_t(w.nc));
    for (std::int64_t p = k2_p0; p < k2_p1; ++p)
      if (w.own_idx[size_t(p)] >= 0) by_color[size_t(w.pcolor[size_t(p)])].push_back(int(p));
    w.cb_off.assign(size_t(w.nc) + 1, 0);
    for (int c = 0; c < w.nc; ++c) {
      for (int p : by_color[size_t(c)]) {
        const int a = ld.pairs[size_t(p)].first, rows = e.count(a);
        const std::int64_t base = w.soff[size_t(w.own_idx[size_t(p)])];
        for (int i = 0; i < rows; ++i) w.cb_rows.push_back(GatherRow{base + i, int(e.start(a) + i), rows, r, 0});
      }
      w.cb_off[size_t(c) + 1] = std::int64_t(w.cb_rows.size());
    }
  } else {
    // inside this rank's range, the target rows of all pairs served by one
    // color are packed into full tiles, largest payload lists first
    const int tile = k2_tile_rows(e.dop.symmetric ? 2 * r : r);
    std::vector<std::vector<int>> by_color(size_t(w.nc));
    for (std::int64_t p = k2_p0; p < k2_p1; ++p)
      if (w.own_idx[size_t(p)] >= 0) by_color[size_t(w.pcolor[size_t(p)])].push_back(int(p));
    auto& tl = w.k2;
    for (int c = 0; c < w.nc; ++c) {
      // whole tiles of big boxes run in place; their remainders and the small
      // boxes are packed through the row table
      const std::int64_t first = std::int64_t(w.rowtab.size());
      for (int p : by_color[size_t(c)]) {
        const int a = ld.pairs[size_t(p)].first;
        const int rows = e.count(a);
        const int full = rows / tile * tile;
        const std::int64_t base = w.soff[size_t(w.own_idx[size_t(p)])];
        for (int t0r = 0; t0r < full; t0r += tile)
          tl.push_back(K2Task{base + t0r, tile, c, rows, int(e.start(a) + t0r)});
        for (int i = full; i < rows; ++i) w.rowtab.push_back(K2Row{base + i, int(e.start(a) + i), rows});
      }
      const std::int64_t last = std::int64_t(w.rowtab.size());
      for (std::int64_t t0r = first; t0r < last; t0r += tile)
        tl.push_back(K2Task{t0r, int(std::min<std::int64_t>(tile, last - t0r)), c, 0, 0});
    }
    std::stable_sort(tl.begin(), tl.end(), [&](const K2Task& x, const K2Task& y) {
      return w.pay_off[size_t(x.color) + 1] - w.pay_off[size_t(x.color)] >
             w.pay_off[size_t(y.color) + 1] - w.pay_off[size_t(y.color)];
    });
  }
  lap("k2 tasks");
  // K3 (prev_level = l - 1 >= 2) on this rank's blocks
  if (l - 1 >= 2) {
    std::vector<SampleBlock> blocks(w.own.size());
    for (size_t i = 0; i < w.own.size(); ++i)
      blocks[i] = SampleBlock{ld.pairs[size_t(w.own[i])].first, w.pcolor[size_t(w.own[i])], w.soff[i]};
    w.peel = plan_peel(e, rep, blocks, color_boxes, l - 1, r, true);
    lap("plan_peel");
    w.has_peel = true;
  }
  // K5a middle = G'_a^T Y_p; K4 QR; K5b grams -- on the pairs this rank
  // solves (outputs by pair: U_p from Y_p, V from the adjoint columns)
  const int gld = 2 * r;
  std::vector<GramReq> mid, gu, vg;
  std::vector<QrRequest> qr;
  if (w.replicated) {
    std::vector<double> w45(np);
    for (size_t p = 0; p < np; ++p)
      w45[p] = double(e.count(ld.pairs[p].first) + e.count(ld.pairs[p].second)) * double(r) * double(r);
    w.fb = partition_ranges(w45, world);
    for (std::int64_t p = w.fb[size_t(me)]; p < w.fb[size_t(me) + 1]; ++p) w.solve.push_back(int(p));
    for (int p : w.solve) {
      const auto [a, b] = ld.pairs[size_t(p)];
      const int rows_b = e.count(b);
      const std::int64_t sp = w.swap[size_t(p)];  // block (b, a): its adjoint columns give V_p
      qr.push_back(QrRequest{w.soff[size_t(p)], ld.uoff[size_t(p)], e.count(a), e.count(a), p});
      qr.push_back(QrRequest{w.soff[size_t(sp)] + std::int64_t(rows_b) * r, ld.voff[size_t(p)], rows_b, rows_b,
                             int(np) + p});
    }
    const std::int64_t fend = ld.boff[np - 1] + std::int64_t(k) * k;
    w.fseg.resize(size_t(world) + 1);
    w.useg.resize(size_t(world) + 1);
    w.vseg.resize(size_t(world) + 1);
    for (int q = 0; q <= world; ++q) {
      const std::int64_t p = w.fb[size_t(q)];
      w.fseg[size_t(q)] = p < std::int64_t(np) ? ld.uoff[size_t(p)] : fend;
      w.useg[size_t(q)] = p;
      w.vseg[size_t(q)] = std::int64_t(np) + p;
    }
  } else {
    w.solve = w.own;
    for (size_t i = 0; i < w.own.size(); ++i) {
      const int p = w.own[i];
      const int a = ld.pairs[size_t(p)].first;
      const int sp = w.swap[size_t(p)];  // pair (b, a): V of it comes from the adjoint columns of block p
      qr.push_back(QrRequest{w.soff[i], ld.uoff[size_t(p)], e.count(a), e.count(a), p});
      qr.push_back(QrRequest{w.soff[i] + std::int64_t(e.count(a)) * r, ld.voff[size_t(sp)], e.count(a), e.count(a),
                             int(np) + sp});
    }
    if (world > 1) {
      w.x1 = make_exchange(ld, o, e.tree, k, true);
      w.x2 = make_exchange(ld, o, e.tree, k, false);
    }
  }
  for (int p : w.solve) {
    const auto [a, b] = ld.pairs[size_t(p)];
    const int rows = e.count(a), rows_b = e.count(b);
    const std::int64_t so = w.soff[size_t(w.own_idx[size_t(p)])];
    mid.push_back(GramReq{e.start(a) * gld + r, so, rows, gld, rows, 1, 0});
    gu.push_back(GramReq{e.start(a) * gld + r, ld.uoff[size_t(p)], rows, gld, rows, 1, 0});
    vg.push_back(GramReq{ld.voff[size_t(p)], e.start(b) * gld, rows_b, rows_b, gld, 0, 1});
    w.solve_boff.push_back(ld.boff[size_t(p)]);
  }
  w.g_mid = plan_gram(mid, r, r);
  w.g_gpu = plan_gram(gu, r, k);
  w.g_vg = plan_gram(vg, k, r);
  w.qr = plan_qr(qr, r, k);
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
  std::vector<std::int64_t> cb_off;   // callback: per color, rows of this rank's dense blocks
  std::vector<GatherRow> cb_rows;
};

LeafWork build_leaf(const Engine& e, const H1Rep& rep, const PeelConfig& cfg, const Ownership& o) {
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
      make_plan(tree, e.adj, tree.depth(), SampleMode::kLeaf, lw.w, cfg.seed, kForwardPhase,
                cfg.strategy == ColoringStrategy::kFallbackPattern);
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
  const auto& pairs = rep.dense.pairs;
  std::vector<SampleBlock> blocks;
  std::vector<std::vector<GatherRow>> cb(size_t(lw.nc));
  for (size_t p = 0; p < pairs.size(); ++p) {
    const std::int64_t off = rep.dense.off[p];
    if (off < 0) continue;
    const auto [lam, mu] = pairs[p];
    const int c = plan.block_to_matrix.at(pairs[p]);
    const int rows = e.count(lam), cols = e.count(mu);
    for (int r0 = 0; r0 < rows; r0 += kTile)
      lw.tasks.push_back(SampleTask{e.start(lam) + r0, off + r0, std::min(kTile, rows - r0), c, rows, cols});
    blocks.push_back(SampleBlock{lam, c, off, cols});
    if (e.op.is_callback())
      for (int i = 0; i < rows; ++i) cb[size_t(c)].push_back(GatherRow{off + i, int(e.start(lam) + i), rows, cols, 0});
    std::int64_t nnz = 0;
    for (std::int64_t q = lw.pay_off[size_t(c)]; q < lw.pay_off[size_t(c) + 1]; ++q)
      nnz += e.count(lw.pay_box[size_t(q)]);
    lw.evals += double(rows) * double(nnz);
  }
  if (e.op.is_callback()) {
    lw.cb_off.assign(size_t(lw.nc) + 1, 0);
    for (int c = 0; c < lw.nc; ++c) {
      lw.cb_rows.insert(lw.cb_rows.end(), cb[size_t(c)].begin(), cb[size_t(c)].end());
      lw.cb_off[size_t(c) + 1] = std::int64_t(lw.cb_rows.size());
    }
  }
  (void)o;
  lap("tasks");
  if (tree.depth() >= 2) {
    // the leaf plan is the last one the device needs but the largest one:
    // its peel plan runs on several threads
    const int threads = int(std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2)));
    lw.peel = plan_peel_parallel(e, rep, blocks, color_boxes, tree.depth(), lw.w, false, threads);
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
  DevBuf<K2Task> d_tasks;
  DevBuf<GatherRow> d_cb_rows;
  DevBuf<double> omega, yprod;

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
                  std::int64_t* dense_doubles, int world, int shard) {
  const AdjacencyInfo adj = adjacency(tree);
  const TreeLayout lay = tree_layout(tree);
  const Ownership o = make_ownership(tree, lay, world, shard);
  const ArenaLayout L = arena_layout(tree, adj, o, rank);
  if (factor_doubles) *factor_doubles = L.factors;
  if (dense_doubles) *dense_doubles = L.dense;
}

void shard_memory_plan(const BoxTree& tree, int rank, int oversample, int world, double* out) {
  const AdjacencyInfo adj = adjacency(tree);
  const TreeLayout lay = tree_layout(tree);
  const std::int64_t n = tree.num_points();
  const int r = rank + oversample;
  for (int g = 0; g < world; ++g) {
    const Ownership o = make_ownership(tree, lay, world, g);
    const ArenaLayout L = arena_layout(tree, adj, o, rank);
    // largest level: own sample blocks (|I_a| x 2r) + the apply stage's
    // color-ordered payload / coordinate / digit copies (~ N rows each) and
    // the two payload buffers (N x 2r)
    double level_max = 0.0;
    // levels overlap (two stages alive) only on the int8 K2 path (r <= 48)
    const double stages = k2i8::group_split(k2i8::padded_width(r)) ? 2.0 : 1.0;
    for (int l = 2; l <= tree.depth(); ++l) {
      const auto& ld = L.levels[size_t(l)];
      double rows = 0.0, solve = 0.0;
      for (auto [a, b] : ld.pairs)
        if (o.replicated(l) || o.mine(a)) {
          rows += double(tree.box(a).points.size());
          solve += 1.0;
        }
      if (o.replicated(l)) solve /= world;
      const double samples = rows * 2 * r * 8.0;
      const double stage = double(n) * (2 * r * 8.0 + 3 * 8.0 + 7.0 * k2i8::padded_width(r) / 2.0);
      // grams (middle, G'^T U, V^T G) and their row-chunk partials
      const double grams = solve * (double(r) * r + 2.0 * r * rank) * 8.0 * 2.0;
      level_max = std::max(level_max, stages * (samples + stage) + grams);
    }
    const double factors = double(L.factors) * 8.0, dense = double(L.dense) * 8.0;
    const double fixed = 2.0 * double(n) * 2 * r * 8.0 + double(n) * 4 * 8.0;  // payload buffers, coordinates
    out[g * 4 + 0] = factors;
    out[g * 4 + 1] = dense;
    out[g * 4 + 2] = level_max;
    out[g * 4 + 3] = factors + dense + level_max + fixed;
  }
}

void shard_exchange_counts(const BoxTree& tree, int rank, int world, int shard, int level, int phase,
                           std::int64_t* send, std::int64_t* recv) {
  if (level < 2 || level > tree.depth()) throw std::invalid_argument("level out of range");
  const AdjacencyInfo adj = adjacency(tree);
  const TreeLayout lay = tree_layout(tree);
  const Ownership o = make_ownership(tree, lay, world, shard);
  const ArenaLayout L = arena_layout(tree, adj, o, rank);
  const auto& ld = L.levels[size_t(level)];
  for (int j = 0; j < world; ++j) send[j] = recv[j] = 0;
  if (world == 1 || o.replicated(level) || ld.pairs.empty()) return;
  const Exchange X = make_exchange(ld, o, tree, rank, phase == 1);
  for (int j = 0; j < world; ++j) {
    send[j] = X.soff[size_t(j) + 1] - X.soff[size_t(j)];
    recv[j] = X.roff[size_t(j) + 1] - X.roff[size_t(j)];
  }
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

/// Memory high-water of this thread's compress (RunReport::peak_device_bytes).
class TrackScope {
 public:
  TrackScope() : prev_(MemTracker::current()) { MemTracker::current() = &t_; }
  ~TrackScope() { MemTracker::current() = prev_; }
  MemTracker& get() { return t_; }

 private:
  MemTracker t_;
  MemTracker* prev_;
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
  if (config.strategy == ColoringStrategy::kFallbackPattern && !tree->is_fully_populated())
    throw std::invalid_argument("pattern test matrices require a fully populated uniform tree");
  if (op.kind() != kOpDense && !op.is_callback() && op.dim() != tree->dim())
    throw std::invalid_argument("operator and tree dimensions differ");
  if (config.comm && config.comm->device() != op.device())
    throw std::invalid_argument("communicator and operator on different devices");
  const int r = config.sample_width();
  const int k = config.rank;
  if (2 * r > 160) throw std::invalid_argument("sample width k + p > 80 is not supported");
  if (k > 64) throw std::invalid_argument("rank k > 64 is not supported");

  DeviceGuard guard(op.device());
  TrackScope track;
  const auto t_begin = Clock::now();
  auto adj = std::make_shared<const AdjacencyInfo>(adjacency(*tree));
  auto lay = std::make_shared<const TreeLayout>(tree_layout(*tree));
  const int world = config.comm ? config.comm->world() : 1;
  const int my_rank = config.comm ? config.comm->rank() : 0;
  const Ownership own = make_ownership(*tree, *lay, world, my_rank);

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
  rep->world = world;
  rep->shard_rank = my_rank;
  if (world > 1) rep->box_owner = own.owner;
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

    // Factor arena: U (|I_a| x k), V (|I_b| x k), B (k x k) per held pair.
    {
      ArenaLayout L = arena_layout(*tree, *adj, own, k);
      rep->levels = std::move(L.levels);
      rep->factor_doubles = L.factors;
      rep->dense.pairs = std::move(L.dense_pairs);
      rep->dense.off = std::move(L.dense_off);
      rep->dense_doubles = L.dense;
    }
    std::int64_t rank_total = 0;
    for (int l = 2; l <= tree->depth(); ++l) rank_total += 2 * std::int64_t(rep->levels[size_t(l)].pairs.size());
    // stream-ordered from the retained device pool: repeated compress() calls reuse the memory
    HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rep->d_factors),
                            size_t(std::max<std::int64_t>(rep->factor_doubles, 1)) * 8, s));
    MemTracker::add(std::max<std::int64_t>(rep->factor_doubles, 1) * 8);
    h_ranks = static_cast<int*>(persistent_pinned(size_t(std::max<std::int64_t>(rank_total, 1)) * sizeof(int), 0));

    // Host plans of every level and of the leaf phase, built concurrently.
    // (the leaf plan is the longest -- its DSatur colors the densest graph -- so it starts first)
    auto leaf_fut = std::async(std::launch::async, build_leaf, std::cref(e), std::cref(*rep), std::cref(config),
                               std::cref(own));
    std::vector<std::future<LevelWork>> futs(size_t(tree->depth()) + 1);
    for (int l = 2; l <= tree->depth(); ++l)
      futs[size_t(l)] = std::async(std::launch::async, build_level, std::cref(e), std::cref(*rep), l,
                                   std::cref(config), std::cref(own));

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

    const bool int8_ok = op.kind() != kOpDense && !op.is_callback() && op.symmetric() &&
                         k2i8::group_split(k2i8::padded_width(r)) && k2_mode() == 0 && k2_int8_enabled();

    // K1 + K2 of level l: uploads on s, launches on sa after `ready`
    auto issue_apply = [&](int l) {
      auto st = std::make_unique<ApplyStage>(s);
      const auto t_wait = Clock::now();
      st->w = futs[size_t(l)].get();
      wait_ms[size_t(l)] = std::chrono::duration<double, std::milli>(Clock::now() - t_wait).count();
      LevelWork& w = st->w;
      if (w.empty) return st;  // proj/src/peeling.cpp:221 (built_level not advanced)
      if (!w.symmetric) throw std::logic_error("asymmetric admissibility structure");
      st->tm = std::make_unique<LevelTimers>();
      LevelTimers* tm = st->tm.get();
      colors[size_t(l)] = w.nc;
      fcols[size_t(l)] = w.fwd_cols;
      evals[size_t(l)] = w.evals;
      peel_flops[size_t(l)] = w.peel.coeff_flops + w.peel.apply_flops;
      double* g = gbuf[l & 1].get();

      st->d_pos_box.upload(w.pos_box, s);
      st->d_local.upload(w.local, s);
      st->d_pay_off.upload(w.pay_off, s);
      st->d_pay_pos.upload(w.pay_pos, s);
      st->samples.alloc(size_t(w.soff.back()), s);
      const std::int64_t nnz = std::int64_t(w.pay_pos.size());
      if (op.is_callback()) {
        st->d_cb_rows.upload(w.cb_rows, s);
        st->omega.alloc(size_t(n) * size_t(r), s);
        st->yprod.alloc(size_t(n) * size_t(r), s);
        HP_CUDA(cudaEventRecord(st->ready, s));
        HP_CUDA(cudaStreamWaitEvent(sa, st->ready, 0));
        launch_payload_gaussian(g, gld, r, n, st->d_pos_box.get(), st->d_local.get(), config.seed, l, sa);
        HP_CUDA(cudaEventRecord(tm->apply.a, sa));
        // residual_samples (proj/src/peeling.cpp:165-177): per color, realize
        // the dense test matrix, apply the black box, keep the rows read back
        for (int side = 0; side < 2; ++side) {
          for (int c = 0; c < w.nc; ++c) {
            const std::int64_t q0 = w.pay_off[size_t(c)], q1 = w.pay_off[size_t(c) + 1];
            if (q1 == q0) continue;  // empty payload: no apply (peeling.cpp:166)
            HP_CUDA(cudaMemsetAsync(st->omega.get(), 0, size_t(n) * size_t(r) * 8, sa));
            launch_scatter_payload(g, gld, side * r, r, st->d_pay_pos.get() + q0, q1 - q0, e.d_perm.get(),
                                   st->omega.get(), n, sa);
            op.call(side == 1, st->omega.get(), r, st->yprod.get(), sa);
            launch_gather_sample_rows(st->yprod.get(), n, e.d_perm.get(), st->d_cb_rows.get() + w.cb_off[size_t(c)],
                                      w.cb_off[size_t(c) + 1] - w.cb_off[size_t(c)], r, st->samples.get(),
                                      side * r, sa);
          }
        }
        HP_CUDA(cudaEventRecord(tm->apply.b, sa));
        HP_CUDA(cudaEventRecord(st->done, sa));
        return st;
      }
      st->d_rowtab.upload(w.rowtab, s);
      // payload rows and coordinates in color order (contiguous K2 chunks)
      st->gcol.alloc(size_t(nnz) * size_t(gld), s);
      st->xcol.alloc(op.kind() == kOpDense ? 1 : size_t(nnz) * size_t(op.dim()), s);
      const bool checked = w.k2_checked || e.has_dups;
      // int8 tensor-core K2 (k2_i8.cuh): on-the-fly symmetric kernels,
      // unchecked tiles, widths with the group split (r <= 48). At r = 64 the
      // column-split int8 kernel is no faster than DMMA (config 4 scaled:
      // 1.74 s both) and its sample error (5e-13) sits closest to the 1e-12
      // bar, so those widths keep FP64 DMMA.
      const bool use_i8 = int8_ok && !checked;
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
      st->d_tasks.upload(w.k2, s);
      HP_CUDA(cudaEventRecord(st->ready, s));
      HP_CUDA(cudaStreamWaitEvent(sa, st->ready, 0));

      // K1 payload
      launch_payload_gaussian(g, gld, r, n, st->d_pos_box.get(), st->d_local.get(), config.seed, l, sa);
      // K2 apply (forward + adjoint samples of this rank's row blocks)
      HP_CUDA(cudaEventRecord(tm->apply.a, sa));
      launch_permute_rows(g, gld, 1, st->d_pay_pos.get(), nnz, gld, st->gcol.get(), gld, 1, sa);
      if (op.kind() != kOpDense)
        launch_permute_rows(e.dop.x, 1, n, st->d_pay_pos.get(), nnz, op.dim(), st->xcol.get(), 1, nnz, sa);
      if (use_i8) {
        // group split: the CTA pair adds two partial sums per sample element
        HP_CUDA(cudaMemsetAsync(st->samples.get(), 0, size_t(w.soff.back()) * sizeof(double), sa));
        k2i8::launch_payload_digits(st->gcol.get(), gld, r, st->d_pay_off.get(), st->d_step_off.get(),
                                    st->d_step_color.get(), tsteps, st->bdig.get(), half_stride, sa);
        k2i8::launch_step_coords(st->xcol.get(), nnz, op.dim(), st->d_pay_off.get(), st->d_step_off.get(),
                                 st->d_step_color.get(), tsteps, st->xstep.get(), sa);
      }
      const K2Task* tasks = st->d_tasks.get();
      const int nt = int(w.k2.size());
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
      HP_CUDA(cudaEventRecord(tm->apply.b, sa));
      HP_CUDA(cudaEventRecord(st->done, sa));
      return st;
    };
    // HP_SERIAL_LEVELS=1: no overlap (each level's apply after the previous
    // level's factorization), so K2 can be timed alone (bench.py)
    // Overlap only pays when K2 runs on the int8 tensor cores: the FP64 DMMA
    // K2 and the peel / QR / B kernels share the FP64 datapath, and there the
    // overlapped order measured slower (config 5 scaled 3.12 s vs 3.02 s
    // serialized; config 4 scaled 3.767 vs 3.757 s). A callback black box
    // runs serialized (the caller's apply is synchronous).
    const char* serial_env = std::getenv("HP_SERIAL_LEVELS");
    const bool serial = op.is_callback() || (serial_env ? std::atoi(serial_env) != 0 : !int8_ok);
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
        if (w.replicated) {
          config.comm->broadcast_segments(samples, w.seg, s);
          report.exchange_bytes += double(w.seg[size_t(my_rank) + 1] - w.seg[size_t(my_rank)]) * 8.0 * (world - 1);
        }

        auto capture = [&](std::map<int, std::vector<Matrix>>& into) {
          HP_CUDA(cudaStreamSynchronize(s));
          std::vector<Matrix> cap(np);
          for (size_t i = 0; i < w.own.size(); ++i) {
            const int p = w.own[i];
            const int rows = e.count(ld.pairs[size_t(p)].first);
            Matrix m(rows, 2 * r);
            HP_CUDA(cudaMemcpy(m.data(), samples + w.soff[i], size_t(rows) * 2 * r * 8, cudaMemcpyDeviceToHost));
            cap[size_t(p)] = std::move(m);
          }
          into[l] = std::move(cap);
        };
        if (config.capture_samples) capture(rep->captured_raw);

        // K3 peel
        HP_CUDA(cudaEventRecord(tm->peel.a, s));
        if (w.has_peel) run_peel(w.peel, e, *rep, g, gld, r, false, samples, r, s);
        HP_CUDA(cudaEventRecord(tm->peel.b, s));

        if (config.capture_samples) capture(rep->captured);

        // K5a: middle = G'_a^T Y_p before the QR overwrites Y; K4 QR; K5b grams
        // and B (DESIGN.md §7 for the sharded variants)
        const size_t ns = w.solve.size();
        DevBuf<double> middle(ns * size_t(r) * size_t(r), s), gpu(ns * size_t(r) * size_t(k), s),
            vg(ns * size_t(k) * size_t(r), s);
        DevBuf<int> d_ranks(2 * np, s);
        DevBuf<std::int64_t> d_boff;
        d_boff.upload(w.solve_boff, s);
        HP_CUDA(cudaEventRecord(tm->mid.a, s));
        run_gram(w.g_mid, g, samples, middle.get(), s);
        HP_CUDA(cudaEventRecord(tm->mid.b, s));
        HP_CUDA(cudaEventRecord(tm->qr.a, s));
        run_qr(w.qr, samples, rep->d_factors, d_ranks.get(), r, k, s);
        HP_CUDA(cudaEventRecord(tm->qr.b, s));
        HP_CUDA(cudaEventRecord(tm->bsolve.a, s));
        if (!w.replicated && world > 1)  // V of crossing pairs to their row owner
          report.exchange_bytes += run_exchange(w.x1, *config.comm, rep->d_factors, d_ranks.get(), s);
        run_gram(w.g_gpu, g, rep->d_factors, gpu.get(), s);
        run_gram(w.g_vg, rep->d_factors, g, vg.get(), s);
        launch_bsolve(int(ns), gpu.get(), middle.get(), vg.get(), r, k, kPinvCutoff, d_boff.get(), rep->d_factors, s);
        if (w.replicated) {
          config.comm->broadcast_segments(rep->d_factors, w.fseg, s);
          config.comm->broadcast_segments_i32(d_ranks.get(), w.useg, s);
          config.comm->broadcast_segments_i32(d_ranks.get(), w.vseg, s);
          report.exchange_bytes += double(w.fseg[size_t(my_rank) + 1] - w.fseg[size_t(my_rank)]) * 8.0 * (world - 1);
        } else if (world > 1) {  // U and B of crossing pairs to their column owner
          report.exchange_bytes += run_exchange(w.x2, *config.comm, rep->d_factors, d_ranks.get(), s);
        }
        HP_CUDA(cudaEventRecord(tm->bsolve.b, s));
        HP_CUDA(cudaMemcpyAsync(h_ranks + roff, d_ranks.get(), 2 * np * sizeof(int), cudaMemcpyDeviceToHost, s));
        rank_off[size_t(l)] = roff;
        roff += 2 * std::int64_t(np);
        timers[size_t(l)] = std::move(cur->tm);
        if (exporter.active()) {  // this level's U, V, B are final
          std::int64_t f0 = -1, f1 = -1;
          for (size_t p = 0; p < np; ++p)
            if (ld.uoff[p] >= 0) {
              if (f0 < 0) f0 = ld.uoff[p];
              f1 = ld.boff[p] + std::int64_t(k) * k;
            }
          if (f0 >= 0)
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
    HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rep->d_dense),
                            size_t(std::max<std::int64_t>(rep->dense_doubles, 1)) * 8, s));
    MemTracker::add(std::max<std::int64_t>(rep->dense_doubles, 1) * 8);
    Events leaf_apply, leaf_peel;
    {
      DevBuf<std::int64_t> d_pay_off;
      d_pay_off.upload(lw.pay_off, s);
      DevBuf<int> d_pay_box;
      d_pay_box.upload(lw.pay_box, s);
      DevBuf<SampleTask> d_tasks;
      d_tasks.upload(lw.tasks, s);
      HP_CUDA(cudaEventRecord(leaf_apply.a, s));
      if (op.is_callback()) {
        // extract_leaf (proj/src/peeling.cpp:490-524): identity probes per color
        DevBuf<GatherRow> d_rows;
        d_rows.upload(lw.cb_rows, s);
        DevBuf<double> om(size_t(n) * size_t(lw.w), s), yp(size_t(n) * size_t(lw.w), s);
        for (int c = 0; c < lw.nc; ++c) {
          const std::int64_t q0 = lw.pay_off[size_t(c)], q1 = lw.pay_off[size_t(c) + 1];
          if (q1 == q0) continue;
          HP_CUDA(cudaMemsetAsync(om.get(), 0, size_t(n) * size_t(lw.w) * 8, s));
          launch_scatter_identity(d_pay_box.get() + q0, int(q1 - q0), e.d_box_start.get(), e.d_box_count.get(),
                                  e.d_perm.get(), lw.w, om.get(), n, s);
          op.call(false, om.get(), lw.w, yp.get(), s);
          launch_gather_sample_rows(yp.get(), n, e.d_perm.get(), d_rows.get() + lw.cb_off[size_t(c)],
                                    lw.cb_off[size_t(c) + 1] - lw.cb_off[size_t(c)], lw.w, rep->d_dense, 0, s);
        }
      } else {
        launch_identity_apply(e.dop, d_tasks.get(), int(lw.tasks.size()), d_pay_off.get(), d_pay_box.get(),
                              e.d_box_start.get(), e.d_box_count.get(), lw.w, rep->d_dense, s);
      }
      HP_CUDA(cudaEventRecord(leaf_apply.b, s));
      HP_CUDA(cudaEventRecord(leaf_peel.a, s));
      if (lw.has_peel) run_peel(lw.peel, e, *rep, nullptr, 0, lw.w, true, rep->d_dense, 0, s);
      HP_CUDA(cudaEventRecord(leaf_peel.b, s));
      if (exporter.active()) exporter.copy(exporter.dense(), rep->d_dense, rep->dense_doubles, s);
    }
    exporter.finish(s);
    HP_CUDA(cudaStreamSynchronize(s));
    if (config.capture_samples) {
      rep->captured_leaf.assign(rep->dense.pairs.size(), Matrix());
      for (size_t p = 0; p < rep->dense.pairs.size(); ++p) {
        if (rep->dense.off[p] < 0) continue;
        const int rows = e.count(rep->dense.pairs[p].first), cols = e.count(rep->dense.pairs[p].second);
        Matrix m(rows, cols);
        HP_CUDA(cudaMemcpy(m.data(), rep->d_dense + rep->dense.off[p], size_t(rows) * cols * 8,
                           cudaMemcpyDeviceToHost));
        rep->captured_leaf[p] = std::move(m);
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
        if (ld.uoff[p] < 0) continue;
        ld.ku[p] = h_ranks[rank_off[size_t(l)] + std::int64_t(p)];
        ld.kv[p] = h_ranks[rank_off[size_t(l)] + std::int64_t(np + p)];
        // qr_orthonormal's check (proj/src/linalg.cpp:59), reported by K4 as rank -1
        if (ld.ku[p] < 0 || ld.kv[p] < 0) throw std::invalid_argument("non-finite matrix in qr");
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
        if (!rep->counts_pair(l, int(p))) continue;
        const std::int64_t ma = e.count(ld.pairs[p].first), mb = e.count(ld.pairs[p].second);
        const std::int64_t ku = ld.ku[p], kv = ld.kv[p];
        ph.net_flops += 2 * ma * r * r + 2 * mb * r * r;
        ph.qr_flops += 2.0 * double(ma) * r * r + 2.0 * double(mb) * r * r;
        std::int64_t bf = gemm_flops(r, r, ma) + gemm_flops(r, ku, ma) + gemm_flops(kv, r, mb);
        if (ku > 0) bf += svd_flops(r, ku) + gemm_flops(ku, r, r);
        if (kv > 0) bf += svd_flops(r, kv) + gemm_flops(kv, ku, r);
        ph.net_flops += bf;
        ph.bsolve_flops += double(bf);
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
  report.peak_device_bytes = double(track.get().peak);
  cudaStreamDestroy(sa);
  cudaStreamDestroy(s);
  result.rep = rep;
  return result;
}

std::vector<PeelResult> compress_group(const DeviceOperator& op, std::shared_ptr<const BoxTree> tree,
                                       const PeelConfig& config, int world) {
  if (world < 1) throw std::invalid_argument("world size must be >= 1");
  if (config.comm) throw std::invalid_argument("compress_group builds its own communicators");
  auto group = std::make_shared<LocalGroup>(world);
  std::vector<PeelResult> out(static_cast<size_t>(world));
  std::exception_ptr first_err;
  std::mutex err_mu;
  std::vector<std::thread> threads;
  for (int g = 0; g < world; ++g)
    threads.emplace_back([&, g] {
      try {
        LocalComm comm(group, g, op.device());
        PeelConfig cfg = config;
        cfg.comm = &comm;
        out[size_t(g)] = compress(op, tree, cfg);
        // keep the communicator's events alive until every rank is done
        group->barrier();
      } catch (...) {
        {
          // the first failure is the cause; peers then fail in the aborted barrier
          std::lock_guard<std::mutex> lock(err_mu);
          if (!first_err) first_err = std::current_exception();
        }
        group->abort();
      }
    });
  for (auto& t : threads) t.join();
  if (first_err) std::rethrow_exception(first_err);
  return out;
}

}  // namespace hpeel
