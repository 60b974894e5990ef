// Engine and batched task builders (see engine.cuh).
#include "engine.cuh"
#include "k2_i8.cuh"

#include <mutex>
#include <thread>

#include "shard.hpp"

#include <algorithm>
#include <cstdlib>
#include <string>
#include <map>
#include <limits>
#include <unordered_map>

namespace hpeel::detail {

namespace {
std::mutex& pool_mutex() {
  static std::mutex m;
  return m;
}
std::vector<std::pair<char*, size_t>>& pool() {
  static std::vector<std::pair<char*, size_t>> p;
  return p;
}
}  // namespace

void retain_default_pool(int dev) {
  static std::mutex mu;
  static std::vector<char> done;
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0) return;
  if (size_t(dev) >= done.size()) done.resize(size_t(dev) + 1, 0);
  if (done[size_t(dev)]) return;
  cudaMemPool_t pool;
  HP_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  std::uint64_t thr = ~std::uint64_t(0);
  HP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done[size_t(dev)] = 1;
}

PinnedStaging*& PinnedStaging::current() {
  thread_local PinnedStaging* cur = nullptr;
  return cur;
}

void* PinnedStaging::take(size_t bytes) {
  bytes = (bytes + 255) / 256 * 256;
  for (Chunk& c : chunks_)
    if (c.size - c.used >= bytes) {
      void* p = c.p + c.used;
      c.used += bytes;
      return p;
    }
  {
    std::lock_guard<std::mutex> lock(pool_mutex());
    auto& pl = pool();
    for (size_t i = 0; i < pl.size(); ++i)
      if (pl[i].second >= bytes) {
        chunks_.push_back({pl[i].first, pl[i].second, bytes});
        pl.erase(pl.begin() + std::ptrdiff_t(i));
        return chunks_.back().p;
      }
  }
  const size_t size = std::max<size_t>(bytes, size_t(64) << 20);
  char* p = nullptr;
  HP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), size));
  chunks_.push_back({p, size, bytes});
  return p;
}

void* persistent_pinned(size_t bytes, int slot) {
  // grow-only, per thread: cudaMallocHost / cudaFreeHost on every compress()
  // serialized the return path behind the process's memory-map lock
  struct Buf {
    void* p = nullptr;
    size_t n = 0;
    ~Buf() {
      if (p) cudaFreeHost(p);
    }
  };
  thread_local Buf bufs[4];
  Buf& b = bufs[slot];
  if (b.n < bytes) {
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    HP_CUDA(cudaMallocHost(&b.p, bytes));
    b.n = bytes;
  }
  return b.p;
}

void PinnedStaging::release_to_pool() {
  std::lock_guard<std::mutex> lock(pool_mutex());
  for (const Chunk& c : chunks_) pool().push_back({c.p, c.size});
  chunks_.clear();
}

void Engine::ensure_box_bbox() {
  if (d_box_bbox.get() || op.kind() == kOpDense) return;
  const int nb = tree.num_boxes();
  d_box_bbox.alloc(size_t(nb) * 2 * size_t(op.dim()), s);
  k2i8::launch_box_bbox(xt.get(), n, op.dim(), d_box_start.get(), d_box_count.get(), nb, d_box_bbox.get(), s);
}

Engine::Engine(const BoxTree& t, const AdjacencyInfo& a, const TreeLayout& l,
               const DeviceOperator& o, cudaStream_t st)
    : tree(t), adj(a), lay(l), op(o), s(st) {
  n = tree.num_points();
  d_perm.upload(lay.perm, s);
  d_inv.upload(lay.inv, s);
  dop.kind = op.kind();
  dop.dim = op.dim();
  dop.n = n;
  dop.param = op.param();
  dop.symmetric = op.symmetric() ? 1 : 0;
  dop.ltab = log_table_device(op.device());
  if (op.kind() == kOpDense) {
    DevBuf<double> tmp(size_t(n) * size_t(n), s);
    at.alloc(size_t(n) * size_t(n), s);
    // rows then columns: at[s + t n] = a[perm[s] + perm[t] n]
    launch_permute_rows(op.device_matrix(), 1, n, d_perm.get(), n, int(n), tmp.get(), 1, n, s);
    launch_permute_rows(tmp.get(), n, 1, d_perm.get(), n, int(n), at.get(), n, 1, s);
    dop.a = at.get();
  } else if (op.kind() != kOpCallback) {
    xt.alloc(size_t(op.dim()) * size_t(n), s);
    launch_permute_rows(op.device_points(), 1, n, d_perm.get(), n, op.dim(), xt.get(), 1, n, s);
    dop.x = xt.get();
  }
  d_box_start.upload(lay.start, s);
  d_box_count.upload(lay.count, s);
  anc.assign(size_t(tree.depth() + 1), std::vector<int>(size_t(tree.num_boxes()), -1));
  for (const Box& b : tree.boxes()) {
    int cur = b.id;
    for (int lv = b.level; lv >= 0; --lv) {
      anc[size_t(lv)][size_t(b.id)] = cur;
      cur = tree.box(cur).parent;
    }
  }
  int* h_flag = nullptr;
  DevBuf<int> d_flag;
  if (op.kind() != kOpDense && op.kind() != kOpCallback) {
    // coincident points can only share a leaf
    std::vector<std::int64_t> ls, lc;
    for (const Box& b : tree.boxes())
      if (b.is_leaf() && lay.count[size_t(b.id)] > 1) {
        ls.push_back(lay.start[size_t(b.id)]);
        lc.push_back(lay.count[size_t(b.id)]);
      }
    DevBuf<std::int64_t> d_ls, d_lc;
    d_ls.upload(ls, s);
    d_lc.upload(lc, s);
    d_flag.alloc(1, s);
    HP_CUDA(cudaMemsetAsync(d_flag.get(), 0, sizeof(int), s));
    launch_find_duplicates(xt.get(), op.dim(), n, d_ls.get(), d_lc.get(), int(ls.size()), d_flag.get(), s);
    h_flag = static_cast<int*>(persistent_pinned(sizeof(int), 1));
    HP_CUDA(cudaMemcpyAsync(h_flag, d_flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  }
  HP_CUDA(cudaStreamSynchronize(s));
  if (h_flag) {
    has_dups = *h_flag != 0;
    // (persistent pinned buffer: not freed)
  }
}

void Engine::op_apply(bool adjoint, const double* x, int w, double* y) const {
  if (w <= 0) return;
  if (op.kind() != kOpCallback) {
    launch_full_apply(dop, adjoint, x, w, y, s);
    return;
  }
  // the caller's black box works in its own point order
  DevBuf<double> xi(size_t(n) * size_t(w), s), yi(size_t(n) * size_t(w), s);
  launch_permute_rows(x, 1, n, d_inv.get(), n, w, xi.get(), 1, n, s);
  op.call(adjoint, xi.get(), w, yi.get(), s);
  launch_permute_rows(yi.get(), 1, n, d_perm.get(), n, w, y, 1, n, s);
}

int pair_index(const std::vector<std::pair<int, int>>& pairs, int a, int b) {
  auto it = std::lower_bound(pairs.begin(), pairs.end(), std::make_pair(a, b));
  if (it == pairs.end() || *it != std::make_pair(a, b)) return -1;
  return int(it - pairs.begin());
}

std::pair<int, int> first_range(const std::vector<std::pair<int, int>>& pairs, int a) {
  const int lo_key = std::numeric_limits<int>::min();
  auto lo = std::lower_bound(pairs.begin(), pairs.end(), std::make_pair(a, lo_key));
  auto hi = std::lower_bound(pairs.begin(), pairs.end(), std::make_pair(a + 1, lo_key));
  return {int(lo - pairs.begin()), int(hi - pairs.begin())};
}

// ---------------------------------------------------------------- K4

// HP_QR=householder selects the register-resident Householder kernels
// (k_qr2.cu) instead of the Gram-based range finder (k_gqr.cu).
static bool qr_use_gram(int r, int kmax) {
  const char* e = std::getenv("HP_QR");
  if (e && std::string(e) == "householder") return false;
  return gqr_supported(r, kmax);
}

// Blocks the register-resident Householder kernel still factors faster than
// the Gram path: short blocks of narrow samples (<= 128 rows at r <= 48, where
// a Gram stage is dominated by per-kernel set-up; profiles/r02_qr_bench.txt:
// 128 x 42, 8000 blocks, 2.9 ms vs 3.9 ms). Depends on the block's shape only,
// so sharded runs route every block as the unsharded run does.
static bool qr_small_block(int rows, int r, int kmax) {
  return rows <= 128 && r <= 48 && qr_reg_cols(r) != 0 && qr_reg_cols(kmax) != 0 &&
         std::min(qr_reg_rows_max(r), qr_reg_rows_max(kmax)) >= 128;
}

QrPlan plan_qr(const std::vector<QrRequest>& reqs, int r, int kmax) {
  QrPlan pl;
  std::vector<QrRequest> house;  // requests left to the Householder kernels
  if (qr_use_gram(r, kmax)) {
    pl.gram = true;
    pl.gblocks.reserve(reqs.size());
    for (const QrRequest& q : reqs) {
      if (qr_small_block(q.rows, r, kmax)) {
        house.push_back(q);
        GqrBlock hb{};
        hb.a = q.a;
        hb.lda = q.rows;
        hb.rows = q.rows;
        hb.rank_slot = q.rank_slot;
        hb.task0 = int(pl.htasks.size());
        hb.ntasks = 1;
        pl.htasks.push_back(GqrTask{int(pl.hblocks.size()), 0, q.rows});
        pl.hblocks.push_back(hb);
        continue;
      }
      GqrBlock b{};
      b.a = q.a;
      b.out = q.out;
      b.lda = q.rows;
      b.ldo = q.ldo;
      b.rows = q.rows;
      b.rank_slot = q.rank_slot;
      b.task0 = int(pl.gtasks.size());
      // row tasks of equal size: <= kGqrTaskRows rows, 4x that for very tall blocks (their
      // partial Gram matrices would otherwise add a quarter of the block's own volume)
      const int cap = q.rows >= 8 * kGqrTaskRows ? 4 * kGqrTaskRows : kGqrTaskRows;
      const int nt = std::max(1, (q.rows + cap - 1) / cap);
      const int base = q.rows / nt, extra = q.rows % nt;
      int row = 0;
      for (int i = 0; i < nt; ++i) {
        const int rr = base + (i < extra ? 1 : 0);
        pl.gtasks.push_back(GqrTask{int(pl.gblocks.size()), row, rr});
        row += rr;
      }
      b.ntasks = nt;
      pl.gblocks.push_back(b);
    }
    if (house.empty()) return pl;
  }
  const std::vector<QrRequest>& todo = pl.gram ? house : reqs;
  // register-resident kernels when the widths allow, else shared-memory ones
  // (chunks must hold more than r rows or TSQR cannot shrink the stack)
  pl.reg = qr_reg_cols(r) != 0 && qr_reg_cols(kmax) != 0 &&
           std::min(qr_reg_rows_max(r), qr_reg_rows_max(kmax)) >= 2 * r;
  const int rm = pl.reg ? std::min(qr_reg_rows_max(r), qr_reg_rows_max(kmax)) : qr_rows_max(r);
  const int rc = pl.reg ? rm : qr_chunk_rows(r, kmax);  // TSQR chunk
  for (const QrRequest& q : todo) {
    if (q.rows <= rm) {
      pl.direct.push_back(QrBlock{q.a, q.out, 0, 0, q.rows, q.rows, q.ldo, 0, q.rank_slot, 0});
      continue;
    }
    // TSQR: chunks of <= rm rows, stacked R factors reduced the same way.
    std::int64_t cur_off = q.a;
    int cur_rows = q.rows, cur_ld = q.rows;
    std::int64_t cur_c = -1;  // Q of the current stacked matrix (workspace)
    int round = 0;
    while (cur_rows > rm) {
      const int nch = (cur_rows + rc - 1) / rc;
      const int base = cur_rows / nch, extra = cur_rows % nch;
      int next_rows = 0;
      for (int i = 0; i < nch; ++i) next_rows += std::min(base + (i < extra ? 1 : 0), r);
      const std::int64_t stacked = pl.wsize;
      pl.wsize += std::int64_t(next_rows) * r;
      const std::int64_t c_next = pl.wsize;
      pl.wsize += std::int64_t(next_rows) * kmax;
      if (int(pl.chunk_rounds.size()) <= round) {
        pl.chunk_rounds.resize(size_t(round) + 1);
        pl.back_rounds.resize(size_t(round) + 1);
      }
      int row = 0, srow = 0;
      for (int i = 0; i < nch; ++i) {
        const int cr = base + (i < extra ? 1 : 0);
        const std::int64_t tau = pl.tausize;
        pl.tausize += r;
        pl.chunk_rounds[size_t(round)].push_back(
            QrBlock{cur_off + row, stacked + srow, tau, 0, cr, cur_ld, next_rows, 0, -1, 0});
        QrBlock bp{};
        bp.a = cur_off + row;
        bp.tau = tau;
        bp.c = c_next + srow;
        bp.ldc = next_rows;
        bp.rows = cr;
        bp.lda = cur_ld;
        bp.out = round == 0 ? q.out + row : cur_c + row;
        bp.ldo = round == 0 ? q.ldo : cur_rows;
        bp.rank_slot = -1;
        pl.back_rounds[size_t(round)].push_back(bp);
        row += cr;
        srow += std::min(cr, r);
      }
      if (next_rows >= cur_rows) throw std::logic_error("plan_qr: TSQR does not shrink");
      cur_off = stacked;
      cur_rows = next_rows;
      cur_ld = next_rows;
      cur_c = c_next;
      ++round;
    }
    pl.tops.push_back(QrBlock{cur_off, cur_c, 0, 0, cur_rows, cur_ld, cur_rows, 0, q.rank_slot, 0});
  }
  return pl;
}

// Batches of whole blocks bounded by the workspace they need (Gram partials
// per row task, transforms and state per block).
static void run_gqr(const QrPlan& pl, double* data, double* out, int* d_ranks, int r, int kmax,
                    cudaStream_t s) {
  const std::int64_t psz = gqr_part_doubles(r, kmax), wsz = gqr_w_doubles(r, kmax);
  constexpr std::int64_t kBudget = std::int64_t(3) << 27;  // doubles (3 GiB)
  const size_t nb = pl.gblocks.size();
  size_t b0 = 0;
  while (b0 < nb) {
    size_t b1 = b0;
    std::int64_t need = 0;
    while (b1 < nb) {
      const std::int64_t add = std::int64_t(pl.gblocks[b1].ntasks) * psz + wsz;
      if (b1 > b0 && need + add > kBudget) break;
      need += add;
      ++b1;
    }
    std::vector<GqrBlock> blocks(pl.gblocks.begin() + std::ptrdiff_t(b0), pl.gblocks.begin() + std::ptrdiff_t(b1));
    const int t0 = blocks.front().task0, t1 = blocks.back().task0 + blocks.back().ntasks;
    std::vector<GqrTask> tasks(pl.gtasks.begin() + t0, pl.gtasks.begin() + t1);
    for (GqrBlock& b : blocks) b.task0 -= t0;
    for (GqrTask& t : tasks) t.block -= int(b0);
    DevBuf<GqrBlock> d_blocks;
    d_blocks.upload(blocks, s);
    DevBuf<GqrTask> d_tasks;
    d_tasks.upload(tasks, s);
    DevBuf<GqrState> d_state(blocks.size(), s);
    DevBuf<double> part(size_t(tasks.size()) * size_t(psz), s), wbuf(blocks.size() * size_t(wsz), s);
    launch_gqr(d_blocks.get(), int(blocks.size()), d_tasks.get(), int(tasks.size()), d_state.get(), data, out,
               part.get(), wbuf.get(), d_ranks, r, kmax, kQrRankDropTol, s);
    b0 = b1;
  }
}

void run_qr(const QrPlan& pl, double* data, double* out, int* d_ranks, int r, int kmax,
            cudaStream_t s) {
  DevBuf<GqrBlock> d_hb;
  DevBuf<GqrState> d_hs;
  if (pl.gram) {
    if (!pl.gblocks.empty()) run_gqr(pl, data, out, d_ranks, r, kmax, s);
    if (pl.direct.empty()) return;  // (the blocks left to the Householder kernels are all direct)
    d_hb.upload(pl.hblocks, s);
    DevBuf<GqrTask> d_ht;
    d_ht.upload(pl.htasks, s);
    d_hs.alloc(pl.hblocks.size(), s);
    launch_qr_rescale(d_hb.get(), int(pl.hblocks.size()), d_ht.get(), int(pl.htasks.size()), d_hs.get(), data, r, s);
  }
  auto max_rows = [](const std::vector<QrBlock>& v) {
    int m = 1;
    for (const QrBlock& b : v) m = std::max(m, b.rows);
    return m;
  };
  // register kernels: one launch per rows-per-thread class, so a block's
  // arithmetic does not depend on which other blocks share its batch (sharded
  // runs reproduce the unsharded factors bit for bit)
  auto by_class = [&](const std::vector<QrBlock>& v, int cols, auto&& launch) {
    if (v.empty()) return;
    if (!pl.reg) {
      DevBuf<QrBlock> d;
      d.upload(v, s);
      launch(d.get(), int(v.size()), max_rows(v));
      return;
    }
    std::map<int, std::vector<QrBlock>> cls;
    for (const QrBlock& b : v) cls[qr_reg_rpt(cols, b.rows)].push_back(b);
    for (auto& [rpt, list] : cls) {
      DevBuf<QrBlock> d;
      d.upload(list, s);
      launch(d.get(), int(list.size()), max_rows(list));
    }
  };
  DevBuf<double> w(size_t(std::max<std::int64_t>(pl.wsize, 1)), s);
  DevBuf<double> tau(size_t(std::max<std::int64_t>(pl.tausize, 1)), s);
  by_class(pl.direct, r, [&](const QrBlock* d, int nb, int mr) {
    if (pl.reg)
      launch_qr_reg(0, d, nb, data, out, nullptr, d_ranks, r, kmax, kQrRankDropTol, mr, s);
    else
      launch_qr_top(d, nb, data, out, d_ranks, r, kmax, kQrRankDropTol, mr, s);
  });
  if (pl.gram && d_ranks)  // non-finite blocks among the Householder-routed ones report rank -1
    launch_qr_flag(d_hb.get(), int(pl.hblocks.size()), d_hs.get(), d_ranks, s);
  for (size_t rd = 0; rd < pl.chunk_rounds.size(); ++rd) {
    by_class(pl.chunk_rounds[rd], r, [&](const QrBlock* d, int nb, int mr) {
      if (pl.reg)
        launch_qr_reg(1, d, nb, rd == 0 ? data : w.get(), w.get(), tau.get(), nullptr, r, kmax, 0.0, mr, s);
      else
        launch_qr_chunk(d, nb, rd == 0 ? data : w.get(), w.get(), tau.get(), r, mr, s);
    });
  }
  by_class(pl.tops, r, [&](const QrBlock* d, int nb, int mr) {
    if (pl.reg)
      launch_qr_reg(0, d, nb, w.get(), w.get(), nullptr, d_ranks, r, kmax, kQrRankDropTol, mr, s);
    else
      launch_qr_top(d, nb, w.get(), w.get(), d_ranks, r, kmax, kQrRankDropTol, mr, s);
  });
  for (size_t rd = pl.back_rounds.size(); rd-- > 0;) {
    by_class(pl.back_rounds[rd], kmax, [&](const QrBlock* d, int nb, int mr) {
      if (pl.reg)
        launch_qr_reg_backprop(d, nb, rd == 0 ? data : w.get(), tau.get(), w.get(), rd == 0 ? out : w.get(), r,
                               kmax, mr, s);
      else
        launch_qr_backprop(d, nb, rd == 0 ? data : w.get(), tau.get(), w.get(), rd == 0 ? out : w.get(), r, kmax,
                           mr, s);
    });
  }
}

// ---------------------------------------------------------------- K5 grams

GramPlan plan_gram(const std::vector<GramReq>& reqs, int nx, int ny) {
  constexpr int kChunk = 512;
  GramPlan pl;
  pl.nx = nx;
  pl.ny = ny;
  pl.off.assign(reqs.size() + 1, 0);
  for (size_t i = 0; i < reqs.size(); ++i) {
    const GramReq& q = reqs[i];
    for (int r0 = 0; r0 < q.rows; r0 += kChunk) {
      GramTask t{};
      t.x = q.x + (q.x_rowmajor ? std::int64_t(r0) * q.lx : r0);
      t.y = q.y + (q.y_rowmajor ? std::int64_t(r0) * q.ly : r0);
      t.out = std::int64_t(pl.tasks.size()) * nx * ny;
      t.rows = std::min(kChunk, q.rows - r0);
      t.lx = q.lx;
      t.ly = q.ly;
      t.x_rowmajor = q.x_rowmajor;
      t.y_rowmajor = q.y_rowmajor;
      pl.tasks.push_back(t);
    }
    pl.off[i + 1] = std::int64_t(pl.tasks.size());
  }
  return pl;
}

void run_gram(const GramPlan& pl, const double* xb, const double* yb, double* out,
              cudaStream_t s) {
  if (pl.tasks.empty()) return;
  DevBuf<GramTask> d_tasks;
  d_tasks.upload(pl.tasks, s);
  DevBuf<std::int64_t> d_off;
  d_off.upload(pl.off, s);
  DevBuf<double> partial(pl.tasks.size() * size_t(pl.nx) * size_t(pl.ny), s);
  launch_gram(d_tasks.get(), int(pl.tasks.size()), xb, yb, pl.nx, pl.ny, partial.get(), s);
  launch_sum_partials(d_off.get(), int(pl.off.size()) - 1, partial.get(), pl.nx * pl.ny, out, s);
}

// ---------------------------------------------------------------- K3

PeelPlan plan_peel(const Engine& e, const H1Rep& rep, const std::vector<SampleBlock>& blocks,
                   const std::vector<std::vector<int>>& payload_boxes, int top_level, int w,
                   bool with_adjoint) {
  PeelPlan pp;
  const int k = e.k;
  const int nc = int(payload_boxes.size());
  // group[(lp, box, c)] -> payload boxes of color c under `box` (level lp)
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
  for (int c = 0; c < nc; ++c) {
    for (int v : payload_boxes[size_t(c)]) {
      const int lv = e.tree.box(v).level;
      for (int lp = 2; lp <= std::min(lv, top_level); ++lp)
        groups[Key{lp, e.anc[size_t(lp)][size_t(v)], c}].push_back(v);
    }
  }
  // coefficient index per (side, lp, q, c): -2 unknown, -1 none
  std::vector<std::vector<int>> cidx[2];
  for (int side = 0; side < 2; ++side) {
    cidx[side].resize(size_t(top_level) + 1);
    for (int lp = 2; lp <= top_level; ++lp)
      cidx[side][size_t(lp)].assign(rep.levels[size_t(lp)].pairs.size() * size_t(nc), -2);
  }
  auto coeff = [&](int side, int lp, int q, int c) -> int {
    int& slot = cidx[side][size_t(lp)][size_t(q) * size_t(nc) + size_t(c)];
    if (slot != -2) return slot;
    const auto& ld = rep.levels[size_t(lp)];
    const auto [x, y] = ld.pairs[size_t(q)];
    const int src = side == 0 ? y : x;
    auto g = groups.find(Key{lp, src, c});
    if (g == groups.end()) return slot = -1;
    if (ld.uoff[size_t(q)] < 0 || ld.voff[size_t(q)] < 0)
      throw std::logic_error("peel: a coarse pair's factors are not held by this rank");
    CoeffTask t{};
    t.f = side == 0 ? ld.voff[size_t(q)] : ld.uoff[size_t(q)];
    t.btrans = side == 0 ? 0 : 1;
    t.b = ld.boff[size_t(q)];
    t.f_row0 = e.start(src);
    t.frows = e.count(src);
    t.seg_begin = int(pp.seg_start.size());
    for (int v : g->second) {
      pp.seg_start.push_back(e.start(v));
      pp.seg_count.push_back(e.count(v));
      pp.coeff_flops += 2.0 * double(e.count(v)) * k * w;
    }
    pp.coeff_flops += 2.0 * k * k * w;
    t.seg_end = int(pp.seg_start.size());
    auto& list = side == 0 ? pp.coeff_fwd : pp.coeff_adj;
    t.t_out = std::int64_t(list.size()) * k * w;
    list.push_back(t);
    return slot = int(list.size()) - 1;
  };
  // term list per (side, lp, ancestor box, color), shared by every tile of
  // every target box under that ancestor: forward terms U_q T_{q,c} over the
  // pairs (ap, x), adjoint terms V_q T'_{q,c} over the pairs (x, ap)
  std::unordered_map<Key, std::pair<int, int>, KeyHash> lists[2];
  auto term_list = [&](int side, int lp, int ap, int c) -> std::pair<int, int> {
    auto it = lists[side].find(Key{lp, ap, c});
    if (it != lists[side].end()) return it->second;
    const auto& ld = rep.levels[size_t(lp)];
    auto& terms = side == 0 ? pp.terms_fwd : pp.terms_adj;
    const int b0 = int(terms.size());
    if (side == 0) {
      const auto [q0, q1] = first_range(ld.pairs, ap);
      for (int q = q0; q < q1; ++q) {
        const int ti = coeff(0, lp, q, c);
        if (ti >= 0) terms.push_back(PeelTerm{ld.uoff[size_t(q)], std::int64_t(ti) * k * w, e.count(ap), 0});
      }
    } else {
      for (int x : e.adj.interaction[size_t(ap)]) {
        const int q = pair_index(ld.pairs, x, ap);
        if (q < 0) continue;
        const int ti = coeff(1, lp, q, c);
        if (ti >= 0) terms.push_back(PeelTerm{ld.voff[size_t(q)], std::int64_t(ti) * k * w, e.count(ap), 0});
      }
    }
    const std::pair<int, int> r{b0, int(terms.size())};
    lists[side].emplace(Key{lp, ap, c}, r);
    return r;
  };
  for (const SampleBlock& sb : blocks) {
    const int a = sb.box;
    const int la = e.tree.box(a).level;
    const int rows = e.count(a);
    for (int t0 = 0; t0 < rows; t0 += kTile) {
      const int trows = std::min(kTile, rows - t0);
      const int cols = std::min(sb.cols, w);
      PeelTask tf{sb.off + t0, trows, rows, int(pp.refs_fwd.size()), 0, cols, 0};
      PeelTask ta{sb.off + t0, trows, rows, int(pp.refs_adj.size()), 0, cols, 0};
      for (int lp = 2; lp <= std::min(la, top_level); ++lp) {
        const auto& ld = rep.levels[size_t(lp)];
        if (ld.pairs.empty()) continue;
        const int ap = e.anc[size_t(lp)][size_t(a)];
        const std::int64_t roff = e.start(a) - e.start(ap) + t0;
        const auto lf = term_list(0, lp, ap, sb.color);
        if (lf.second > lf.first) {
          pp.refs_fwd.push_back(PeelRef{lf.first, lf.second, roff});
          pp.apply_flops += 2.0 * trows * k * w * (lf.second - lf.first);
        }
        if (!with_adjoint) continue;
        const auto la2 = term_list(1, lp, ap, sb.color);
        if (la2.second > la2.first) {
          pp.refs_adj.push_back(PeelRef{la2.first, la2.second, roff});
          pp.apply_flops += 2.0 * trows * k * w * (la2.second - la2.first);
        }
      }
      tf.ref_end = int(pp.refs_fwd.size());
      ta.ref_end = int(pp.refs_adj.size());
      if (tf.ref_end > tf.ref_begin) pp.tasks_fwd.push_back(tf);
      if (with_adjoint && ta.ref_end > ta.ref_begin) pp.tasks_adj.push_back(ta);
    }
  }
  return pp;
}

PeelPlan plan_peel_parallel(const Engine& e, const H1Rep& rep, const std::vector<SampleBlock>& blocks,
                            const std::vector<std::vector<int>>& payload_boxes, int top_level, int w,
                            bool with_adjoint, int threads) {
  const int nc = int(payload_boxes.size());
  if (threads <= 1 || nc < 2 || blocks.size() < 2048)
    return plan_peel(e, rep, blocks, payload_boxes, top_level, w, with_adjoint);
  // colors partitioned over the threads (balanced by block rows): coefficient
  // tasks (q, c) and term lists (side, level, ancestor, c) never straddle two
  // parts, so the merged plan is the serial one up to the order of its tasks
  std::vector<double> rows_of_color(static_cast<size_t>(nc), 0.0);
  for (const SampleBlock& b : blocks) rows_of_color[size_t(b.color)] += double(e.count(b.box));
  const auto cuts = partition_ranges(rows_of_color, threads);
  std::vector<std::vector<SampleBlock>> part(static_cast<size_t>(threads));
  std::vector<int> part_of(static_cast<size_t>(nc), 0);
  for (int t = 0; t < threads; ++t)
    for (std::int64_t c = cuts[size_t(t)]; c < cuts[size_t(t) + 1]; ++c) part_of[size_t(c)] = t;
  for (const SampleBlock& b : blocks) part[size_t(part_of[size_t(b.color)])].push_back(b);
  std::vector<PeelPlan> plans(static_cast<size_t>(threads));
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] { plans[size_t(t)] = plan_peel(e, rep, part[size_t(t)], payload_boxes, top_level, w, with_adjoint); });
  for (auto& th : pool) th.join();
  PeelPlan out;
  const std::int64_t kw = std::int64_t(e.k) * w;
  for (PeelPlan& pl : plans) {
    const int seg0 = int(out.seg_start.size());
    out.seg_start.insert(out.seg_start.end(), pl.seg_start.begin(), pl.seg_start.end());
    out.seg_count.insert(out.seg_count.end(), pl.seg_count.begin(), pl.seg_count.end());
    auto merge_side = [&](std::vector<CoeffTask>& coeff_out, std::vector<CoeffTask>& coeff,
                          std::vector<PeelTask>& tasks_out, std::vector<PeelTask>& tasks,
                          std::vector<PeelRef>& refs_out, std::vector<PeelRef>& refs,
                          std::vector<PeelTerm>& terms_out, std::vector<PeelTerm>& terms) {
      const std::int64_t c0 = std::int64_t(coeff_out.size()) * kw;
      const int t0 = int(terms_out.size()), r0 = int(refs_out.size());
      for (CoeffTask c : coeff) {
        c.seg_begin += seg0;
        c.seg_end += seg0;
        c.t_out += c0;
        coeff_out.push_back(c);
      }
      for (PeelTerm tm : terms) {
        tm.t += c0;
        terms_out.push_back(tm);
      }
      for (PeelRef rf : refs) {
        rf.term_begin += t0;
        rf.term_end += t0;
        refs_out.push_back(rf);
      }
      for (PeelTask tk : tasks) {
        tk.ref_begin += r0;
        tk.ref_end += r0;
        tasks_out.push_back(tk);
      }
    };
    merge_side(out.coeff_fwd, pl.coeff_fwd, out.tasks_fwd, pl.tasks_fwd, out.refs_fwd, pl.refs_fwd, out.terms_fwd,
               pl.terms_fwd);
    merge_side(out.coeff_adj, pl.coeff_adj, out.tasks_adj, pl.tasks_adj, out.refs_adj, pl.refs_adj, out.terms_adj,
               pl.terms_adj);
    out.coeff_flops += pl.coeff_flops;
    out.apply_flops += pl.apply_flops;
  }
  return out;
}

void run_peel(const PeelPlan& pp, const Engine& e, const H1Rep& rep, const double* g, int gld,
              int w, bool identity, double* samples, int adj_col, cudaStream_t s) {
  const int k = e.k;
  DevBuf<std::int64_t> d_ss, d_sc;
  d_ss.upload(pp.seg_start, s);
  d_sc.upload(pp.seg_count, s);
  for (int side = 0; side < 2; ++side) {
    const auto& coeff = side == 0 ? pp.coeff_fwd : pp.coeff_adj;
    const auto& tasks = side == 0 ? pp.tasks_fwd : pp.tasks_adj;
    const auto& refs = side == 0 ? pp.refs_fwd : pp.refs_adj;
    const auto& terms = side == 0 ? pp.terms_fwd : pp.terms_adj;
    if (coeff.empty() || tasks.empty()) continue;
    DevBuf<CoeffTask> d_coeff;
    d_coeff.upload(coeff, s);
    DevBuf<double> tbuf(coeff.size() * size_t(k) * size_t(w), s);
    launch_peel_coeff(d_coeff.get(), int(coeff.size()), rep.d_factors, rep.d_factors, d_ss.get(),
                      d_sc.get(), g, gld, identity ? -1 : (side == 0 ? 0 : e.r), k, w, tbuf.get(), s);
    DevBuf<PeelTask> d_tasks;
    d_tasks.upload(tasks, s);
    DevBuf<PeelRef> d_refs;
    d_refs.upload(refs, s);
    DevBuf<PeelTerm> d_terms;
    d_terms.upload(terms, s);
    launch_peel_apply(d_tasks.get(), int(tasks.size()), d_refs.get(), d_terms.get(), rep.d_factors, tbuf.get(),
                      k, w, samples, side == 0 ? 0 : adj_col, -1.0, s);
  }
}

}  // namespace hpeel::detail
