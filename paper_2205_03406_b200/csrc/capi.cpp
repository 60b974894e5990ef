// C ABI over the hpeel host layer and device engine (include/hpeel_b200.h).
#include "../../include/hpeel_b200.h"
#include "hpeel_probe.h"

#include <array>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "hpeel/box_tree.hpp"
#include "hpeel/coloring.hpp"
#include "hpeel/peeling.hpp"
#include "hpeel/rng.hpp"
#include "hpeel/serialize.hpp"
#include "hpeel/shard.hpp"

using namespace hpeel;

struct hp_tree {
  std::shared_ptr<const BoxTree> tree;
  std::shared_ptr<const AdjacencyInfo> adj;
  std::shared_ptr<const TreeLayout> layout;
};
struct hp_plan {
  std::vector<ConstraintSet> sets;
  IncompatibilityGraph graph;
  Coloring coloring, dsatur;
  std::vector<BlockTestMatrix> mats;
  std::vector<std::array<int, 3>> block_map;  // fallback pattern: (alpha, beta, matrix)
  std::shared_ptr<const BoxTree> tree;
};
struct hp_op {
  std::shared_ptr<DeviceOperator> op;
};
struct hp_rep {
  PeelResult result;
};
struct hp_comm {
  std::unique_ptr<Comm> comm;
};

namespace hpeel {
std::int64_t& launch_counter();
void set_k2_mode(int mode);
void set_k2_path(int path);
void debug_fast_log(const double* x, std::int64_t n, double* y, int device);
Matrix debug_payload(const BoxTree& tree, const TreeLayout& lay, int level, int r,
                     std::uint64_t seed, int device);
double debug_qr(const double* blocks, const int* rows, int nb, int cols, int kmax, int device,
                double* q, int* ranks);
}

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return HP_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HP_ERR_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return HP_ERR_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HP_ERR_RUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return HP_ERR_RUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null ") + what);
}

Matrix from_host(const double* p, std::int64_t rows, std::int64_t cols) {
  Matrix m(rows, cols);
  if (rows * cols > 0) std::memcpy(m.data(), p, size_t(rows * cols) * sizeof(double));
  return m;
}
}  // namespace

extern "C" {

const char* hp_last_error(void) { return g_err.c_str(); }

int hp_device_count(int* count) {
  return guard([&] {
    need(count, "count");
    if (cudaGetDeviceCount(count) != cudaSuccess) *count = 0;
  });
}

int64_t hp_launch_count(void) { return launch_counter(); }

void hp_debug_set_k2_mode(int mode) { set_k2_mode(mode); }
void hp_debug_set_k2_path(int path) { set_k2_path(path); }

int hp_device_synchronize(void) {
  return guard([&] {
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  });
}

uint64_t hp_mix_seed(uint64_t seed, uint64_t tag) { return mix_seed(seed, tag); }

int hp_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  return guard([&] {
    const Matrix g = gaussian_matrix(rows, cols, seed);
    if (g.size()) need(out, "out");
    std::memcpy(out, g.data(), size_t(g.size()) * sizeof(double));
  });
}

int hp_random_cloud(int64_t n, int dim, uint64_t seed, double* out) {
  return guard([&] {
    if (n < 0 || dim < 1) throw std::invalid_argument("bad shape");
    need(out, "out");
    SplitMix64 st(seed);
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < dim; ++j) out[i + j * n] = st.next_closed_open();
  });
}

int hp_tree_build(const double* raw, int64_t n, int dim, int leaf_capacity, hp_tree** out) {
  return guard([&] {
    need(out, "out");
    if (n > 0) need(raw, "raw");
    auto t = std::make_unique<hp_tree>();
    t->tree = std::make_shared<const BoxTree>(
        BoxTree::build(PointCloud::from_raw(from_host(raw, n, dim)), leaf_capacity));
    t->adj = std::make_shared<const AdjacencyInfo>(adjacency(*t->tree));
    t->layout = std::make_shared<const TreeLayout>(tree_layout(*t->tree));
    *out = t.release();
  });
}

void hp_tree_free(hp_tree* tree) { delete tree; }

int hp_tree_info(const hp_tree* t, int64_t* info) {
  return guard([&] {
    need(t, "tree");
    need(info, "info");
    const BoxTree& tr = *t->tree;
    int64_t pts = 0;
    for (const Box& b : tr.boxes()) pts += int64_t(b.points.size());
    info[0] = tr.num_points();
    info[1] = tr.dim();
    info[2] = tr.depth();
    info[3] = tr.num_boxes();
    info[4] = tr.max_leaf_size();
    info[5] = tr.is_fully_populated() ? 1 : 0;
    info[6] = tr.leaf_capacity();
    info[7] = pts;
  });
}

int hp_tree_boxes(const hp_tree* t, int* level, int* parent, int64_t* coord, int64_t* pt_off,
                  int* pts) {
  return guard([&] {
    need(t, "tree");
    const BoxTree& tr = *t->tree;
    int64_t o = 0;
    for (const Box& b : tr.boxes()) {
      const size_t i = size_t(b.id);
      if (level) level[i] = b.level;
      if (parent) parent[i] = b.parent;
      if (coord)
        for (int j = 0; j < tr.dim(); ++j) coord[i * size_t(tr.dim()) + size_t(j)] = b.coord[size_t(j)];
      if (pt_off) pt_off[i] = o;
      if (pts)
        for (int p : b.points) pts[o++] = p;
      else
        o += int64_t(b.points.size());
    }
    if (pt_off) pt_off[tr.num_boxes()] = o;
  });
}

int hp_tree_lists(const hp_tree* t, int which, int64_t* off, int* items) {
  return guard([&] {
    need(t, "tree");
    need(off, "off");
    const BoxTree& tr = *t->tree;
    const AdjacencyInfo& a = *t->adj;
    int64_t o = 0;
    for (int b = 0; b < tr.num_boxes(); ++b) {
      const std::vector<int>* v = nullptr;
      switch (which) {
        case 0: v = &a.neighbors[size_t(b)]; break;
        case 1: v = &a.interaction[size_t(b)]; break;
        case 2: v = &a.coarse_leaf_neighbors[size_t(b)]; break;
        case 3: v = &a.dense_partners[size_t(b)]; break;
        case 4: v = &tr.box(b).children; break;
        default: throw std::invalid_argument("unknown list");
      }
      off[b] = o;
      if (items)
        for (int x : *v) items[o++] = x;
      else
        o += int64_t(v->size());
    }
    off[tr.num_boxes()] = o;
  });
}

int64_t hp_tree_cross_level_adjacencies(const hp_tree* t) {
  return t ? int64_t(t->adj->cross_level_adjacencies) : -1;
}

int hp_tree_pairs(const hp_tree* t, int level, int64_t* count, int* pairs) {
  return guard([&] {
    need(t, "tree");
    need(count, "count");
    const auto v = level < 0 ? dense_pairs(*t->tree, *t->adj) : admissible_pairs(*t->tree, *t->adj, level);
    *count = int64_t(v.size());
    if (pairs)
      for (size_t i = 0; i < v.size(); ++i) {
        pairs[2 * i] = v[i].first;
        pairs[2 * i + 1] = v[i].second;
      }
  });
}

int hp_tree_layout(const hp_tree* t, int* perm, int64_t* start, int64_t* count) {
  return guard([&] {
    need(t, "tree");
    const TreeLayout& l = *t->layout;
    if (perm) std::memcpy(perm, l.perm.data(), l.perm.size() * sizeof(int));
    if (start) std::memcpy(start, l.start.data(), l.start.size() * sizeof(int64_t));
    if (count) std::memcpy(count, l.count.data(), l.count.size() * sizeof(int64_t));
  });
}

int hp_plan_build(const hp_tree* t, int level, int mode, int width, uint64_t seed, int phase,
                  int pairwise_graph, hp_plan** out) {
  return guard([&] {
    need(t, "tree");
    need(out, "out");
    if (mode < 0 || mode > 3) throw std::invalid_argument("unknown sampling mode");
    const SampleMode m = SampleMode(mode);
    auto p = std::make_unique<hp_plan>();
    p->tree = t->tree;
    if (pairwise_graph == 3) {  // ColoringStrategy::kFallbackPattern: no sets, graph or coloring
      const SamplingPlan sp = make_plan(*t->tree, *t->adj, level, m, width, seed, phase, true);
      p->mats = sp.matrices;
      p->coloring.num_colors = int(sp.matrices.size());
      p->graph.num_vertices = 0;
      for (const auto& [key, c] : sp.block_to_matrix) p->block_map.push_back({key.first, key.second, c});
      *out = p.release();
      return;
    }
    p->sets = build_constraints(*t->tree, *t->adj, level, m);
    if (pairwise_graph == 2) {  // implicit graph (the driver's path): no edge lists kept
      if (!ImplicitGraph::applicable(p->sets)) throw std::invalid_argument("implicit graph needs single-payload sets");
      const ImplicitGraph g(p->sets);
      p->dsatur = dsatur_color(g);
      p->coloring = plan_coloring(*t->tree, p->sets, p->dsatur, m);
      p->graph.num_vertices = int(p->sets.size());
      p->graph.edges.assign(p->sets.size(), {});
    } else {
      p->graph = pairwise_graph ? build_graph_pairwise(p->sets) : build_graph(p->sets);
      p->dsatur = dsatur_color(p->graph);
      p->coloring = plan_coloring(*t->tree, p->sets, p->graph, m);
    }
    if (!p->sets.empty())
      p->mats = assemble_test_matrices(p->sets, p->coloring, *t->tree, level, width, seed, phase);
    *out = p.release();
  });
}

void hp_plan_free(hp_plan* plan) { delete plan; }

int hp_plan_info(const hp_plan* p, int64_t* info) {
  return guard([&] {
    need(p, "plan");
    need(info, "info");
    int64_t pay = 0, zero = 0, own = 0, mp = 0;
    for (const auto& s : p->sets) {
      pay += int64_t(s.payload.size());
      zero += int64_t(s.zero.size());
      own += int64_t(s.owners.size());
    }
    for (const auto& m : p->mats) mp += int64_t(m.payload.size());
    info[0] = int64_t(p->sets.size());
    info[1] = int64_t(p->graph.num_edges());
    info[2] = p->coloring.num_colors;
    info[3] = int64_t(p->dsatur.queue_ops);
    info[4] = pay;
    info[5] = zero;
    info[6] = own;
    info[7] = mp;
  });
}

int hp_plan_sets(const hp_plan* p, int64_t* pay_off, int* pay_box, int* pay_tag, int64_t* zero_off,
                 int* zero, int64_t* own_off, int* owners) {
  return guard([&] {
    need(p, "plan");
    int64_t a = 0, b = 0, c = 0;
    size_t i = 0;
    for (const auto& s : p->sets) {
      if (pay_off) pay_off[i] = a;
      if (zero_off) zero_off[i] = b;
      if (own_off) own_off[i] = c;
      for (auto [box, tag] : s.payload) {
        if (pay_box) pay_box[a] = box;
        if (pay_tag) pay_tag[a] = int(tag);
        ++a;
      }
      for (int z : s.zero) {
        if (zero) zero[b] = z;
        ++b;
      }
      for (auto [x, y] : s.owners) {
        if (owners) {
          owners[2 * c] = x;
          owners[2 * c + 1] = y;
        }
        ++c;
      }
      ++i;
    }
    if (pay_off) pay_off[i] = a;
    if (zero_off) zero_off[i] = b;
    if (own_off) own_off[i] = c;
  });
}

int hp_plan_graph(const hp_plan* p, int64_t* off, int* adj) {
  return guard([&] {
    need(p, "plan");
    need(off, "off");
    int64_t o = 0;
    for (size_t v = 0; v < p->graph.edges.size(); ++v) {
      off[v] = o;
      for (int w : p->graph.edges[v]) {
        if (adj) adj[o] = w;
        ++o;
      }
    }
    off[p->graph.edges.size()] = o;
  });
}

int hp_plan_coloring(const hp_plan* p, int* color, int* dsatur, int* dsatur_colors) {
  return guard([&] {
    need(p, "plan");
    if (color) std::memcpy(color, p->coloring.color.data(), p->coloring.color.size() * sizeof(int));
    if (dsatur) std::memcpy(dsatur, p->dsatur.color.data(), p->dsatur.color.size() * sizeof(int));
    if (dsatur_colors) *dsatur_colors = p->dsatur.num_colors;
  });
}

int hp_plan_matrices(const hp_plan* p, int64_t* off, int* boxes) {
  return guard([&] {
    need(p, "plan");
    need(off, "off");
    int64_t o = 0;
    for (size_t c = 0; c < p->mats.size(); ++c) {
      off[c] = o;
      for (auto [box, tag] : p->mats[c].payload) {
        if (boxes) boxes[o] = box;
        ++o;
      }
    }
    off[p->mats.size()] = o;
  });
}

int hp_plan_block_map(const hp_plan* p, int64_t* count, int* triples) {
  return guard([&] {
    need(p, "plan");
    need(count, "count");
    *count = int64_t(p->block_map.size());
    if (triples)
      for (size_t i = 0; i < p->block_map.size(); ++i)
        for (int j = 0; j < 3; ++j) triples[3 * i + size_t(j)] = p->block_map[i][size_t(j)];
  });
}

int hp_plan_realize(const hp_plan* p, int color, double* out) {
  return guard([&] {
    need(p, "plan");
    need(out, "out");
    if (color < 0 || color >= int(p->mats.size())) throw std::invalid_argument("color out of range");
    const Matrix m = p->mats[size_t(color)].realize(*p->tree);
    std::memcpy(out, m.data(), size_t(m.size()) * sizeof(double));
  });
}

int hp_dsatur(int nv, const int64_t* off, const int* adj, int* color, int* num_colors,
              int64_t* queue_ops) {
  return guard([&] {
    IncompatibilityGraph g;
    g.num_vertices = nv;
    g.edges.resize(size_t(nv));
    for (int v = 0; v < nv; ++v) g.edges[size_t(v)].assign(adj + off[v], adj + off[v + 1]);
    const Coloring c = dsatur_color(g);
    if (color) std::memcpy(color, c.color.data(), c.color.size() * sizeof(int));
    if (num_colors) *num_colors = c.num_colors;
    if (queue_ops) *queue_ops = int64_t(c.queue_ops);
  });
}

int hp_op_dense(const double* a, int64_t n, int device, hp_op** out) {
  return guard([&] {
    need(out, "out");
    need(a, "matrix");
    auto o = std::make_unique<hp_op>();
    o->op = DeviceOperator::dense(from_host(a, n, n), device);
    *out = o.release();
  });
}

int hp_op_kernel(int kind, const double* points, int64_t n, int dim, double param, int device,
                 hp_op** out) {
  return guard([&] {
    need(out, "out");
    need(points, "points");
    auto o = std::make_unique<hp_op>();
    o->op = DeviceOperator::kernel(kind, from_host(points, n, dim), param, device);
    *out = o.release();
  });
}

void hp_op_free(hp_op* op) { delete op; }

int hp_op_callback(int64_t n, int symmetric, int device_pointers, hp_apply_fn fn, void* ctx, int device,
                   hp_op** out) {
  return guard([&] {
    need(out, "out");
    need(reinterpret_cast<const void*>(fn), "apply function");
    auto o = std::make_unique<hp_op>();
    o->op = DeviceOperator::callback(n, symmetric != 0, device_pointers != 0, fn, ctx, device);
    *out = o.release();
  });
}

int hp_op_apply(const hp_op* op, int adjoint, const double* x, int64_t w, double* y) {
  return guard([&] {
    need(op, "op");
    const Matrix r = op->op->apply(from_host(x, op->op->rows(), w), adjoint != 0);
    std::memcpy(y, r.data(), size_t(r.size()) * sizeof(double));
  });
}

int hp_compress(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                int format, int strategy, int capture, hp_rep** out) {
  return guard([&] {
    need(op, "op");
    need(tree, "tree");
    need(out, "out");
    if (format < 0 || format > 3) throw std::invalid_argument("unknown format");
    PeelConfig cfg;
    cfg.rank = rank;
    cfg.oversample = oversample;
    cfg.leaf_capacity = tree->tree->leaf_capacity();
    cfg.seed = seed;
    cfg.format = PeelFormat(format);
    cfg.strategy = strategy == HP_STRATEGY_FALLBACK_PATTERN ? ColoringStrategy::kFallbackPattern
                                                            : ColoringStrategy::kGraph;
    cfg.capture_samples = capture != 0;
    auto r = std::make_unique<hp_rep>();
    r->result = compress(*op->op, tree->tree, cfg);
    *out = r.release();
  });
}

void hp_rep_free(hp_rep* rep) { delete rep; }

int hp_comm_unique_id(unsigned char* id128) {
  return guard([&] {
    need(id128, "id");
    NcclComm::unique_id(id128);
  });
}

int hp_comm_create(const unsigned char* id128, int rank, int world, int device, hp_comm** out) {
  return guard([&] {
    need(out, "out");
    if (world > 1) need(id128, "id");
    auto c = std::make_unique<hp_comm>();
    c->comm = std::make_unique<NcclComm>(id128, rank, world, device);
    *out = c.release();
  });
}

void hp_comm_free(hp_comm* comm) { delete comm; }

namespace {
PeelConfig make_config(const hp_tree* tree, int rank, int oversample, uint64_t seed, int format, int strategy,
                       int capture) {
  if (format < 0 || format > 3) throw std::invalid_argument("unknown format");
  PeelConfig cfg;
  cfg.rank = rank;
  cfg.oversample = oversample;
  cfg.leaf_capacity = tree->tree->leaf_capacity();
  cfg.seed = seed;
  cfg.format = PeelFormat(format);
  cfg.strategy = strategy == HP_STRATEGY_FALLBACK_PATTERN ? ColoringStrategy::kFallbackPattern
                                                          : ColoringStrategy::kGraph;
  cfg.capture_samples = capture != 0;
  return cfg;
}
}  // namespace

int hp_compress_ex(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                   int format, int strategy, int capture, hp_comm* comm, hp_rep** out) {
  return guard([&] {
    need(op, "op");
    need(tree, "tree");
    need(out, "out");
    PeelConfig cfg = make_config(tree, rank, oversample, seed, format, strategy, capture);
    cfg.comm = comm ? comm->comm.get() : nullptr;
    auto r = std::make_unique<hp_rep>();
    static const bool timing = std::getenv("HP_DRIVER_TIMING") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    r->result = compress(*op->op, tree->tree, cfg);
    if (timing)
      std::fprintf(stderr, "[capi] compress() returned after %.1f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    *out = r.release();
  });
}

int hp_compress_group(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                      int format, int strategy, int capture, int world, hp_rep** outs) {
  return guard([&] {
    need(op, "op");
    need(tree, "tree");
    need(outs, "outs");
    if (world < 1) throw std::invalid_argument("world size must be >= 1");
    const PeelConfig cfg = make_config(tree, rank, oversample, seed, format, strategy, capture);
    auto results = compress_group(*op->op, tree->tree, cfg, world);
    for (int g = 0; g < world; ++g) {
      auto r = std::make_unique<hp_rep>();
      r->result = std::move(results[size_t(g)]);
      outs[g] = r.release();
    }
  });
}

int hp_shard_owners(const hp_tree* tree, int world, int* owner, int* cut, int64_t* point_bounds) {
  return guard([&] {
    need(tree, "tree");
    const Ownership o = make_ownership(*tree->tree, *tree->layout, world, 0);
    if (owner) std::memcpy(owner, o.owner.data(), o.owner.size() * sizeof(int));
    if (cut) *cut = o.cut;
    if (point_bounds) std::memcpy(point_bounds, o.point_bounds.data(), o.point_bounds.size() * sizeof(int64_t));
  });
}

int hp_shard_memory_plan(const hp_tree* tree, int rank, int oversample, int world, double* out) {
  return guard([&] {
    need(tree, "tree");
    need(out, "out");
    if (rank < 1 || oversample < 0 || world < 1) throw std::invalid_argument("bad rank / oversampling / world");
    shard_memory_plan(*tree->tree, rank, oversample, world, out);
  });
}

int hp_shard_exchange_counts(const hp_tree* tree, int rank, int world, int shard, int level, int phase,
                             int64_t* send, int64_t* recv) {
  return guard([&] {
    need(tree, "tree");
    need(send, "send");
    need(recv, "recv");
    if (rank < 1 || world < 1 || shard < 0 || shard >= world || (phase != 1 && phase != 2))
      throw std::invalid_argument("bad rank / shard / world / phase");
    shard_exchange_counts(*tree->tree, rank, world, shard, level, phase, send, recv);
  });
}

int hp_export_sizes_shard(const hp_tree* tree, int rank, int world, int shard, int64_t* factor_doubles,
                          int64_t* dense_doubles) {
  return guard([&] {
    need(tree, "tree");
    if (rank < 1) throw std::invalid_argument("fixed rank must be >= 1");
    if (world < 1 || shard < 0 || shard >= world) throw std::invalid_argument("bad shard / world size");
    export_sizes(*tree->tree, rank, factor_doubles, dense_doubles, world, shard);
  });
}

int hp_rep_shard(const hp_rep* rep, int level, int64_t pair, int* world, int* shard, int* held) {
  return guard([&] {
    need(rep, "rep");
    const H1Rep& h = *rep->result.rep;
    if (world) *world = h.world;
    if (shard) *shard = h.shard_rank;
    if (held) {
      if (level < 0) {
        *held = pair >= 0 && size_t(pair) < h.dense.off.size() && h.dense.off[size_t(pair)] >= 0;
      } else {
        *held = size_t(level) < h.levels.size() && pair >= 0 && size_t(pair) < h.levels[size_t(level)].uoff.size() &&
                h.levels[size_t(level)].uoff[size_t(pair)] >= 0;
      }
    }
  });
}

int hp_partition_ranges(const double* work, int64_t n, int world, int64_t* bounds) {
  return guard([&] {
    need(bounds, "bounds");
    if (n > 0) need(work, "work");
    const auto b = partition_ranges(std::vector<double>(work, work + n), world);
    std::memcpy(bounds, b.data(), b.size() * sizeof(int64_t));
  });
}

int hp_rep_report(const hp_rep* rep, double* totals, int64_t* nphases) {
  return guard([&] {
    need(rep, "rep");
    const RunReport& r = rep->result.report;
    if (totals) {
      totals[0] = double(r.forward_cols);
      totals[1] = double(r.adjoint_cols);
      totals[2] = r.max_sampling_colors;
      totals[3] = r.wall_s_total;
      totals[4] = r.wall_s_net;
      totals[5] = double(r.net_flops);
      totals[7] = r.peak_device_bytes;
      totals[8] = r.exchange_bytes;
      totals[6] = r.setup_ms;
    }
    if (nphases) *nphases = int64_t(r.phases.size());
  });
}

int hp_rep_phase(const hp_rep* rep, int64_t phase, int64_t* ints, double* times) {
  return guard([&] {
    need(rep, "rep");
    const auto& ph = rep->result.report.phases.at(size_t(phase));
    if (ints) {
      ints[0] = ph.phase == "leaf" ? 1 : 0;
      ints[1] = ph.level;
      ints[2] = ph.colors;
      ints[3] = ph.forward_cols;
      ints[4] = ph.adjoint_cols;
      ints[5] = ph.net_flops;
      ints[6] = ph.apply_path;
    }
    if (times) {
      times[0] = ph.wall_ms_total;
      times[1] = ph.wall_ms_net;
      times[2] = ph.apply_ms;
      times[3] = ph.peel_ms;
      times[4] = ph.qr_ms;
      times[5] = ph.bsolve_ms;
      times[6] = ph.apply_flops;
      times[7] = ph.kernel_evals;
      times[8] = ph.host_wait_ms;
      times[9] = ph.start_ms;
      times[10] = ph.peel_flops;
      times[11] = ph.qr_flops;
      times[12] = ph.bsolve_flops;
    }
  });
}

int hp_rep_csv(const hp_rep* rep, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    need(rep, "rep");
    const std::string s = rep->result.report.to_csv();
    if (len) *len = int64_t(s.size());
    if (buf && cap > 0) {
      const size_t n = std::min(size_t(cap - 1), s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

int hp_rep_num_pairs(const hp_rep* rep, int level, int64_t* count) {
  return guard([&] {
    need(rep, "rep");
    need(count, "count");
    const H1Rep& h = *rep->result.rep;
    if (level < 0) *count = int64_t(h.dense.pairs.size());
    else if (size_t(level) < h.levels.size()) *count = int64_t(h.levels[size_t(level)].pairs.size());
    else *count = 0;
  });
}

int hp_rep_block(const hp_rep* rep, int level, int64_t pair, int* ku, int* kv, double* u,
                 double* b, double* v) {
  return guard([&] {
    need(rep, "rep");
    const H1Rep& h = *rep->result.rep;
    const auto& ld = h.levels.at(size_t(level));
    if (ku) *ku = ld.ku.at(size_t(pair));
    if (kv) *kv = ld.kv.at(size_t(pair));
    if (!u && !b && !v) return;
    const LowRankBlockHost blk = h.block(level, int(pair));
    if (u) std::memcpy(u, blk.u.data(), size_t(blk.u.size()) * 8);
    if (b) std::memcpy(b, blk.b.data(), size_t(blk.b.size()) * 8);
    if (v) std::memcpy(v, blk.v.data(), size_t(blk.v.size()) * 8);
  });
}

int hp_rep_dense_block(const hp_rep* rep, int64_t pair, double* d) {
  return guard([&] {
    need(rep, "rep");
    need(d, "out");
    const Matrix m = rep->result.rep->dense_block(int(pair));
    std::memcpy(d, m.data(), size_t(m.size()) * 8);
  });
}

int hp_rep_apply(const hp_rep* rep, int adjoint, const double* x, int64_t w, double* y) {
  return guard([&] {
    need(rep, "rep");
    const H1Rep& h = *rep->result.rep;
    const Matrix r = h.apply(from_host(x, h.tree->num_points(), w), adjoint != 0);
    std::memcpy(y, r.data(), size_t(r.size()) * 8);
  });
}

int hp_rep_storage(const hp_rep* rep, int64_t* total) {
  return guard([&] {
    need(rep, "rep");
    need(total, "total");
    *total = rep->result.rep->storage_total();
  });
}

int hp_rep_sizes(const hp_rep* rep, int64_t* f, int64_t* d) {
  return guard([&] {
    need(rep, "rep");
    if (f) *f = rep->result.rep->factor_doubles;
    if (d) *d = rep->result.rep->dense_doubles;
  });
}

int hp_rep_export(const hp_rep* rep, double* hf, double* hd, int64_t* bytes) {
  return guard([&] {
    need(rep, "rep");
    need(hf, "host_factors");
    need(hd, "host_dense");
    const int64_t b = rep->result.rep->export_all(hf, hd);
    if (bytes) *bytes = b;
  });
}

int hp_export_sizes(const hp_tree* tree, int rank, int64_t* factor_doubles, int64_t* dense_doubles) {
  return guard([&] {
    need(tree, "tree");
    if (rank < 1) throw std::invalid_argument("fixed rank must be >= 1");
    export_sizes(*tree->tree, rank, factor_doubles, dense_doubles);
  });
}

int hp_host_alloc(int64_t bytes, void** out) {
  return guard([&] {
    need(out, "out");
    if (bytes < 0) throw std::invalid_argument("negative size");
    void* p = nullptr;
    const cudaError_t e = cudaHostAlloc(&p, size_t(bytes > 0 ? bytes : 1), cudaHostAllocPortable);
    if (e != cudaSuccess) throw std::runtime_error(std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    *out = p;
  });
}

void hp_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int hp_compress_export(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                       int format, int strategy, hp_comm* comm, double* host_factors,
                       int64_t factor_doubles, double* host_dense, int64_t dense_doubles,
                       hp_rep** out) {
  return guard([&] {
    need(op, "op");
    need(tree, "tree");
    need(out, "out");
    need(host_factors, "host_factors");
    need(host_dense, "host_dense");
    if (format < 0 || format > 3) throw std::invalid_argument("unknown format");
    std::int64_t nf = 0, nd = 0;
    if (rank >= 1)
      export_sizes(*tree->tree, rank, &nf, &nd, comm ? comm->comm->world() : 1, comm ? comm->comm->rank() : 0);
    if (factor_doubles < nf || dense_doubles < nd)
      throw std::invalid_argument("export arrays smaller than hp_export_sizes");
    PeelConfig cfg;
    cfg.rank = rank;
    cfg.oversample = oversample;
    cfg.leaf_capacity = tree->tree->leaf_capacity();
    cfg.seed = seed;
    cfg.format = PeelFormat(format);
    cfg.strategy = strategy == HP_STRATEGY_FALLBACK_PATTERN ? ColoringStrategy::kFallbackPattern
                                                            : ColoringStrategy::kGraph;
    cfg.comm = comm ? comm->comm.get() : nullptr;
    cfg.export_factors = host_factors;
    cfg.export_dense = host_dense;
    auto r = std::make_unique<hp_rep>();
    r->result = compress(*op->op, tree->tree, cfg);
    *out = r.release();
  });
}

int hp_rep_save(const hp_rep* rep, const char* path) {
  return guard([&] {
    need(rep, "rep");
    need(path, "path");
    save_rep(path, *rep->result.rep);
  });
}

int hp_rep_load(const char* path, int device, hp_rep** out, hp_tree** tree_out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    need(tree_out, "tree_out");
    auto r = std::make_unique<hp_rep>();
    r->result.rep = load_rep(path, device);
    auto t = std::make_unique<hp_tree>();
    t->tree = r->result.rep->tree;
    t->adj = r->result.rep->adj;
    t->layout = r->result.rep->layout;
    *tree_out = t.release();
    *out = r.release();
  });
}

int hp_save_dense_matrix(const char* path, const double* a, int64_t rows, int64_t cols) {
  return guard([&] {
    need(path, "path");
    if (rows < 0 || cols < 0) throw std::invalid_argument("negative shape");
    if (rows * cols > 0) need(a, "a");
    Matrix m(rows, cols);
    if (rows * cols > 0) std::memcpy(m.data(), a, size_t(rows * cols) * 8);
    save_dense_matrix(path, m);
  });
}

int hp_load_dense_matrix(const char* path, int64_t* rows, int64_t* cols, double* out, int64_t cap) {
  return guard([&] {
    need(path, "path");
    const Matrix m = load_dense_matrix(path);
    if (rows) *rows = m.rows();
    if (cols) *cols = m.cols();
    if (out) {
      if (cap < m.size()) throw std::invalid_argument("output buffer too small");
      std::memcpy(out, m.data(), size_t(m.size()) * 8);
    }
  });
}

namespace {
int captured_block(const hp_rep* rep, int level, int64_t pair, int64_t* rows, int64_t* cols, double* out,
                   bool raw) {
  return guard([&] {
    need(rep, "rep");
    const H1Rep& h = *rep->result.rep;
    const Matrix* m = nullptr;
    int box = -1;
    if (level < 0) {
      if (raw) throw std::invalid_argument("pre-peel captures exist for H1 levels only");
      m = &h.captured_leaf.at(size_t(pair));
      box = h.dense.pairs.at(size_t(pair)).first;
    } else {
      m = &(raw ? h.captured_raw : h.captured).at(level).at(size_t(pair));
      box = h.levels.at(size_t(level)).pairs.at(size_t(pair)).first;
    }
    if (rows) *rows = m->rows();
    if (cols) *cols = m->cols();
    if (!out) return;
    const auto& pts = h.tree->box(box).points;
    const int64_t st = h.layout->start[size_t(box)];
    for (size_t s = 0; s < pts.size(); ++s) {
      const int64_t tr = h.layout->inv[size_t(pts[s])] - st;
      for (int64_t c = 0; c < m->cols(); ++c) out[int64_t(s) + c * m->rows()] = (*m)(tr, c);
    }
  });
}
}  // namespace

int hp_rep_captured(const hp_rep* rep, int level, int64_t pair, int64_t* rows, int64_t* cols,
                    double* out) {
  return captured_block(rep, level, pair, rows, cols, out, false);
}

int hp_rep_captured_raw(const hp_rep* rep, int level, int64_t pair, int64_t* rows, int64_t* cols,
                        double* out) {
  return captured_block(rep, level, pair, rows, cols, out, true);
}

int hp_rel_error_power_method(const hp_rep* rep, const hp_op* op, int iters, uint64_t seed,
                              double* out) {
  return guard([&] {
    need(rep, "rep");
    need(op, "op");
    need(out, "out");
    *out = rel_error_power_method(*rep->result.rep, *op->op, iters, seed);
  });
}

int hp_debug_payload(const hp_tree* t, int level, int r, uint64_t seed, int device, double* out) {
  return guard([&] {
    need(t, "tree");
    need(out, "out");
    const Matrix m = debug_payload(*t->tree, *t->layout, level, r, seed, device);
    std::memcpy(out, m.data(), size_t(m.size()) * 8);
  });
}

int hp_debug_qr(const double* blocks, const int* rows, int nb, int cols, int kmax, int device,
                double* q, int* ranks, double* ms) {
  return guard([&] {
    need(blocks, "blocks");
    need(rows, "rows");
    need(q, "q");
    need(ranks, "ranks");
    if (nb < 0 || cols < 1 || cols > 160 || kmax < 0 || kmax > cols)
      throw std::invalid_argument("debug_qr: bad sizes");
    const double t = debug_qr(blocks, rows, nb, cols, kmax, device, q, ranks);
    if (ms) *ms = t;
  });
}

int hp_debug_log(const double* x, int64_t n, int device, double* out) {
  return guard([&] {
    need(x, "x");
    need(out, "out");
    debug_fast_log(x, n, out, device);
  });
}

}  // extern "C"
