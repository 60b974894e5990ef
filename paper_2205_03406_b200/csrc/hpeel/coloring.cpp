// Sampling plan; see coloring.hpp for the reference mapping.
#include "coloring.hpp"

#include <algorithm>
#include <atomic>
#include <functional>
#include <memory>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <queue>
#include <stdexcept>
#include <thread>
#include <tuple>
#include <unordered_map>

#include "rng.hpp"

namespace hpeel {

namespace {

// Constraint sets keyed by their literal (payload, zero) requirement
// (proj/src/coloring.cpp:26-51): a repeated requirement only gains an owner,
// so the first occurrence fixes the vertex id. Requirements are hashed and
// compared only within a hash bucket.
class RequirementTable {
 public:
  void add(std::vector<std::pair<int, PayloadTag>>&& payload, std::vector<int>&& zero, std::pair<int, int> owner) {
    const std::uint64_t h = digest(payload, zero);
    auto& bucket = by_hash_[h];
    for (int id : bucket) {
      ConstraintSet& s = sets_[size_t(id)];
      if (s.payload == payload && s.zero == zero) {
        s.owners.push_back(owner);
        return;
      }
    }
    bucket.push_back(int(sets_.size()));
    ConstraintSet s;
    s.payload = std::move(payload);
    s.zero = std::move(zero);
    s.owners.push_back(owner);
    sets_.push_back(std::move(s));
  }
  std::vector<ConstraintSet> release() { return std::move(sets_); }

 private:
  static std::uint64_t digest(const std::vector<std::pair<int, PayloadTag>>& payload, const std::vector<int>& zero) {
    std::uint64_t h = 0x84222325cbf29ce4ull;
    auto mix = [&](std::uint64_t v) { h = (h ^ v) * 0x100000001b3ull + (h >> 29); };
    for (const auto& [box, tag] : payload) mix((std::uint64_t(unsigned(box)) << 8) | std::uint64_t(tag));
    mix(~std::uint64_t(0));
    for (int z : zero) mix(std::uint64_t(unsigned(z)));
    return h;
  }
  std::unordered_map<std::uint64_t, std::vector<int>> by_hash_;
  std::vector<ConstraintSet> sets_;
};

// sorted union of sorted lists
std::vector<int> union_of(std::initializer_list<const std::vector<int>*> lists) {
  std::vector<int> out;
  for (const auto* l : lists) out.insert(out.end(), l->begin(), l->end());
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

// copy of a sorted list without one value
std::vector<int> without(const std::vector<int>& sorted, int value) {
  std::vector<int> out;
  out.reserve(sorted.size());
  const auto at = std::lower_bound(sorted.begin(), sorted.end(), value);
  out.insert(out.end(), sorted.begin(), at);
  out.insert(out.end(), at != sorted.end() && *at == value ? at + 1 : at, sorted.end());
  return out;
}

}  // namespace

std::vector<ConstraintSet> build_constraints(const BoxTree& tree, const AdjacencyInfo& adj,
                                             int level, SampleMode mode) {
  RequirementTable table;
  if (mode == SampleMode::kUnifStage2) {
    // (alpha, beta): adjoint-side probe carrying the alpha basis, observed at
    // I_beta; zero N(beta) u I(beta) u CL(beta) minus alpha
    std::vector<int> reach;
    for (const auto& [alpha, beta] : admissible_pairs(tree, adj, level)) {
      reach = union_of({&adj.neighbors[size_t(beta)], &adj.interaction[size_t(beta)],
                        &adj.coarse_leaf_neighbors[size_t(beta)]});
      table.add({{alpha, PayloadTag::kBasis}}, without(reach, alpha), {alpha, beta});
    }
  } else if (mode == SampleMode::kH1) {
    // (alpha, beta): payload {beta: Gaussian}, zero N(alpha) u I(alpha) u
    // CL(alpha) minus beta; one union per row box alpha
    std::vector<int> reach;
    int reach_of = -1;
    for (const auto& [alpha, beta] : admissible_pairs(tree, adj, level)) {
      if (alpha != reach_of) {
        reach = union_of({&adj.neighbors[size_t(alpha)], &adj.interaction[size_t(alpha)],
                          &adj.coarse_leaf_neighbors[size_t(alpha)]});
        reach_of = alpha;
      }
      table.add({{beta, PayloadTag::kGaussian}}, without(reach, beta), {alpha, beta});
    }
  } else if (mode == SampleMode::kUnifStage1) {
    if (level < 2 || level > tree.depth()) throw std::invalid_argument("sampling level out of range");
    // alpha: payload = every interaction box, zero = N(alpha) u CL(alpha)
    for (int alpha : tree.level_boxes(level)) {
      const auto& il = adj.interaction[size_t(alpha)];
      if (il.empty()) continue;
      std::vector<std::pair<int, PayloadTag>> payload;
      payload.reserve(il.size());
      for (int beta : il) payload.emplace_back(beta, PayloadTag::kGaussian);
      table.add(std::move(payload),
                union_of({&adj.neighbors[size_t(alpha)], &adj.coarse_leaf_neighbors[size_t(alpha)]}),
                {alpha, -1});
    }
  } else {
    // leaf probes (lambda, mu): identity payload on mu, zero = the other dense partners
    for (const auto& [lambda, mu] : dense_pairs(tree, adj))
      table.add({{mu, PayloadTag::kIdentity}}, without(adj.dense_partners[size_t(lambda)], mu), {lambda, mu});
  }
  return table.release();
}

bool incompatible(const ConstraintSet& a, const ConstraintSet& b) {
  // proj/src/coloring.cpp:115-146: a payload box of one set lies in the
  // other's zero set, or both carry a box with different tags. Payload lists
  // are short, so each entry is looked up in the other sorted lists.
  auto payload_hits_zero = [](const ConstraintSet& p, const ConstraintSet& z) {
    return std::any_of(p.payload.begin(), p.payload.end(), [&](const std::pair<int, PayloadTag>& e) {
      return std::binary_search(z.zero.begin(), z.zero.end(), e.first);
    });
  };
  if (payload_hits_zero(a, b) || payload_hits_zero(b, a)) return true;
  for (const auto& [box, tag] : a.payload) {
    const auto it = std::lower_bound(b.payload.begin(), b.payload.end(), box,
                                     [](const std::pair<int, PayloadTag>& e, int v) { return e.first < v; });
    if (it != b.payload.end() && it->first == box && it->second != tag) return true;
  }
  return false;
}

std::size_t IncompatibilityGraph::num_edges() const {
  std::size_t e = 0;
  for (const auto& a : edges) e += a.size();
  return e / 2;
}

int IncompatibilityGraph::max_degree() const {
  std::size_t d = 0;
  for (const auto& a : edges) d = std::max(d, a.size());
  return int(d);
}

IncompatibilityGraph build_graph(const std::vector<ConstraintSet>& sets) {
  IncompatibilityGraph g;
  g.num_vertices = int(sets.size());
  g.edges.resize(sets.size());
  int max_box = -1;
  for (const auto& s : sets) {
    for (auto& p : s.payload) max_box = std::max(max_box, p.first);
    for (int z : s.zero) max_box = std::max(max_box, z);
  }
  // CSR inverted indexes: which sets zero a box, which sets carry it.
  const size_t nb = size_t(max_box + 1);
  std::vector<int> zoff(nb + 1, 0), poff(nb + 1, 0);
  for (const auto& s : sets) {
    for (int z : s.zero) ++zoff[size_t(z) + 1];
    for (auto& p : s.payload) ++poff[size_t(p.first) + 1];
  }
  for (size_t b = 0; b < nb; ++b) {
    zoff[b + 1] += zoff[b];
    poff[b + 1] += poff[b];
  }
  std::vector<int> zsets(size_t(zoff[nb])), psets(size_t(poff[nb]));
  std::vector<PayloadTag> ptags(size_t(poff[nb]));
  {
    std::vector<int> zc(zoff.begin(), zoff.end() - 1), pc(poff.begin(), poff.end() - 1);
    for (size_t i = 0; i < sets.size(); ++i) {
      for (int z : sets[i].zero) zsets[size_t(zc[size_t(z)]++)] = int(i);
      for (auto& p : sets[i].payload) {
        ptags[size_t(pc[size_t(p.first)])] = p.second;
        psets[size_t(pc[size_t(p.first)]++)] = int(i);
      }
    }
  }
  // Neighbors of i, each list built independently (threads over vertices):
  // sets that zero one of i's payload boxes, sets whose payload box i zeroes,
  // and sets carrying one of i's payload boxes with another tag.
  auto neighbors = [&](size_t i, std::vector<int>& e) {
    for (auto& [box, tag] : sets[i].payload) {
      for (int k = zoff[size_t(box)]; k < zoff[size_t(box) + 1]; ++k) e.push_back(zsets[size_t(k)]);
      for (int k = poff[size_t(box)]; k < poff[size_t(box) + 1]; ++k)
        if (ptags[size_t(k)] != tag) e.push_back(psets[size_t(k)]);
    }
    for (int z : sets[i].zero)
      for (int k = poff[size_t(z)]; k < poff[size_t(z) + 1]; ++k) e.push_back(psets[size_t(k)]);
    std::sort(e.begin(), e.end());
    e.erase(std::unique(e.begin(), e.end()), e.end());
    auto self = std::lower_bound(e.begin(), e.end(), int(i));
    if (self != e.end() && *self == int(i)) e.erase(self);
  };
  const size_t n = sets.size();
  const unsigned nt = n < 4096 ? 1u : std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (;;) {
      const size_t b = next.fetch_add(256);
      if (b >= n) return;
      for (size_t i = b; i < std::min(n, b + 256); ++i) neighbors(i, g.edges[i]);
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  return g;
}

IncompatibilityGraph build_graph_pairwise(const std::vector<ConstraintSet>& sets) {
  IncompatibilityGraph g;
  g.num_vertices = int(sets.size());
  g.edges.resize(sets.size());
  for (size_t i = 0; i < sets.size(); ++i)
    for (size_t j = i + 1; j < sets.size(); ++j)
      if (incompatible(sets[i], sets[j])) {
        g.edges[i].push_back(int(j));
        g.edges[j].push_back(int(i));
      }
  return g;
}

namespace {
// 4-ary max-heap of packed 64-bit keys (smaller and shallower than a binary
// heap of tuples: the DSatur queue sees ~V x colors pushes on leaf graphs)
class KeyHeap {
 public:
  void reserve(size_t n) { h_.reserve(n); }
  bool empty() const { return h_.empty(); }
  std::uint64_t top() const { return h_[0]; }
  void push(std::uint64_t k) {
    size_t i = h_.size();
    h_.push_back(k);
    while (i > 0) {
      const size_t p = (i - 1) >> 2;
      if (h_[p] >= k) break;
      h_[i] = h_[p];
      i = p;
    }
    h_[i] = k;
  }
  void pop() {
    const std::uint64_t k = h_.back();
    h_.pop_back();
    const size_t n = h_.size();
    if (n == 0) return;
    size_t i = 0;
    for (;;) {
      const size_t c0 = 4 * i + 1;
      if (c0 >= n) break;
      size_t best = c0;
      const size_t ce = std::min(n, c0 + 4);
      for (size_t c = c0 + 1; c < ce; ++c)
        if (h_[c] > h_[best]) best = c;
      if (h_[best] <= k) break;
      h_[i] = h_[best];
      i = best;
    }
    h_[i] = k;
  }

 private:
  std::vector<std::uint64_t> h_;
};

}  // namespace

template <class Degree, class Sweep>
Coloring dsatur_impl(int n, Degree&& degree, Sweep&& sweep) {
  Coloring out;
  out.color.assign(size_t(n), -1);
  if (n == 0) return out;
  // Selection = max (saturation, uncolored degree, -v) over uncolored
  // vertices, as the reference's eager heap (proj/src/coloring.cpp:184-213).
  // Queue: one lazy max-heap of (uncolored degree, -v) per saturation value;
  // a vertex is pushed into bucket sat whenever its saturation rises, so the
  // highest non-empty bucket holds every candidate. A popped entry whose
  // vertex is colored or has moved to a higher bucket is dropped; one with an
  // outdated degree is re-pushed with the current degree; a popped entry that
  // is exactly current dominates its bucket -- the selection is identical to
  // the eager heap with far fewer and shallower queue operations.
  // Per-vertex state is one 16-byte record (color, saturation, uncolored
  // degree) plus a flat neighbor-color bitset of W words (grown on demand),
  // and the neighbor sweep prefetches ahead.
  struct VState {
    int color;
    int sat;
    int udeg;
    int pad;
  };
  auto key = [](int udeg, int v) {
    return (std::uint64_t(unsigned(udeg)) << 32) | (0xFFFFFFFFull - std::uint64_t(unsigned(v)));
  };
  std::vector<VState> st(static_cast<size_t>(n));
  size_t words = 4;
  std::vector<std::uint64_t> seen(size_t(n) * words, 0);
  std::vector<KeyHeap> bucket(1);
  bucket[0].reserve(size_t(n));
  for (int v = 0; v < n; ++v) {
    const int d = degree(v);
    st[size_t(v)] = VState{-1, 0, d, 0};
    bucket[0].push(key(d, v));
  }
  out.queue_ops += size_t(n);
  int top = 0;  // highest bucket that may be non-empty
  int done = 0;
  while (done < n) {
    while (bucket[size_t(top)].empty()) --top;
    KeyHeap& hb = bucket[size_t(top)];
    const std::uint64_t k = hb.top();
    hb.pop();
    ++out.queue_ops;
    const int ud = int(k >> 32);
    const int v = int(0xFFFFFFFFull - (k & 0xFFFFFFFFull));
    VState& sv = st[size_t(v)];
    if (sv.color != -1 || sv.sat != top) continue;
    if (ud != sv.udeg) {
      hb.push(key(sv.udeg, v));
      ++out.queue_ops;
      continue;
    }
    // smallest color absent among the neighbors
    const std::uint64_t* row = seen.data() + size_t(v) * words;
    size_t wi = 0;
    while (wi < words && row[wi] == ~std::uint64_t(0)) ++wi;
    const int c = int(64 * wi) + (wi < words ? __builtin_ctzll(~row[wi]) : 0);
    if (size_t(c) >= 64 * words) {
      std::vector<std::uint64_t> grown(size_t(n) * words * 2, 0);
      for (size_t u = 0; u < size_t(n); ++u)
        std::copy(seen.begin() + std::ptrdiff_t(u * words), seen.begin() + std::ptrdiff_t((u + 1) * words),
                  grown.begin() + std::ptrdiff_t(u * words * 2));
      seen.swap(grown);
      words *= 2;
    }
    sv.color = c;
    out.color[size_t(v)] = c;
    out.num_colors = std::max(out.num_colors, c + 1);
    ++done;
    const size_t cw = size_t(c) >> 6;
    const std::uint64_t cb = std::uint64_t(1) << (c & 63);
    auto visit = [&](int w) {
      VState& sw = st[size_t(w)];
      if (sw.color != -1) return;
      --sw.udeg;
      std::uint64_t& word = seen[size_t(w) * words + cw];
      if (!(word & cb)) {
        word |= cb;
        const int ns = ++sw.sat;
        if (size_t(ns) >= bucket.size()) bucket.resize(size_t(ns) + 1);
        bucket[size_t(ns)].push(key(sw.udeg, w));
        if (ns > top) top = ns;
        ++out.queue_ops;
      }
    };
    sweep(v, visit, st, seen, words, cw);
  }
  return out;
}

Coloring dsatur_color(const IncompatibilityGraph& graph) {
  return dsatur_impl(
      graph.num_vertices, [&](int v) { return int(graph.edges[size_t(v)].size()); },
      [&](int v, auto&& visit, auto& st, auto& seen, size_t words, size_t cw) {
        constexpr int kAhead = 12;
        const std::vector<int>& nb = graph.edges[size_t(v)];
        const size_t m = nb.size();
        for (size_t i = 0; i < m; ++i) {
          if (i + kAhead < m) {
            const size_t u = size_t(nb[i + kAhead]);
            __builtin_prefetch(&st[u], 1, 1);
            __builtin_prefetch(&seen[u * words + cw], 1, 1);
          }
          visit(nb[i]);
        }
      });
}

namespace {

// Max tournament tree over the vertices' packed DSatur keys
// (saturation, uncolored degree, -v). Keys are lazy upper bounds: the
// saturation part is exact, the degree part may be stale-high (degree
// decrements are not propagated), so the selection re-keys a stale winner and
// looks again -- a winner whose stored key is exact beats every true key.
// Saturation increases only raise a key: `raise` is safe from several
// threads (compare-and-swap maximum up the path, stopping where an ancestor
// already dominates); `set` is single-threaded.
class KeyTree {
 public:
  explicit KeyTree(int n) {
    while (size_ < size_t(std::max(n, 1))) size_ <<= 1;
    node_ = std::vector<std::atomic<std::uint64_t>>(2 * size_);
    for (auto& x : node_) x.store(0, std::memory_order_relaxed);
  }
  void init(int v, std::uint64_t k) { node_[size_ + size_t(v)].store(k, std::memory_order_relaxed); }
  void build() {
    for (size_t i = size_ - 1; i >= 1; --i) node_[i].store(std::max(get(2 * i), get(2 * i + 1)), std::memory_order_relaxed);
  }
  std::uint64_t leaf(int v) const { return get(size_ + size_t(v)); }
  void raise(int v, std::uint64_t k) {
    size_t i = size_ + size_t(v);
    node_[i].store(k, std::memory_order_relaxed);
    for (i >>= 1; i >= 1; i >>= 1) {
      std::uint64_t cur = node_[i].load(std::memory_order_relaxed);
      bool raised = false;
      while (cur < k)
        if (node_[i].compare_exchange_weak(cur, k, std::memory_order_relaxed)) {
          raised = true;
          break;
        }
      if (!raised) return;
    }
  }
  // raise from one thread only (no other thread touches the tree)
  void raise_serial(int v, std::uint64_t k) {
    size_t i = size_ + size_t(v);
    node_[i].store(k, std::memory_order_relaxed);
    for (i >>= 1; i >= 1 && get(i) < k; i >>= 1) node_[i].store(k, std::memory_order_relaxed);
  }
  void set(int v, std::uint64_t k) {
    size_t i = size_ + size_t(v);
    node_[i].store(k, std::memory_order_relaxed);
    for (i >>= 1; i >= 1; i >>= 1) node_[i].store(std::max(get(2 * i), get(2 * i + 1)), std::memory_order_relaxed);
  }
  int argmax() const {
    size_t i = 1;
    while (i < size_) i = get(2 * i) >= get(2 * i + 1) ? 2 * i : 2 * i + 1;
    return int(i - size_);
  }

 private:
  std::uint64_t get(size_t i) const { return node_[i].load(std::memory_order_relaxed); }
  size_t size_ = 1;
  std::vector<std::atomic<std::uint64_t>> node_;
};

// Spinning worker team for the neighbor sweeps (a sweep is ~10 us of work:
// thread start-up or a condition variable per sweep would cost more).
class SpinTeam {
 public:
  explicit SpinTeam(int workers) {
    for (int t = 0; t < workers; ++t) threads_.emplace_back([this, t] { loop(t + 1); });
  }
  ~SpinTeam() {
    stop_.store(true, std::memory_order_release);
    epoch_.fetch_add(1, std::memory_order_acq_rel);
    for (auto& th : threads_) th.join();
  }
  int size() const { return int(threads_.size()) + 1; }
  // run job(t) on every member t (0 = the caller) and wait for all
  template <class F>
  void run(F&& job) {
    job_ = [&](int t) { job(t); };
    pending_.store(int(threads_.size()), std::memory_order_relaxed);
    epoch_.fetch_add(1, std::memory_order_acq_rel);
    job(0);
    while (pending_.load(std::memory_order_acquire) != 0) pause();
  }

 private:
  static void pause() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  void loop(int t) {
    std::uint64_t seen = 0;
    for (;;) {
      std::uint64_t e;
      while ((e = epoch_.load(std::memory_order_acquire)) == seen) pause();
      seen = e;
      if (stop_.load(std::memory_order_acquire)) return;
      job_(t);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> threads_;
  std::function<void(int)> job_;
  std::atomic<std::uint64_t> epoch_{0};
  std::atomic<int> pending_{0};
  std::atomic<bool> stop_{false};
};

}  // namespace

// DSatur on the implicit graph (same selection rule and result as
// dsatur_impl): the tournament tree replaces the per-saturation heaps, and
// the sweeps of high-degree vertices run on a spinning thread team -- first
// the sets whose zero set holds v's payload box (each once), then, after a
// barrier, the sets carrying a box of v's zero set that the first part did
// not reach; every neighbor is updated by exactly one thread.
Coloring dsatur_heap(const ImplicitGraph& graph) {
  std::vector<int> stamp(size_t(graph.num_vertices()), -1);
  return dsatur_impl(graph.num_vertices(), [&](int v) { return graph.degree(v); },
                     [&](int v, auto&& visit, auto&, auto&, size_t, size_t) {
                       graph.for_each_neighbor(v, stamp, v, visit);
                     });
}

Coloring dsatur_color_threaded(const ImplicitGraph& graph, int threads) {
  const int n = graph.num_vertices();
  Coloring out;
  out.color.assign(size_t(n), -1);
  if (n == 0) return out;
  constexpr int kSatBits = 14, kDegBits = 26, kVBits = 24;
  int max_deg = 0;
  for (int v = 0; v < n; ++v) max_deg = std::max(max_deg, graph.degree(v));
  if (n >= (1 << kVBits) - 1 || max_deg >= (1 << kDegBits)) return dsatur_heap(graph);
  auto key = [](int sat, int udeg, int v) {
    return (std::uint64_t(unsigned(sat)) << (kDegBits + kVBits)) | (std::uint64_t(unsigned(udeg)) << kVBits) |
           std::uint64_t((1u << kVBits) - 1u - unsigned(v));
  };
  auto key_deg = [](std::uint64_t k) { return int((k >> kVBits) & ((1u << kDegBits) - 1u)); };
  struct VState {
    int color, sat, udeg, stamp;
  };
  std::vector<VState> st(static_cast<size_t>(n));
  // neighbor-color bits color-major: plane q holds colors [64 q, 64 q + 64)
  // of every vertex, so a sweep (one color) touches one n-word plane
  std::vector<std::vector<std::uint64_t>> seen;
  seen.emplace_back(static_cast<size_t>(n), 0);
  KeyTree tree(n);
  for (int v = 0; v < n; ++v) {
    st[size_t(v)] = VState{-1, 0, graph.degree(v), -1};
    tree.init(v, key(0, graph.degree(v), v));
  }
  tree.build();
  out.queue_ops += size_t(n);
  std::unique_ptr<SpinTeam> team;
  if (threads > 1) team = std::make_unique<SpinTeam>(threads - 1);
  const int nt = team ? team->size() : 1;
  std::atomic<int> zcursor{0};
  bool sat_overflow = false;
  static const bool prof = std::getenv("HP_DSATUR_PROFILE") != nullptr;
  using PClock = std::chrono::steady_clock;
  double t_sel = 0, t_sweep = 0;
  std::size_t n_threaded = 0, rekeys = 0, cand1 = 0, cand2 = 0;
  auto tp = PClock::now();
  auto lapp = [&](double& acc) {
    if (!prof) return;
    const auto t1 = PClock::now();
    acc += std::chrono::duration<double>(t1 - tp).count();
    tp = t1;
  };
  for (int done = 0; done < n; ++done) {
    lapp(t_sweep);
    int v;
    for (;;) {
      v = tree.argmax();
      const std::uint64_t k = tree.leaf(v);
      if (key_deg(k) == st[size_t(v)].udeg) break;
      tree.set(v, key(st[size_t(v)].sat, st[size_t(v)].udeg, v));  // stale degree: re-key, look again
      ++out.queue_ops;
      ++rekeys;
    }
    VState& sv = st[size_t(v)];
    size_t wi = 0;
    while (wi < seen.size() && seen[wi][size_t(v)] == ~std::uint64_t(0)) ++wi;
    const int c = int(64 * wi) + (wi < seen.size() ? __builtin_ctzll(~seen[wi][size_t(v)]) : 0);
    if (size_t(c >> 6) >= seen.size()) seen.emplace_back(static_cast<size_t>(n), 0);
    if (c + 1 >= (1 << kSatBits)) sat_overflow = true;
    sv.color = c;
    out.color[size_t(v)] = c;
    out.num_colors = std::max(out.num_colors, c + 1);
    tree.set(v, 0);
    lapp(t_sel);
    std::uint64_t* plane = seen[size_t(c) >> 6].data();
    const std::uint64_t cb = std::uint64_t(1) << (c & 63);
    auto visit = [&](int w) {
      VState& sw = st[size_t(w)];
      if (sw.color != -1) return;
      --sw.udeg;
      std::uint64_t& word = plane[size_t(w)];
      if (!(word & cb)) {
        word |= cb;
        ++sw.sat;
        tree.raise(w, key(sw.sat, sw.udeg, w));  // concurrent-safe maximum up the path
      }
    };
    const int pb = graph.payload_box(v);
    const int* z0 = graph.zero_sets_begin(pb);
    const int* z1 = graph.zero_sets_end(pb);
    const auto& zero = graph.zero_of(v);
    static const int sweep_min =
        std::getenv("HP_DSATUR_SWEEP_MIN") ? std::atoi(std::getenv("HP_DSATUR_SWEEP_MIN")) : 4096;
    if (!team || graph.degree(v) < sweep_min) {
      // serial sweep
      sv.stamp = v;
      for (const int* q = z0; q < z1; ++q)
        if (st[size_t(*q)].stamp != v) {
          st[size_t(*q)].stamp = v;
          visit(*q);
        }
      for (int z : zero)
        for (const int* q = graph.payload_sets_begin(z); q < graph.payload_sets_end(z); ++q)
          if (st[size_t(*q)].stamp != v) {
            st[size_t(*q)].stamp = v;
            visit(*q);
          }
      out.queue_ops += 1;
      continue;
    }
    ++n_threaded;
    if (prof) {
      cand1 += std::size_t(z1 - z0);
      for (int z : zero) cand2 += std::size_t(graph.payload_sets_end(z) - graph.payload_sets_begin(z));
    }
    // threaded sweep: part 1 (each set once) in static slices; part 2 over
    // the zero boxes, skipping part 1's sets and v itself
    sv.stamp = v;
    const std::int64_t n1 = z1 - z0;
    constexpr int kAhead = 16;  // prefetch distance: the visits are independent cache misses
    auto prefetch = [&](int w) {
      __builtin_prefetch(&st[size_t(w)], 1, 1);
      __builtin_prefetch(&plane[size_t(w)], 1, 1);
    };
    team->run([&](int t) {
      const std::int64_t a = n1 * t / nt, b = n1 * (t + 1) / nt;
      for (std::int64_t q = a; q < b; ++q) {
        if (q + kAhead < b) prefetch(z0[q + kAhead]);
        const int w = z0[q];
        if (w == v) continue;
        st[size_t(w)].stamp = v;
        visit(w);
      }
    });
    zcursor.store(0, std::memory_order_relaxed);
    const int nz = int(zero.size());
    team->run([&](int) {
      for (;;) {
        const int i0 = zcursor.fetch_add(4, std::memory_order_relaxed);
        if (i0 >= nz) return;
        for (int i = i0; i < std::min(nz, i0 + 4); ++i) {
          const int z = zero[size_t(i)];
          const int* qe = graph.payload_sets_end(z);
          for (const int* q = graph.payload_sets_begin(z); q < qe; ++q) {
            if (q + kAhead < qe) prefetch(q[kAhead]);
            if (st[size_t(*q)].stamp != v) visit(*q);
          }
        }
      }
    });
    out.queue_ops += 1;
  }
  lapp(t_sweep);
  if (prof)
    std::fprintf(stderr,
                 "[dsatur] n %d threads %d select %.2f s (re-keys %zu) sweeps %.2f s (threaded %zu, candidates %zu + %zu)\n",
                 n, nt, t_sel, rekeys, t_sweep, n_threaded, cand1, cand2);
  if (sat_overflow) return dsatur_heap(graph);
  return out;
}

Coloring dsatur_color(const ImplicitGraph& graph, int threads) {
  // the tournament-tree selection is also the faster serial one (config 3
  // plans: 127 -> 65 ms); HP_DSATUR_HEAP=1 keeps the heap implementation
  static const bool heap = std::getenv("HP_DSATUR_HEAP") != nullptr;
  if (!heap) return dsatur_color_threaded(graph, std::max(threads, 1));
  std::vector<int> stamp(size_t(graph.num_vertices()), -1);
  return dsatur_impl(graph.num_vertices(), [&](int v) { return graph.degree(v); },
                     [&](int v, auto&& visit, auto&, auto&, size_t, size_t) {
                       graph.for_each_neighbor(v, stamp, v, visit);
                     });
}

Coloring dsatur_color(const ImplicitGraph& graph) {
  // large leaf graphs (config 4: 3.9e5 vertices, 1.5e9 edges) on a thread team
  static const int env = std::getenv("HP_DSATUR_THREADS") ? std::atoi(std::getenv("HP_DSATUR_THREADS")) : -1;
  int threads = env;
  if (threads < 0) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    // measured (8 cores): 1.0-1.2e8 edges (configs 4 / 5 at 1/4 size) color in 0.84-0.96 s on one
    // thread and 1.0-1.3 s on a team; 1.5e9 edges (config 4) in 58 s vs 22 s
    threads = graph.num_edges() > 500'000'000 ? int(std::min(16u, hw)) : 1;
  }
  return dsatur_color(graph, threads);
}

bool ImplicitGraph::applicable(const std::vector<ConstraintSet>& sets) {
  if (sets.empty()) return true;
  const PayloadTag t0 = sets[0].payload.empty() ? PayloadTag::kGaussian : sets[0].payload[0].second;
  for (const auto& s : sets)
    if (s.payload.size() != 1 || s.payload[0].second != t0) return false;
  return true;
}

ImplicitGraph::ImplicitGraph(const std::vector<ConstraintSet>& sets) : sets_(&sets) {
  n_ = int(sets.size());
  int max_box = -1;
  payload_.resize(sets.size());
  for (size_t i = 0; i < sets.size(); ++i) {
    payload_[i] = sets[i].payload[0].first;
    max_box = std::max(max_box, payload_[i]);
    for (int z : sets[i].zero) max_box = std::max(max_box, z);
  }
  const size_t nb = size_t(max_box + 1);
  zoff_.assign(nb + 1, 0);
  poff_.assign(nb + 1, 0);
  for (size_t i = 0; i < sets.size(); ++i) {
    for (int z : sets[i].zero) ++zoff_[size_t(z) + 1];
    ++poff_[size_t(payload_[i]) + 1];
  }
  for (size_t b = 0; b < nb; ++b) {
    zoff_[b + 1] += zoff_[b];
    poff_[b + 1] += poff_[b];
  }
  zsets_.resize(size_t(zoff_[nb]));
  psets_.resize(size_t(poff_[nb]));
  {
    std::vector<int> zc(zoff_.begin(), zoff_.end() - 1), pc(poff_.begin(), poff_.end() - 1);
    for (size_t i = 0; i < sets.size(); ++i) {
      for (int z : sets[i].zero) zsets_[size_t(zc[size_t(z)]++)] = int(i);
      psets_[size_t(pc[size_t(payload_[i])]++)] = int(i);
    }
  }
  // degrees: threads over vertices, each with its own stamp array
  deg_.assign(sets.size(), 0);
  const size_t n = sets.size();
  const unsigned nt = n < 4096 ? 1u : std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::atomic<size_t> next{0};
  std::atomic<std::size_t> total{0};
  auto work = [&] {
    std::vector<int> stamp(n, -1);
    std::size_t local = 0;
    for (;;) {
      const size_t b = next.fetch_add(256);
      if (b >= n) break;
      for (size_t i = b; i < std::min(n, b + 256); ++i) {
        int d = 0;
        for_each_neighbor(int(i), stamp, int(i), [&](int) { ++d; });
        deg_[i] = d;
        local += size_t(d);
      }
    }
    total += local;
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  edges2_ = total.load();
}

Coloring plan_coloring(const BoxTree& tree, const std::vector<ConstraintSet>& sets,
                       const IncompatibilityGraph& graph, SampleMode mode) {
  return plan_coloring(tree, sets, dsatur_color(graph), mode);
}

Coloring plan_coloring(const BoxTree& tree, const std::vector<ConstraintSet>& sets, Coloring dsatur,
                       SampleMode mode) {
  Coloring best = std::move(dsatur);
  if (mode == SampleMode::kUnifStage2 || !tree.is_fully_populated()) return best;
  const int mod = mode == SampleMode::kH1 ? 6 : mode == SampleMode::kUnifStage1 ? 5 : 3;
  std::vector<int> tile(sets.size());
  std::map<int, int> relabel;
  for (size_t i = 0; i < sets.size(); ++i) {
    const int box = mode == SampleMode::kUnifStage1 ? sets[i].owners.front().first
                                                    : sets[i].payload.front().first;
    int idx = 0, mul = 1;
    for (std::int64_t c : tree.box(box).coord) {
      idx += int(c % mod) * mul;
      mul *= mod;
    }
    auto ins = relabel.emplace(idx, int(relabel.size()));
    tile[i] = ins.first->second;
  }
  if (int(relabel.size()) < best.num_colors) {
    best.color = std::move(tile);
    best.num_colors = int(relabel.size());
  }
  return best;
}

Matrix gaussian_matrix(Index rows, Index cols, std::uint64_t seed) {
  if (rows < 0 || cols < 0) throw std::invalid_argument("negative shape");
  Matrix out(rows, cols);
  SplitMix64 stream(seed);
  bool have_spare = false;
  double spare = 0.0;
  for (Index i = 0; i < rows; ++i) {
    for (Index j = 0; j < cols; ++j) {
      if (have_spare) {
        out(i, j) = spare;
        have_spare = false;
        continue;
      }
      const double u1 = stream.next_open_closed();
      const double u2 = stream.next_closed_open();
      const double radius = std::sqrt(-2.0 * std::log(u1));
      const double angle = 2.0 * M_PI * u2;
      out(i, j) = radius * std::cos(angle);
      spare = radius * std::sin(angle);
      have_spare = true;
    }
  }
  return out;
}

Matrix payload_gaussian(const BoxTree& tree, int box, int width, std::uint64_t seed, int level,
                        int phase) {
  return gaussian_matrix(Index(tree.box(box).points.size()), width,
                         payload_seed(seed, level, box, phase));
}

Matrix BlockTestMatrix::realize(const BoxTree& tree) const {
  Matrix out(rows, width);
  for (auto [box, tag] : payload) {
    const auto& pts = tree.box(box).points;
    if (tag == PayloadTag::kGaussian) {
      const Matrix g = payload_gaussian(tree, box, width, seed, level, phase);
      for (size_t r = 0; r < pts.size(); ++r)
        for (int c = 0; c < width; ++c) out(pts[r], c) = g(Index(r), c);
    } else if (tag == PayloadTag::kIdentity) {
      for (size_t r = 0; r < pts.size(); ++r)
        for (int c = 0; c < width; ++c) out(pts[r], c) = (Index(r) == c) ? 1.0 : 0.0;
    } else {
      throw std::runtime_error("missing basis for payload box");
    }
  }
  return out;
}

std::vector<BlockTestMatrix> assemble_test_matrices(const std::vector<ConstraintSet>& sets,
                                                    const Coloring& coloring, const BoxTree& tree,
                                                    int level, int width, std::uint64_t seed,
                                                    int phase) {
  std::vector<BlockTestMatrix> mats(size_t(coloring.num_colors));
  std::vector<std::map<int, PayloadTag>> merged(size_t(coloring.num_colors));
  std::vector<std::vector<int>> zeros(size_t(coloring.num_colors));
  for (size_t i = 0; i < sets.size(); ++i) {
    const int c = coloring.color[i];
    mats[size_t(c)].serves.push_back(int(i));
    for (auto [box, tag] : sets[i].payload) {
      auto ins = merged[size_t(c)].emplace(box, tag);
      if (!ins.second && ins.first->second != tag) {
        throw std::logic_error("conflicting payload tags within a color");
      }
    }
    zeros[size_t(c)].insert(zeros[size_t(c)].end(), sets[i].zero.begin(), sets[i].zero.end());
  }
  for (int c = 0; c < coloring.num_colors; ++c) {
    auto& m = mats[size_t(c)];
    m.payload.assign(merged[size_t(c)].begin(), merged[size_t(c)].end());
    auto& z = zeros[size_t(c)];
    std::sort(z.begin(), z.end());
    z.erase(std::unique(z.begin(), z.end()), z.end());
    m.zero = std::move(z);
    m.rows = tree.num_points();
    m.level = level;
    m.seed = seed;
    m.phase = phase;
    m.width = width;
  }
  return mats;
}

namespace {
int pattern_modulus(SampleMode mode) {
  return mode == SampleMode::kH1 ? 6 : mode == SampleMode::kUnifStage1 ? 5 : 3;
}
}  // namespace

int pattern_index(const Box& box, int mod) {
  int idx = 0, weight = 1;
  for (const std::int64_t c : box.coord) {
    idx += int(c % mod) * weight;
    weight *= mod;
  }
  return idx;
}

std::vector<BlockTestMatrix> fallback_pattern_matrices(const BoxTree& tree, const AdjacencyInfo&, int level,
                                                       SampleMode mode, int width, std::uint64_t seed,
                                                       int phase) {
  if (!tree.is_fully_populated())
    throw std::invalid_argument("pattern test matrices require a fully populated uniform tree");
  if (mode == SampleMode::kUnifStage2) throw std::invalid_argument("no pattern construction for basis probes");
  if (mode == SampleMode::kLeaf) level = tree.depth();
  if (level < 2 || level > tree.depth()) throw std::invalid_argument("sampling level out of range");
  const int d = tree.dim(), mod = pattern_modulus(mode);
  int count = 1;
  for (int j = 0; j < d; ++j) count *= mod;
  std::vector<BlockTestMatrix> mats(static_cast<size_t>(count));
  for (BlockTestMatrix& m : mats) {
    m.rows = tree.num_points();
    m.width = width;
    m.seed = seed;
    m.level = level;
    m.phase = phase;
  }
  const PayloadTag tag = mode == SampleMode::kLeaf ? PayloadTag::kIdentity : PayloadTag::kGaussian;
  // One pass over the level (ascending ids keep every list sorted): a box
  // carries payload in the one pattern its coordinates select (pairs, leaf
  // probes) or in every pattern whose shifted 3^d clusters miss it (stage 1).
  std::vector<char> active(static_cast<size_t>(count), 0);
  for (const int id : tree.level_boxes(level)) {
    const Box& b = tree.box(id);
    if (mode == SampleMode::kUnifStage1) {
      for (int idx = 0; idx < count; ++idx) {
        bool in_cluster = true;
        for (int j = 0, rem = idx; j < d && in_cluster; ++j, rem /= mod) {
          const int rel = int(((b.coord[size_t(j)] - rem % mod) % mod + mod) % mod);
          in_cluster = rel == 0 || rel == 1 || rel == mod - 1;
        }
        active[size_t(idx)] = !in_cluster;
      }
    } else {
      std::fill(active.begin(), active.end(), 0);
      active[size_t(pattern_index(b, mod))] = 1;
    }
    for (int idx = 0; idx < count; ++idx) {
      if (active[size_t(idx)])
        mats[size_t(idx)].payload.emplace_back(id, tag);
      else
        mats[size_t(idx)].zero.push_back(id);
    }
  }
  return mats;
}

SamplingPlan make_plan(const BoxTree& tree, const AdjacencyInfo& adj, int level, SampleMode mode,
                       int width, std::uint64_t seed, int phase, bool pattern) {
  SamplingPlan plan;
  if (pattern && mode != SampleMode::kUnifStage2) {  // basis probes always go through the graph
    plan.matrices = fallback_pattern_matrices(tree, adj, level, mode, width, seed, phase);
    const int mod = pattern_modulus(mode);
    if (mode == SampleMode::kH1) {
      for (const auto& [a, b] : admissible_pairs(tree, adj, level))
        plan.block_to_matrix[{a, b}] = pattern_index(tree.box(b), mod);
    } else if (mode == SampleMode::kUnifStage1) {
      for (const int a : tree.level_boxes(level))
        if (!adj.interaction[size_t(a)].empty()) plan.block_to_matrix[{a, -1}] = pattern_index(tree.box(a), mod);
    } else {
      for (const auto& [lam, mu] : dense_pairs(tree, adj))
        plan.block_to_matrix[{lam, mu}] = pattern_index(tree.box(mu), mod);
    }
    return plan;
  }
  static const bool timing = std::getenv("HP_PLAN_TIMING") != nullptr;
  using Clock = std::chrono::steady_clock;
  auto t0 = Clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = Clock::now();
    std::fprintf(stderr, "[plan l=%d mode=%d] %s %.1f ms\n", level, int(mode), what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const auto sets = build_constraints(tree, adj, level, mode);
  lap("constraints");
  if (sets.empty()) return plan;
  Coloring coloring;
  if (ImplicitGraph::applicable(sets)) {
    const ImplicitGraph graph(sets);
    lap("graph (implicit: degrees)");
    coloring = plan_coloring(tree, sets, dsatur_color(graph), mode);
    plan.n_edges = graph.num_edges();
  } else {
    const auto graph = build_graph(sets);
    lap("graph");
    coloring = plan_coloring(tree, sets, graph, mode);
    plan.n_edges = graph.num_edges();
  }
  lap("coloring");
  plan.n_vertices = sets.size();
  plan.matrices = assemble_test_matrices(sets, coloring, tree, level, width, seed, phase);
  lap("matrices");
  for (size_t i = 0; i < sets.size(); ++i)
    for (const auto& owner : sets[i].owners) plan.block_to_matrix[owner] = coloring.color[i];
  lap("block map");
  return plan;
}

}  // namespace hpeel
