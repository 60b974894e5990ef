// Sampling plan: constraint sets, incompatibility graph, DSatur, tile
// coloring and per-color block test matrices.
//
// Restates proj/include/hpeel/coloring.hpp:14-113 and
// proj/src/coloring.cpp:14-332 for the H1 (kH1) and leaf (kLeaf) modes on the
// hot path. `build_graph` produces the reference's edge set through an
// inverted box index instead of the O(V^2) pairwise scan of
// proj/src/coloring.cpp:154-167; DSatur depends only on the edge set and the
// vertex numbering (proj/src/coloring.cpp:169-216), so colorings are
// bit-identical. `build_graph_pairwise` keeps the literal scan for tests.
#pragma once

#include <cstdint>
#include <map>
#include <utility>
#include <vector>

#include "box_tree.hpp"

namespace hpeel {

enum class PayloadTag : std::uint8_t { kGaussian = 0, kIdentity = 1, kBasis = 2 };
enum class SampleMode : std::uint8_t { kH1 = 0, kUnifStage1 = 1, kUnifStage2 = 2, kLeaf = 3 };

struct ConstraintSet {
  std::vector<std::pair<int, PayloadTag>> payload;  // sorted by box id
  std::vector<int> zero;                            // sorted
  std::vector<std::pair<int, int>> owners;
  bool same_requirements(const ConstraintSet& o) const {
    return payload == o.payload && zero == o.zero;
  }
};

/// proj/src/coloring.cpp:55-113: kH1, kUnifStage1, kUnifStage2 (basis
/// payloads: the uniform driver supplies the bases) and kLeaf.
std::vector<ConstraintSet> build_constraints(const BoxTree& tree, const AdjacencyInfo& adj,
                                             int level, SampleMode mode);

struct IncompatibilityGraph {
  int num_vertices = 0;
  std::vector<std::vector<int>> edges;  // sorted adjacency
  std::size_t num_edges() const;
  int max_degree() const;
};

/// proj/src/coloring.cpp:115-146.
bool incompatible(const ConstraintSet& a, const ConstraintSet& b);

/// Same edge set as the reference's pairwise scan, via an inverted index.
IncompatibilityGraph build_graph(const std::vector<ConstraintSet>& sets);
/// Literal O(V^2) scan of proj/src/coloring.cpp:154-167 (tests only).
IncompatibilityGraph build_graph_pairwise(const std::vector<ConstraintSet>& sets);

struct Coloring {
  std::vector<int> color;
  int num_colors = 0;
  std::size_t queue_ops = 0;
};

/// proj/src/coloring.cpp:169-216: max (saturation, uncolored degree, -v),
/// smallest free color; same lazy max-heap, so queue_ops match.
Coloring dsatur_color(const IncompatibilityGraph& graph);

/// The same incompatibility graph without materializing it, for sets with
/// one payload box each and a single payload tag (the H1 and leaf modes):
/// N(v) = {sets whose zero set holds v's payload box} U {sets whose payload
/// box is in v's zero set}, enumerated from two box -> set indexes with a
/// stamp array. Degrees are counted in parallel; DSatur walks the same
/// neighbor sets, so colorings equal dsatur_color(build_graph(sets)).
class ImplicitGraph {
 public:
  static bool applicable(const std::vector<ConstraintSet>& sets);
  explicit ImplicitGraph(const std::vector<ConstraintSet>& sets);
  int num_vertices() const { return n_; }
  std::size_t num_edges() const { return edges2_ / 2; }
  int degree(int v) const { return deg_[size_t(v)]; }
  /// f(w) once per neighbor w of v; stamp (size n, caller-owned) tags
  /// visited vertices with `tag`, which must differ between calls.
  // the two neighbor sources of v (DSatur's threaded sweep walks them directly)
  int payload_box(int v) const { return payload_[size_t(v)]; }
  const std::vector<int>& zero_of(int v) const { return (*sets_)[size_t(v)].zero; }
  const int* zero_sets_begin(int box) const { return zsets_.data() + zoff_[size_t(box)]; }
  const int* zero_sets_end(int box) const { return zsets_.data() + zoff_[size_t(box) + 1]; }
  const int* payload_sets_begin(int box) const { return psets_.data() + poff_[size_t(box)]; }
  const int* payload_sets_end(int box) const { return psets_.data() + poff_[size_t(box) + 1]; }
  int num_boxes() const { return int(zoff_.size()) - 1; }
  template <class F>
  void for_each_neighbor(int v, std::vector<int>& stamp, int tag, F&& f) const {
    stamp[size_t(v)] = tag;
    const int pb = payload_[size_t(v)];
    for (int k = zoff_[size_t(pb)]; k < zoff_[size_t(pb) + 1]; ++k) {
      const int w = zsets_[size_t(k)];
      if (stamp[size_t(w)] != tag) {
        stamp[size_t(w)] = tag;
        f(w);
      }
    }
    for (const int z : (*sets_)[size_t(v)].zero)
      for (int k = poff_[size_t(z)]; k < poff_[size_t(z) + 1]; ++k) {
        const int w = psets_[size_t(k)];
        if (stamp[size_t(w)] != tag) {
          stamp[size_t(w)] = tag;
          f(w);
        }
      }
  }

 private:
  const std::vector<ConstraintSet>* sets_;
  int n_ = 0;
  std::vector<int> payload_, zoff_, zsets_, poff_, psets_, deg_;
  std::size_t edges2_ = 0;
};
Coloring dsatur_color(const ImplicitGraph& graph);
/// The same coloring with `threads` sweep threads (1: the serial heap-based
/// implementation; > 1: tournament-tree selection + threaded sweeps).
Coloring dsatur_color(const ImplicitGraph& graph, int threads);

/// proj/src/coloring.cpp:218-250 (DSatur result given).
Coloring plan_coloring(const BoxTree& tree, const std::vector<ConstraintSet>& sets, Coloring dsatur,
                       SampleMode mode);
/// proj/src/coloring.cpp:218-250.
Coloring plan_coloring(const BoxTree& tree, const std::vector<ConstraintSet>& sets,
                       const IncompatibilityGraph& graph, SampleMode mode);

struct BlockTestMatrix {
  Index rows = 0;
  int width = 0;
  std::uint64_t seed = 0;
  int level = 0;
  int phase = 0;
  std::vector<std::pair<int, PayloadTag>> payload;
  std::vector<int> zero;
  std::vector<int> serves;
  /// Dense N x width realization (proj/src/coloring.cpp:261-291), host
  /// reference used by tests; the device path never forms dense Omega.
  Matrix realize(const BoxTree& tree) const;
};

Matrix payload_gaussian(const BoxTree& tree, int box, int width, std::uint64_t seed, int level,
                        int phase);

/// proj/src/coloring.cpp:293-332 (Gaussian and identity payloads).
std::vector<BlockTestMatrix> assemble_test_matrices(const std::vector<ConstraintSet>& sets,
                                                    const Coloring& coloring, const BoxTree& tree,
                                                    int level, int width, std::uint64_t seed,
                                                    int phase);

/// proj/src/coloring.cpp:334-407: the shifted grid patterns (6^d for H1
/// pairs, 5^d for the uniform stage-1 clusters, 3^d for the leaf probes) of a
/// fully populated uniform tree; matrix pattern_index(box, mod) carries the
/// payload of `box`. No graph is built and nothing is colored.
std::vector<BlockTestMatrix> fallback_pattern_matrices(const BoxTree& tree, const AdjacencyInfo& adj,
                                                       int level, SampleMode mode, int width,
                                                       std::uint64_t seed, int phase);
/// proj/src/peeling.cpp:88-96.
int pattern_index(const Box& box, int mod);

/// Output of make_plan (proj/src/peeling.cpp:98-154).
struct SamplingPlan {
  std::vector<BlockTestMatrix> matrices;
  std::map<std::pair<int, int>, int> block_to_matrix;
  std::size_t n_vertices = 0;
  std::size_t n_edges = 0;
  int colors() const { return int(matrices.size()); }
};
/// `pattern`: ColoringStrategy::kFallbackPattern (every mode but the basis probes).
SamplingPlan make_plan(const BoxTree& tree, const AdjacencyInfo& adj, int level, SampleMode mode,
                       int width, std::uint64_t seed, int phase, bool pattern = false);

}  // namespace hpeel
