// Point cloud, dyadic box tree, adjacency and admissible/dense pair lists.
//
// Host-side restatement of proj/include/hpeel/box_tree.hpp:13-116 and
// proj/src/box_tree.cpp:39-323. Trees, neighbor/interaction lists, coarse
// leaf neighbors and dense partners are bit-identical to the reference's (same
// BFS ids, same point order inside each box, same sorted lists).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "matrix.hpp"

namespace hpeel {

/// N points in d dimensions rescaled per dimension into [0,1]^d
/// (proj/src/box_tree.cpp:55-70). coords(i, j) = coordinate j of point i.
struct PointCloud {
  Matrix coords;
  int dim() const { return int(coords.cols()); }
  Index size() const { return coords.rows(); }
  static PointCloud from_raw(const Matrix& raw);
  static PointCloud from_file(const std::string& path);
};

struct Box {
  int id = -1;
  int level = 0;
  std::vector<std::int64_t> coord;
  int parent = -1;
  std::vector<int> children;          // ascending ids
  std::vector<int> points;            // input order
  std::vector<std::vector<int>> child_rows;
  bool is_leaf() const { return children.empty(); }
};

class BoxTree {
 public:
  static constexpr int kMaxDepth = 62;

  /// proj/src/box_tree.cpp:99-180. Throws std::runtime_error on degenerate
  /// geometry, std::invalid_argument on bad arguments.
  static BoxTree build(const PointCloud& cloud, int leaf_capacity);
  /// proj/src/box_tree.cpp:182-196: rebuild from serialized boxes (level
  /// lists, depth and child rows recomputed).
  static BoxTree from_parts(int dim, int leaf_capacity, Index n, std::vector<Box> boxes);

  int dim() const { return dim_; }
  int depth() const { return depth_; }
  int leaf_capacity() const { return leaf_capacity_; }
  Index num_points() const { return num_points_; }
  const std::vector<Box>& boxes() const { return boxes_; }
  const Box& box(int id) const { return boxes_[size_t(id)]; }
  int num_boxes() const { return int(boxes_.size()); }
  const std::vector<int>& level_boxes(int level) const { return levels_[size_t(level)]; }
  int max_leaf_size() const;
  bool is_fully_populated() const;

 private:
  int dim_ = 0;
  int depth_ = 0;
  int leaf_capacity_ = 0;
  Index num_points_ = 0;
  std::vector<Box> boxes_;
  std::vector<std::vector<int>> levels_;
};

struct AdjacencyInfo {
  std::vector<std::vector<int>> neighbors;
  std::vector<std::vector<int>> interaction;
  std::vector<std::vector<int>> coarse_leaf_neighbors;
  std::vector<std::vector<int>> dense_partners;
  std::size_t cross_level_adjacencies = 0;
};

/// proj/src/box_tree.cpp:214-300.
AdjacencyInfo adjacency(const BoxTree& tree);

/// proj/src/box_tree.cpp:302-313 (level-box order, then interaction order).
std::vector<std::pair<int, int>> admissible_pairs(const BoxTree& tree, const AdjacencyInfo& adj,
                                                  int level);

/// proj/src/box_tree.cpp:315-323.
std::vector<std::pair<int, int>> dense_pairs(const BoxTree& tree, const AdjacencyInfo& adj);

/// Depth-first "tree order": every box is one contiguous range of positions.
/// Inside a leaf the order is the leaf's own (input) point order, so identity
/// payload column t of leaf v is position start[v] + t. Not in the reference:
/// this is the device data layout.
struct TreeLayout {
  std::vector<int> perm;            // tree position -> input point index
  std::vector<int> inv;             // input point index -> tree position
  std::vector<std::int64_t> start;  // per box: first tree position
  std::vector<std::int64_t> count;  // per box: number of points
  /// per box: local row (rank in box.points) of each of its tree positions,
  /// i.e. local[start[b] + s] for s < count[b] is flattened in `local_flat`
  /// at offset local_off[b].
  std::vector<std::int64_t> local_off;
  std::vector<int> local_flat;
};
TreeLayout tree_layout(const BoxTree& tree);

}  // namespace hpeel
