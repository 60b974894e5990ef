// Host planning timer: tree, adjacency and every level's sampling plan (the
// work compress() runs in std::async before the device loop).
// Build: g++ -O2 -std=c++17 -I paper_2205_03406_b200/csrc tools/plan_bench.cpp \
//   -L paper_2205_03406_b200 -lhpeel_b200 -Wl,-rpath,$PWD/paper_2205_03406_b200 -o tools/plan_bench
// Run:   tools/plan_bench points.f64 <n> <dim> <leaf> <width>   (HP_PLAN_TIMING=1 for stages)
#include <chrono>
#include <cstdio>
#include <fstream>
#include <vector>

#include "hpeel/box_tree.hpp"
#include "hpeel/coloring.hpp"

using namespace hpeel;
using Clock = std::chrono::steady_clock;

static double ms(Clock::time_point a) {
  return std::chrono::duration<double, std::milli>(Clock::now() - a).count();
}

int main(int argc, char** argv) {
  if (argc < 6) return 2;
  const long n = std::atol(argv[2]);
  const int dim = std::atoi(argv[3]), leaf = std::atoi(argv[4]), width = std::atoi(argv[5]);
  Matrix raw(n, dim);
  std::ifstream f(argv[1], std::ios::binary);
  f.read(reinterpret_cast<char*>(raw.data()), std::streamsize(n * dim * 8));
  auto t = Clock::now();
  const BoxTree tree = BoxTree::build(PointCloud::from_raw(raw), leaf);
  std::printf("tree %.1f ms depth %d boxes %d\n", ms(t), tree.depth(), tree.num_boxes());
  t = Clock::now();
  const AdjacencyInfo adj = adjacency(tree);
  std::printf("adjacency %.1f ms\n", ms(t));
  for (int l = 2; l <= tree.depth(); ++l) {
    t = Clock::now();
    const SamplingPlan p = make_plan(tree, adj, l, SampleMode::kH1, width, 7, 0);
    std::printf("level %d plan %.1f ms colors %d vertices %zu edges %zu\n", l, ms(t), p.colors(),
                size_t(p.n_vertices), size_t(p.n_edges));
  }
  t = Clock::now();
  const SamplingPlan p = make_plan(tree, adj, tree.depth(), SampleMode::kLeaf, tree.max_leaf_size(), 7, 0);
  std::printf("leaf plan %.1f ms colors %d vertices %zu edges %zu\n", ms(t), p.colors(), size_t(p.n_vertices),
              size_t(p.n_edges));
  return 0;
}
