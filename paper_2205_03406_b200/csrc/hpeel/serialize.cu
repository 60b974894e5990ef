// .hrep representation files in the reference's on-disk format
// (proj/src/serialize.cpp:14-254): little-endian, magic "HPEELRP1", meta,
// the box tree, then per level 0..depth the sorted (alpha, beta) blocks
// U (|I_a| x ku), B (ku x kv), V (|I_b| x kv) with rows in box.points order,
// then the sorted dense blocks D (|I_lam| x |I_mu|). Matrices are
// (rows i64, cols i64, column-major doubles). Only the H1 format is on the
// device path (other format tags are rejected on load).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <fstream>
#include <numeric>
#include <stdexcept>
#include <type_traits>

#include "engine.cuh"
#include "peeling.hpp"
#include "serialize.hpp"

namespace hpeel {

using detail::DeviceGuard;

namespace {

constexpr std::uint64_t kRepMagic = 0x3150524C45455048ull;    // "HPEELRP1"
constexpr std::uint64_t kDenseMagic = 0x314D444C45455048ull;  // "HPEELDM1"
constexpr std::uint8_t kFormatH1 = 1;                         // RepFormat::kH1

// Little-endian byte image of a file, built in memory and written at once.
class ByteSink {
 public:
  template <typename T>
  ByteSink& operator<<(T v) {
    static_assert(std::is_trivially_copyable<T>::value, "plain values only");
    const char* p = reinterpret_cast<const char*>(&v);
    bytes_.insert(bytes_.end(), p, p + sizeof(T));
    return *this;
  }
  void raw(const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    bytes_.insert(bytes_.end(), c, c + n);
  }
  // int32 count, then the values
  void list(const std::vector<int>& v) {
    *this << std::int32_t(v.size());
    for (int x : v) *this << std::int32_t(x);
  }
  // (rows i64, cols i64, column-major doubles)
  void matrix(std::int64_t rows, std::int64_t cols, const double* data) {
    *this << rows << cols;
    raw(data, sizeof(double) * size_t(rows * cols));
  }
  void save(const std::string& path) const {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot write " + path);
    out.write(bytes_.data(), std::streamsize(bytes_.size()));
    if (!out) throw std::runtime_error("write failed: " + path);
  }

 private:
  std::vector<char> bytes_;
};

// Bounds-checked cursor over a whole file read into memory.
class ByteSource {
 public:
  explicit ByteSource(const std::string& path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw std::runtime_error("cannot read " + path);
    bytes_.resize(size_t(in.tellg()));
    in.seekg(0);
    in.read(bytes_.data(), std::streamsize(bytes_.size()));
  }
  template <typename T>
  T take() {
    T v;
    std::memcpy(&v, next(sizeof(T)), sizeof(T));
    return v;
  }
  std::vector<int> list() {
    const auto n = take<std::int32_t>();
    if (n < 0) throw std::runtime_error("corrupt representation file");
    std::vector<int> v(static_cast<size_t>(n));
    for (auto& x : v) x = take<std::int32_t>();
    return v;
  }
  Matrix matrix() {
    const auto rows = take<std::int64_t>();
    const auto cols = take<std::int64_t>();
    if (rows < 0 || cols < 0 || (cols > 0 && rows > std::int64_t(remaining() / 8) / cols))
      throw std::runtime_error("corrupt representation file");
    Matrix m(rows, cols);
    std::memcpy(m.data(), next(sizeof(double) * size_t(rows * cols)), sizeof(double) * size_t(rows * cols));
    return m;
  }

 private:
  size_t remaining() const { return bytes_.size() - pos_; }
  const char* next(size_t n) {
    if (n > remaining()) throw std::runtime_error("truncated representation file");
    const char* p = bytes_.data() + pos_;
    pos_ += n;
    return p;
  }
  std::vector<char> bytes_;
  size_t pos_ = 0;
};

// tree section: dim, leaf capacity, n, box count, then per box level,
// parent, coordinates, children, points (the reference's field order)
void encode_tree(ByteSink& out, const BoxTree& tree) {
  out << std::int32_t(tree.dim()) << std::int32_t(tree.leaf_capacity()) << std::int64_t(tree.num_points())
      << std::int32_t(tree.num_boxes());
  for (const Box& b : tree.boxes()) {
    out << std::int32_t(b.level) << std::int32_t(b.parent);
    for (std::int64_t c : b.coord) out << c;
    out.list(b.children);
    out.list(b.points);
  }
}

std::shared_ptr<const BoxTree> decode_tree(ByteSource& in) {
  const int dim = in.take<std::int32_t>();
  const int leaf = in.take<std::int32_t>();
  const auto n = in.take<std::int64_t>();
  const int count = in.take<std::int32_t>();
  if (dim < 1 || n < 0 || count < 0) throw std::runtime_error("corrupt representation file");
  std::vector<Box> boxes(static_cast<size_t>(count));
  int id = 0;
  for (Box& b : boxes) {
    b.id = id++;
    b.level = in.take<std::int32_t>();
    b.parent = in.take<std::int32_t>();
    b.coord.resize(size_t(dim));
    for (auto& c : b.coord) c = in.take<std::int64_t>();
    b.children = in.list();
    b.points = in.list();
  }
  return std::make_shared<const BoxTree>(BoxTree::from_parts(dim, leaf, n, std::move(boxes)));
}

std::vector<size_t> sorted_order(const std::vector<std::pair<int, int>>& pairs) {
  std::vector<size_t> idx(pairs.size());
  std::iota(idx.begin(), idx.end(), size_t(0));
  std::sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return pairs[x] < pairs[y]; });
  return idx;
}

}  // namespace

void save_rep(const std::string& path, const H1Rep& rep) {
  if (rep.sharded()) throw std::invalid_argument("save_rep: this rank holds a shard of the representation");
  const BoxTree& tree = *rep.tree;
  const TreeLayout& lay = *rep.layout;
  const int k = rep.rank;
  std::vector<double> hf(size_t(std::max<std::int64_t>(rep.factor_doubles, 1)));
  std::vector<double> hd(size_t(std::max<std::int64_t>(rep.dense_doubles, 1)));
  {
    DeviceGuard g(rep.device);
    if (rep.factor_doubles > 0)
      HP_CUDA(cudaMemcpy(hf.data(), rep.d_factors, size_t(rep.factor_doubles) * 8, cudaMemcpyDeviceToHost));
    if (rep.dense_doubles > 0 && rep.d_dense)
      HP_CUDA(cudaMemcpy(hd.data(), rep.d_dense, size_t(rep.dense_doubles) * 8, cudaMemcpyDeviceToHost));
  }
  ByteSink w;
  // magic, then the meta block (proj/src/serialize.cpp:128-138)
  w << kRepMagic << kFormatH1 << std::int64_t(tree.num_points()) << std::int32_t(tree.dim())
    << std::int32_t(tree.depth()) << std::int32_t(tree.leaf_capacity()) << std::int32_t(k)
    << std::int32_t(rep.built_level) << std::uint8_t(rep.dense_ready ? 1 : 0);
  encode_tree(w, tree);
  std::vector<double> buf;
  for (int l = 0; l <= tree.depth(); ++l) {
    const H1Rep::LevelData* ld = size_t(l) < rep.levels.size() ? &rep.levels[size_t(l)] : nullptr;
    const size_t np = ld ? ld->pairs.size() : 0;
    w << std::int32_t(np);
    if (!np) continue;
    for (size_t p : sorted_order(ld->pairs)) {
      const auto [a, b] = ld->pairs[p];
      w << std::int32_t(a) << std::int32_t(b);
      const int ma = int(lay.count[size_t(a)]), mb = int(lay.count[size_t(b)]);
      const int ku = ld->ku[p], kv = ld->kv[p];
      // U rows back to box.points order (arena: tree order, ld = |I_a|)
      auto put_rows = [&](int box, int m, int kk, std::int64_t off) {
        buf.assign(size_t(m) * size_t(kk), 0.0);
        const auto& pts = tree.box(box).points;
        for (int s = 0; s < m; ++s) {
          const std::int64_t tr = lay.inv[size_t(pts[size_t(s)])] - lay.start[size_t(box)];
          for (int j = 0; j < kk; ++j) buf[size_t(s) + size_t(j) * size_t(m)] = hf[size_t(off + tr + std::int64_t(j) * m)];
        }
        w.matrix(m, kk, buf.data());
      };
      put_rows(a, ma, ku, ld->uoff[p]);
      buf.assign(size_t(ku) * size_t(kv), 0.0);
      for (int i = 0; i < ku; ++i)
        for (int j = 0; j < kv; ++j) buf[size_t(i) + size_t(j) * size_t(ku)] = hf[size_t(ld->boff[p] + i + std::int64_t(j) * k)];
      w.matrix(ku, kv, buf.data());
      put_rows(b, mb, kv, ld->voff[p]);
    }
  }
  // dense blocks (leaf rows are in box.points order in the arena)
  const size_t nd = rep.dense_ready ? rep.dense.pairs.size() : 0;
  w << std::int32_t(nd);
  if (nd) {
    for (size_t p : sorted_order(rep.dense.pairs)) {
      const auto [lam, mu] = rep.dense.pairs[p];
      w << std::int32_t(lam) << std::int32_t(mu);
      const std::int64_t ml = std::int64_t(tree.box(lam).points.size()), mm = std::int64_t(tree.box(mu).points.size());
      w.matrix(ml, mm, hd.data() + rep.dense.off[p]);
    }
  }
  w.save(path);
}

std::shared_ptr<H1Rep> load_rep(const std::string& path, int device) {
  ByteSource r(path);
  if (r.take<std::uint64_t>() != kRepMagic) throw std::runtime_error("not a representation file: " + path);
  const std::uint8_t format = r.take<std::uint8_t>();
  const auto n = r.take<std::int64_t>();
  const int dim = r.take<std::int32_t>();
  const int depth = r.take<std::int32_t>();
  (void)r.take<std::int32_t>();  // leaf capacity (also in the tree)
  const int rank = r.take<std::int32_t>();
  const int built_level = r.take<std::int32_t>();
  const bool dense_ready = r.take<std::uint8_t>() != 0;
  if (format != kFormatH1)
    throw std::invalid_argument("only the h1 representation format is on the device path");
  auto tree = decode_tree(r);
  if (tree->num_points() != n || tree->dim() != dim || tree->depth() != depth)
    throw std::runtime_error("representation meta and tree disagree");
  auto rep = std::make_shared<H1Rep>();
  rep->tree = tree;
  rep->adj = std::make_shared<const AdjacencyInfo>(adjacency(*tree));
  rep->layout = std::make_shared<const TreeLayout>(tree_layout(*tree));
  rep->rank = std::max(rank, 1);
  rep->device = device;
  rep->built_level = built_level;
  rep->dense_ready = dense_ready;
  rep->levels.resize(size_t(depth) + 1);
  const TreeLayout& lay = *rep->layout;
  const int k = rep->rank;
  std::vector<double> hf;
  for (int l = 0; l <= depth; ++l) {
    const auto count = r.take<std::int32_t>();
    if (count < 0) throw std::runtime_error("corrupt representation file");
    auto& ld = rep->levels[size_t(l)];
    for (std::int32_t i = 0; i < count; ++i) {
      const int a = r.take<std::int32_t>();
      const int b = r.take<std::int32_t>();
      if (a < 0 || b < 0 || a >= tree->num_boxes() || b >= tree->num_boxes())
        throw std::runtime_error("corrupt representation file");
      const Matrix u = r.matrix(), bb = r.matrix(), v = r.matrix();
      const int ma = int(lay.count[size_t(a)]), mb = int(lay.count[size_t(b)]);
      if (u.rows() != ma || v.rows() != mb || u.cols() > k || v.cols() > k || bb.rows() != u.cols() ||
          bb.cols() != v.cols())
        throw std::runtime_error("representation block shapes disagree with the tree");
      ld.pairs.emplace_back(a, b);
      ld.ku.push_back(int(u.cols()));
      ld.kv.push_back(int(v.cols()));
      const std::int64_t base = std::int64_t(hf.size());
      ld.uoff.push_back(base);
      ld.voff.push_back(base + std::int64_t(ma) * k);
      ld.boff.push_back(base + std::int64_t(ma + mb) * k);
      hf.resize(size_t(base + std::int64_t(ma + mb) * k + std::int64_t(k) * k), 0.0);
      auto take_rows = [&](const Matrix& m, int box, int rows, std::int64_t off) {
        const auto& pts = tree->box(box).points;
        for (int s = 0; s < rows; ++s) {
          const std::int64_t tr = lay.inv[size_t(pts[size_t(s)])] - lay.start[size_t(box)];
          for (Index j = 0; j < m.cols(); ++j) hf[size_t(off + tr + std::int64_t(j) * rows)] = m(s, j);
        }
      };
      take_rows(u, a, ma, ld.uoff.back());
      take_rows(v, b, mb, ld.voff.back());
      for (Index i = 0; i < bb.rows(); ++i)
        for (Index j = 0; j < bb.cols(); ++j) hf[size_t(ld.boff.back() + i + std::int64_t(j) * k)] = bb(i, j);
    }
  }
  std::vector<double> hd;
  const auto nd = r.take<std::int32_t>();
  if (nd < 0) throw std::runtime_error("corrupt representation file");
  for (std::int32_t i = 0; i < nd; ++i) {
    const int lam = r.take<std::int32_t>();
    const int mu = r.take<std::int32_t>();
    const Matrix d = r.matrix();
    if (lam < 0 || mu < 0 || lam >= tree->num_boxes() || mu >= tree->num_boxes() ||
        d.rows() != Index(tree->box(lam).points.size()) || d.cols() != Index(tree->box(mu).points.size()))
      throw std::runtime_error("dense block shapes disagree with the tree");
    rep->dense.pairs.emplace_back(lam, mu);
    rep->dense.off.push_back(std::int64_t(hd.size()));
    hd.insert(hd.end(), d.data(), d.data() + d.size());
  }
  rep->factor_doubles = std::int64_t(hf.size());
  rep->dense_doubles = std::int64_t(hd.size());
  DeviceGuard g(device);
  HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rep->d_factors), std::max<size_t>(hf.size(), 1) * 8, nullptr));
  HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rep->d_dense), std::max<size_t>(hd.size(), 1) * 8, nullptr));
  if (!hf.empty()) HP_CUDA(cudaMemcpy(rep->d_factors, hf.data(), hf.size() * 8, cudaMemcpyHostToDevice));
  if (!hd.empty()) HP_CUDA(cudaMemcpy(rep->d_dense, hd.data(), hd.size() * 8, cudaMemcpyHostToDevice));
  HP_CUDA(cudaStreamSynchronize(nullptr));
  return rep;
}

void save_dense_matrix(const std::string& path, const Matrix& m) {
  ByteSink w;
  w << kDenseMagic;
  w.matrix(m.rows(), m.cols(), m.data());
  w.save(path);
}

Matrix load_dense_matrix(const std::string& path) {
  ByteSource r(path);
  if (r.take<std::uint64_t>() != kDenseMagic) throw std::runtime_error("not a dense matrix file: " + path);
  return r.matrix();
}

}  // namespace hpeel
