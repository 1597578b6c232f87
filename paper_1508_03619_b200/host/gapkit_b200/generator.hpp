// gapkit_b200 host surface: synthetic graph generators.
//
// Host generators produce the same tuple sequences as the reference
// (rng.hpp:12-57, generator.hpp:56-112): one keyed splitmix64 stream per
// 1024-edge block, so output is independent of the thread count.  Two new
// generators the BASELINE configs need and the reference lacks:
//   * PermuteIds: seeded bijection on [0, 2^scale) (configs 1/3/5);
//   * GenerateGrid: road-like grid with deletions + diagonals (config 4).
// GenerateOnDevice builds the same graphs directly in HBM (gk_graph_generate),
// which is how the scale-27+ configs are produced in practice.
#ifndef GAPKIT_B200_GENERATOR_HPP_
#define GAPKIT_B200_GENERATOR_HPP_

#include <algorithm>
#include <cstdint>
#include <optional>
#include <vector>

#include "gk_bfs.h"
#include "gapkit_b200/graph.hpp"
#include "gapkit_b200/types.hpp"

namespace gapkit {

struct Edge {
  NodeId src;
  NodeId dst;
  bool operator==(const Edge&) const = default;
};

struct EdgeList {  // edge_list.hpp:23-40 (unweighted)
  std::vector<Edge> edges;
  std::optional<int64_t> node_count;
  void Add(NodeId s, NodeId d) { edges.push_back({s, d}); }
  size_t size() const { return edges.size(); }
};

inline uint64_t Mix64(uint64_t x) {  // rng.hpp:12-17
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

class Rng {  // rng.hpp:24-57
 public:
  explicit Rng(uint64_t seed, uint64_t stream = 0) : state_(Mix64(seed) ^ Mix64(~stream)) {}
  uint64_t Next() {
    state_ += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state_;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint32_t NextBounded(uint32_t bound) {
    uint32_t mask = bound - 1;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    for (;;) {
      uint32_t v = static_cast<uint32_t>(Next() >> 32) & mask;
      if (v < bound) return v;
    }
  }
  double NextUnit() { return static_cast<double>(Next() >> 11) * 0x1.0p-53; }

 private:
  uint64_t state_;
};

enum class GenKind { kKronecker, kUniformRandom };

struct GenSpec {  // generator.hpp:27-32
  GenKind kind;
  int scale;
  int avg_degree = 16;
  uint64_t seed = kDefaultSeed;
};

inline constexpr int64_t kGenBlockSize = 1024;
inline constexpr uint64_t kEdgeStream = 0;
inline constexpr uint64_t kPermStream = uint64_t{2} << 56;
inline constexpr uint64_t kGridDelStream = uint64_t{3} << 56;
inline constexpr uint64_t kGridDiagStream = uint64_t{4} << 56;

inline void ValidateGenSpec(const GenSpec& spec, GenKind expected) {  // generator.hpp:45-52
  if (spec.kind != expected) throw ConfigError("generator called with mismatched GenSpec kind");
  if (spec.scale < 0 || spec.scale > 31) throw ConfigError("generator scale must be in [0, 31]");
  if (spec.avg_degree < 1) throw ConfigError("generator avg_degree must be >= 1");
}

inline EdgeList GenerateUniform(const GenSpec& spec) {  // generator.hpp:56-77
  ValidateGenSpec(spec, GenKind::kUniformRandom);
  const int64_t n = int64_t{1} << spec.scale, m = spec.avg_degree * n;
  EdgeList el;
  el.node_count = n;
  el.edges.resize(m);
  const int64_t blocks = (m + kGenBlockSize - 1) / kGenBlockSize;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < blocks; b++) {
    Rng rng(spec.seed, kEdgeStream | static_cast<uint64_t>(b));
    for (int64_t i = b * kGenBlockSize; i < std::min(m, (b + 1) * kGenBlockSize); i++) {
      NodeId s = rng.NextBounded(static_cast<uint32_t>(n));
      NodeId d = rng.NextBounded(static_cast<uint32_t>(n));
      el.edges[i] = {s, d};
    }
  }
  return el;
}

inline EdgeList GenerateKronecker(const GenSpec& spec) {  // generator.hpp:79-112
  ValidateGenSpec(spec, GenKind::kKronecker);
  constexpr double kA = 0.57, kB = 0.19, kC = 0.19;
  const int64_t n = int64_t{1} << spec.scale, m = spec.avg_degree * n;
  EdgeList el;
  el.node_count = n;
  el.edges.resize(m);
  const int64_t blocks = (m + kGenBlockSize - 1) / kGenBlockSize;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < blocks; b++) {
    Rng rng(spec.seed, kEdgeStream | static_cast<uint64_t>(b));
    for (int64_t i = b * kGenBlockSize; i < std::min(m, (b + 1) * kGenBlockSize); i++) {
      NodeId s = 0, d = 0;
      for (int depth = 0; depth < spec.scale; depth++) {
        const double p = rng.NextUnit();
        s <<= 1;
        d <<= 1;
        if (p < kA + kB) {
          if (p > kA) d |= 1;
        } else {
          s |= 1;
          if (p > kA + kB + kC) d |= 1;
        }
      }
      el.edges[i] = {s, d};
    }
  }
  return el;
}

// Seeded vertex-ID permutation on [0, 2^scale): four rounds of
// {odd multiply, add, xorshift} mod 2^scale, each a bijection; keys from
// Rng(seed, kPermStream | scale).  Identical on the device build.
class IdPermutation {
 public:
  IdPermutation(uint64_t seed, int scale) : scale_(scale) {
    Rng r(seed, kPermStream | static_cast<uint64_t>(scale));
    for (auto& k : keys_) k = r.Next();
    for (int i = 0; i < 4; i++) keys_[2 * i] |= 1;
    mask_ = scale >= 64 ? ~0ULL : ((1ULL << scale) - 1);
  }
  NodeId operator()(NodeId v) const {
    if (scale_ <= 0) return v;
    const int sh = (scale_ + 1) / 2;
    uint64_t x = v;
    for (int i = 0; i < 4; i++) {
      x = (x * keys_[2 * i]) & mask_;
      x = (x + keys_[2 * i + 1]) & mask_;
      x ^= x >> sh;
    }
    return static_cast<NodeId>(x);
  }

 private:
  int scale_;
  uint64_t mask_;
  uint64_t keys_[8];
};

inline void PermuteIds(EdgeList& el, int scale, uint64_t seed) {
  const IdPermutation perm(seed, scale);
  const int64_t m = static_cast<int64_t>(el.edges.size());
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) el.edges[i] = {perm(el.edges[i].src), perm(el.edges[i].dst)};
}

// Road-like grid (BASELINE config 4): rows x cols cells, vertex r*cols+c.
// Base 4-neighbour edges (horizontals, then verticals) are each deleted with
// probability p_delete (draw i of the edge's 1024-block stream); every cell
// with a row below draws NextUnit() < p_diag for one diagonal shortcut to
// (r+1, c+-1) (second draw's top bit picks the side; reflected at borders).
inline EdgeList GenerateGrid(int64_t rows, int64_t cols, double p_delete, double p_diag,
                             uint64_t seed = kDefaultSeed) {
  if (rows < 1 || cols < 1) throw ConfigError("grid dimensions must be positive");
  const int64_t H = rows * (cols - 1), V = (rows - 1) * cols, B = H + V;
  EdgeList el;
  el.node_count = rows * cols;
  for (int64_t b = 0; b * kGenBlockSize < B; b++) {
    Rng r(seed, kGridDelStream | static_cast<uint64_t>(b));
    for (int64_t i = b * kGenBlockSize; i < std::min(B, (b + 1) * kGenBlockSize); i++) {
      if (r.NextUnit() < p_delete) continue;
      if (i < H) {
        const int64_t a = (i / (cols - 1)) * cols + i % (cols - 1);
        el.Add(static_cast<NodeId>(a), static_cast<NodeId>(a + 1));
      } else {
        el.Add(static_cast<NodeId>(i - H), static_cast<NodeId>(i - H + cols));
      }
    }
  }
  if (cols > 1) {
    for (int64_t b = 0; b * kGenBlockSize < V; b++) {
      Rng r(seed, kGridDiagStream | static_cast<uint64_t>(b));
      for (int64_t j = b * kGenBlockSize; j < std::min(V, (b + 1) * kGenBlockSize); j++) {
        if (!(r.NextUnit() < p_diag)) continue;
        int64_t d = (r.Next() >> 63) ? 1 : -1;
        const int64_t c = j % cols;
        if (c + d < 0 || c + d >= cols) d = -d;
        el.Add(static_cast<NodeId>(j), static_cast<NodeId>(j + cols + d));
      }
    }
  }
  return el;
}

// Generate + build in HBM (gk_graph_generate / gk_graph_generate_grid).
inline CsrGraph GenerateOnDevice(const GenSpec& spec, bool permute, int device = 0) {
  ValidateGenSpec(spec, spec.kind);
  gk_graph* h = nullptr;
  detail::CheckStatus(gk_graph_generate(spec.kind == GenKind::kKronecker ? 0 : 1, spec.scale, spec.avg_degree,
                                        spec.seed, permute ? 1 : 0, device, &h),
                      "gk_graph_generate");
  return CsrGraph::FromDevice(h);
}

inline CsrGraph GenerateGridOnDevice(int64_t rows, int64_t cols, double p_delete, double p_diag,
                                     uint64_t seed = kDefaultSeed, int device = 0) {
  gk_graph* h = nullptr;
  detail::CheckStatus(gk_graph_generate_grid(rows, cols, p_delete, p_diag, seed, device, &h),
                      "gk_graph_generate_grid");
  return CsrGraph::FromDevice(h);
}

}  // namespace gapkit

#endif  // GAPKIT_B200_GENERATOR_HPP_
