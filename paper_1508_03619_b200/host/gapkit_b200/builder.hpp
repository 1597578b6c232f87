// gapkit_b200 host surface: CSR builder.
//
// Same output as the reference BuildCsr (builder.hpp:54-186) for unweighted
// edge lists -- self-loops dropped, duplicates collapsed, neighbour lists
// sorted, optional symmetrization, materialised in-adjacency when directed --
// but 64-bit safe (the reference throws past 2^32 arcs, builder.hpp:71-73,
// because PackAdj keeps a 32-bit origin index) and parallel in every phase
// (the reference counts and scatters serially, builder.hpp:76-99).  For
// unweighted graphs the origin index only breaks ties between equal
// neighbours, which dedup removes, so bare neighbour ids suffice.
#ifndef GAPKIT_B200_BUILDER_HPP_
#define GAPKIT_B200_BUILDER_HPP_

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <numeric>
#include <vector>

#include "gapkit_b200/generator.hpp"
#include "gapkit_b200/graph.hpp"
#include "gapkit_b200/types.hpp"

namespace gapkit {

namespace detail {

inline void ExclusiveScanInPlace(std::vector<int64_t>& a) {
  int64_t run = 0;
  for (auto& x : a) {
    const int64_t t = x;
    x = run;
    run += t;
  }
}

// Counting-sort scatter of (src -> dst) arcs, then per-list sort + dedup.
inline void BuildAdjacency(int64_t n, const std::vector<Edge>& edges, bool both_dirs, bool reverse_only,
                           std::vector<int64_t>& offsets, std::vector<NodeId>& neighbors) {
  std::vector<int64_t> cnt(n + 1, 0);
  const int64_t m = static_cast<int64_t>(edges.size());
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) {
    const Edge e = edges[i];
    if (e.src == e.dst) continue;
    if (!reverse_only) std::atomic_ref<int64_t>(cnt[e.src]).fetch_add(1, std::memory_order_relaxed);
    if (both_dirs || reverse_only) std::atomic_ref<int64_t>(cnt[e.dst]).fetch_add(1, std::memory_order_relaxed);
  }
  ExclusiveScanInPlace(cnt);  // cnt[v] = start of v's raw list, cnt[n] = raw arcs
  std::vector<int64_t> cursor(cnt.begin(), cnt.end() - 1);
  std::vector<NodeId> raw(cnt[n]);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) {
    const Edge e = edges[i];
    if (e.src == e.dst) continue;
    if (!reverse_only)
      raw[std::atomic_ref<int64_t>(cursor[e.src]).fetch_add(1, std::memory_order_relaxed)] = e.dst;
    if (both_dirs || reverse_only)
      raw[std::atomic_ref<int64_t>(cursor[e.dst]).fetch_add(1, std::memory_order_relaxed)] = e.src;
  }
  std::vector<int64_t> deg(n + 1, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; v++) {
    auto b = raw.begin() + cnt[v], e = raw.begin() + cnt[v + 1];
    std::sort(b, e);
    deg[v] = std::unique(b, e) - b;
  }
  offsets.assign(n + 1, 0);
  for (int64_t v = 0; v < n; v++) offsets[v + 1] = offsets[v] + deg[v];
  neighbors.resize(offsets[n]);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; v++)
    std::copy(raw.begin() + cnt[v], raw.begin() + cnt[v] + deg[v], neighbors.begin() + offsets[v]);
}

}  // namespace detail

inline CsrGraph BuildCsr(const EdgeList& el, bool directed, bool symmetrize = false) {
  int64_t max_plus_one = 0;
  const int64_t m = static_cast<int64_t>(el.edges.size());
#pragma omp parallel for reduction(max : max_plus_one)
  for (int64_t i = 0; i < m; i++)
    max_plus_one = std::max<int64_t>(max_plus_one, int64_t{std::max(el.edges[i].src, el.edges[i].dst)} + 1);
  const int64_t n = el.node_count.value_or(max_plus_one);
  if (n < max_plus_one) throw BuildError("edge endpoint exceeds declared node count");  // builder.hpp:66-67
  const bool out_directed = directed && !symmetrize;
  std::vector<int64_t> off;
  std::vector<NodeId> nb;
  detail::BuildAdjacency(n, el.edges, symmetrize, false, off, nb);
  if (!out_directed) {
    CsrGraph g(false, n, std::move(off), std::move(nb));
    if (!symmetrize) {
      if (auto msg = g.CheckInvariants()) throw BuildError("undirected build from asymmetric input: " + *msg);
    }
    return g;
  }
  // builder.hpp:139-173: the transpose of the deduplicated out-edges.
  std::vector<Edge> dedup;
  dedup.reserve(nb.size());
  for (int64_t u = 0; u < n; u++)
    for (int64_t j = off[u]; j < off[u + 1]; j++) dedup.push_back({static_cast<NodeId>(u), nb[j]});
  std::vector<int64_t> in_off;
  std::vector<NodeId> in_nb;
  detail::BuildAdjacency(n, dedup, false, true, in_off, in_nb);
  return CsrGraph(true, n, std::move(off), std::move(nb), std::move(in_off), std::move(in_nb));
}

}  // namespace gapkit

#endif  // GAPKIT_B200_BUILDER_HPP_
