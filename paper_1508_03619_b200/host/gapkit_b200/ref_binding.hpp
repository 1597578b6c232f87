// ref_binding.hpp -- the B200 BFS behind the REFERENCE's own types.
//
// For a gapkit build (proj/include/gapkit, unmodified): include this header
// after "gapkit/gapkit.hpp" and call
//
//     gapkit::ParentArray p = gapkit::b200::Bfs(g, source, opts);
//
// with the reference's gapkit::CsrGraph, NodeId, BfsOptions and ParentArray.
// It is a drop-in for gapkit::Bfs (proj/include/gapkit/kernels/bfs.hpp:117-118):
// same signature and result type, same validation order and ConfigError
// texts (bfs.hpp:120-123), same semantics (parent[src] = src, unreachable
// -1, top-down on out-edges, bottom-up on in-edges of directed graphs,
// alpha/beta/strategy).  Nothing here defines names in namespace gapkit
// itself, so it compiles next to the reference headers.
//
// The graph is read through the reference's public accessors
// (graph.hpp:88-99: out_offsets / out_neighbors / in_offsets / in_neighbors)
// and uploaded to HBM with gk_graph_upload on first use; the device copy is
// cached per graph (its array addresses and sizes plus a sampled content
// fingerprint), as the harness reuses the loaded graph across trials
// (PAPER.md:144).  gapkit::b200::Release(g) drops a graph's device copy.
// Every call allocates its scratch and result inside the call (the C ABI's
// trial), and returns the ParentArray by value like the reference.
//
// Errors: GK_ERR_SOURCE_RANGE / GK_ERR_BAD_PARAM -> gapkit::ConfigError with
// the reference's message; every other failure (no device, out of memory,
// CUDA error) -> gapkit::Error with gk_last_error()'s text.  There is no
// CPU fallback.
//
// Link: -I<repo>/include -I<repo>/paper_1508_03619_b200/host
//       -L<repo>/paper_1508_03619_b200/lib -lgk_bfs
#pragma once

#ifndef GAPKIT_GAPKIT_HPP_
#error "include gapkit/gapkit.hpp (the reference) before gapkit_b200/ref_binding.hpp"
#endif

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "gk_bfs.h"
#include "gapkit_b200/fresh_vector.hpp"

namespace gapkit::b200 {

namespace detail {

// Sampled FNV-1a over up to 2 x 128 entries of each array: catches a graph
// rebuilt at the same addresses with different content (a CsrGraph is
// immutable once built, graph.hpp:25).
template <typename T>
inline uint64_t Fingerprint(const std::vector<T>& a, uint64_t h) {
  const size_t n = a.size();
  const size_t stride = n > 256 ? n / 128 : 1;
  auto mix = [&](uint64_t x) {
    for (int i = 0; i < 8; i++) {
      h ^= (x >> (8 * i)) & 0xff;
      h *= 0x100000001b3ull;
    }
  };
  mix(n);
  for (size_t i = 0; i < n; i += stride) mix(static_cast<uint64_t>(a[i]));
  for (size_t i = n > 128 ? n - 128 : 0; i < n; i++) mix(static_cast<uint64_t>(a[i]));
  return h;
}

using Key = std::tuple<const void*, const void*, int64_t, int64_t, uint64_t>;

inline Key KeyOf(const CsrGraph& g) {
  uint64_t h = 0xcbf29ce484222325ull;
  h = Fingerprint(g.out_offsets(), h);
  h = Fingerprint(g.out_neighbors(), h);
  if (g.directed()) {
    h = Fingerprint(g.in_offsets(), h);
    h = Fingerprint(g.in_neighbors(), h);
  }
  return {g.out_offsets().data(), g.out_neighbors().data(), g.num_nodes(), g.num_edges(), h};
}

struct Handle {
  gk_graph* g = nullptr;
  ~Handle() {
    if (g) gk_graph_free(g);
  }
};

struct Cache {
  std::mutex mu;
  std::map<Key, std::shared_ptr<Handle>> graphs;
};

inline Cache& TheCache() {
  static Cache c;
  return c;
}

[[noreturn]] inline void Throw(gk_status st) {
  const std::string msg = gk_last_error();
  if (st == GK_ERR_SOURCE_RANGE || st == GK_ERR_BAD_PARAM) throw ConfigError(msg);
  throw Error("b200 bfs: " + msg);
}

inline std::shared_ptr<Handle> DeviceGraph(const CsrGraph& g) {
  const Key k = KeyOf(g);
  Cache& c = TheCache();
  std::lock_guard<std::mutex> lock(c.mu);
  auto it = c.graphs.find(k);
  if (it != c.graphs.end()) return it->second;
  gk_csr_view v{};
  v.num_nodes = g.num_nodes();
  v.directed = g.directed() ? 1 : 0;
  v.out_offsets = g.out_offsets().data();
  v.out_neighbors = g.out_neighbors().data();
  if (g.directed()) {  // graph.hpp:64-67: undirected in_* alias the out arrays
    v.in_offsets = g.in_offsets().data();
    v.in_neighbors = g.in_neighbors().data();
  }
  auto h = std::make_shared<Handle>();
  const gk_status st = gk_graph_upload(&v, 0, &h->g);
  if (st != GK_OK) Throw(st);
  c.graphs.emplace(k, h);
  return h;
}

}  // namespace detail

// Drop-in for gapkit::Bfs (bfs.hpp:117-177).
inline ParentArray Bfs(const CsrGraph& g, NodeId source, const BfsOptions& opts = {}) {
  // bfs.hpp:120-123: same checks, same order, same messages
  if (static_cast<int64_t>(source) >= g.num_nodes()) throw ConfigError("bfs source out of range");
  if (opts.alpha <= 0 || opts.beta <= 0) throw ConfigError("bfs alpha and beta must be positive");
  std::shared_ptr<detail::Handle> h = detail::DeviceGraph(g);
  ParentArray parent = gk_host::FreshVector<ParentEntry>(static_cast<size_t>(g.num_nodes()));
  const gk_status st = gk_bfs(h->g, source, opts.alpha, opts.beta, static_cast<int32_t>(opts.strategy),
                              parent.data(), nullptr, nullptr);
  if (st != GK_OK) detail::Throw(st);
  return parent;
}

// Drop-in for gapkit::Brandes (kernels/betweenness.hpp:84-145).
inline ScoreArray Brandes(const CsrGraph& g, std::span<const NodeId> sources) {
  std::shared_ptr<detail::Handle> h = detail::DeviceGraph(g);
  ScoreArray scores = gk_host::FreshVector<Score>(static_cast<size_t>(g.num_nodes()));
  const gk_status st = gk_brandes(h->g, sources.data(), static_cast<int64_t>(sources.size()), scores.data(),
                                  nullptr);
  if (st != GK_OK) detail::Throw(st);
  return scores;
}

// Frees the device copy of g (if any); the next call uploads it again.
inline void Release(const CsrGraph& g) {
  detail::Cache& c = detail::TheCache();
  std::lock_guard<std::mutex> lock(c.mu);
  c.graphs.erase(detail::KeyOf(g));
}

}  // namespace gapkit::b200
