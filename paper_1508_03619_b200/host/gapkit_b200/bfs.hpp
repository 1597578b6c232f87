// gapkit_b200 host surface: Bfs(g, source, opts) -> ParentArray.
//
// Drop-in for the reference's operator API,
//     inline ParentArray Bfs(const CsrGraph& g, NodeId source,
//                            const BfsOptions& opts = {});   (bfs.hpp:117-118)
// with the same options (bfs.hpp:37-43), errors (bfs.hpp:120-123) and output
// convention (parent[source] = source, unreachable = -1, bfs.hpp:171-176).
// The traversal runs in libgk_bfs.so on the B200; the graph is uploaded once
// per CsrGraph and the parent array is returned by value (allocated inside the
// call, as the reference's timed call does, acceptance.cc:223-236).
#ifndef GAPKIT_B200_BFS_HPP_
#define GAPKIT_B200_BFS_HPP_

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "gk_bfs.h"
#include "gapkit_b200/fresh_vector.hpp"
#include "gapkit_b200/graph.hpp"
#include "gapkit_b200/types.hpp"

namespace gapkit {

enum class BfsStrategy { kDirectionOptimizing, kTopDownOnly, kTopDownRescan };  // bfs.hpp:37

struct BfsOptions {  // bfs.hpp:39-43
  int64_t alpha = 15;
  int64_t beta = 18;
  BfsStrategy strategy = BfsStrategy::kDirectionOptimizing;
};

// Per-call telemetry beyond the reference's surface (device time, schedule).
struct BfsTelemetry {
  float device_ms = 0;
  std::string schedule;
  std::vector<gk_step> steps;
  int64_t reached = -1;
  int64_t component_edges = -1;
};

inline ParentArray Bfs(const CsrGraph& g, NodeId source, const BfsOptions& opts = {},
                       BfsTelemetry* telemetry = nullptr) {
  if (static_cast<int64_t>(source) >= g.num_nodes()) throw ConfigError("bfs source out of range");
  if (opts.alpha <= 0 || opts.beta <= 0) throw ConfigError("bfs alpha and beta must be positive");
  gk_graph* dev = g.device();
  ParentArray parent = gk_host::FreshVector<ParentEntry>(static_cast<size_t>(g.num_nodes()));
  gk_bfs_stats st{};
  std::vector<gk_step> steps;
  if (telemetry) {
    steps.resize(4096);
    st.steps = steps.data();
    st.max_steps = static_cast<int32_t>(steps.size());
    st.want_counts = 1;
  }
  detail::CheckStatus(gk_bfs(dev, source, opts.alpha, opts.beta, static_cast<int32_t>(opts.strategy),
                             parent.data(), nullptr, telemetry ? &st : nullptr),
                      "gk_bfs");
  if (telemetry) {
    telemetry->device_ms = st.device_ms;
    steps.resize(std::min<int64_t>(st.num_steps, static_cast<int64_t>(steps.size())));
    telemetry->schedule.clear();
    for (const gk_step& s : steps) telemetry->schedule.push_back(static_cast<char>(s.dir));
    telemetry->steps = std::move(steps);
    telemetry->reached = st.reached;
    telemetry->component_edges = st.component_edges;
  }
  return parent;
}

}  // namespace gapkit

#endif  // GAPKIT_B200_BFS_HPP_
