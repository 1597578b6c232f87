// gapkit_b200 host surface: source selection, verification and the BFS
// benchmark harness.
//
//   SourcePicker / PickSources   source_picker.hpp:22-54
//   BfsDepths / VerifyBfs        verify.hpp:42-98 (host-side checker of the
//                                device output, run untimed like the
//                                reference's, benchmark.hpp:188-192)
//   BenchPlan / RunBenchmark     benchmark.hpp:51-273, BFS kernel only
//   WriteCsv / summary           benchmark.hpp:278-340, plus a GTEPS column
#ifndef GAPKIT_B200_HARNESS_HPP_
#define GAPKIT_B200_HARNESS_HPP_

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <optional>
#include <ostream>
#include <string>
#include <vector>

#include "gapkit_b200/bfs.hpp"
#include "gapkit_b200/generator.hpp"
#include "gapkit_b200/graph.hpp"
#include "gapkit_b200/types.hpp"

namespace gapkit {

class SourcePicker {  // source_picker.hpp:22-45 (host-resident graphs)
 public:
  explicit SourcePicker(const CsrGraph& g, uint64_t seed = kDefaultSeed,
                        std::optional<NodeId> fixed_source = std::nullopt)
      : graph_(g), rng_(seed), fixed_(fixed_source) {
    if (g.num_edges() == 0) throw ConfigError("cannot pick sources: graph has no edges");
    if (!g.host_ready()) throw ConfigError("SourcePicker needs host arrays; use PickSources");
  }
  NodeId PickNext() {
    if (fixed_) return *fixed_;
    NodeId c;
    do {
      c = rng_.NextBounded(static_cast<uint32_t>(graph_.num_nodes()));
    } while (graph_.out_degree(c) == 0);
    return c;
  }

 private:
  const CsrGraph& graph_;
  Rng rng_;
  std::optional<NodeId> fixed_;
};

inline std::vector<NodeId> PickSources(const CsrGraph& g, int64_t count, uint64_t seed = kDefaultSeed) {
  if (!g.host_ready()) {  // device-resident: the device-side picker uses the identical stream
    std::vector<NodeId> out(count);
    detail::CheckStatus(gk_pick_sources(g.device(), count, seed, out.data()), "gk_pick_sources");
    return out;
  }
  SourcePicker picker(g, seed);
  std::vector<NodeId> s(count);
  for (int64_t i = 0; i < count; i++) s[i] = picker.PickNext();
  return s;
}

struct VerifyReport {  // verify.hpp:31-34
  bool ok = true;
  std::string failure_detail;
};

inline std::vector<int32_t> BfsDepths(const CsrGraph& g, NodeId source) {  // verify.hpp:42-58
  std::vector<int32_t> depth(g.num_nodes(), -1);
  std::vector<NodeId> q;
  q.reserve(g.num_nodes());
  depth[source] = 0;
  q.push_back(source);
  for (size_t i = 0; i < q.size(); i++) {
    const NodeId u = q[i];
    for (NodeId v : g.out_neigh(u))
      if (depth[v] == -1) {
        depth[v] = depth[u] + 1;
        q.push_back(v);
      }
  }
  return depth;
}

inline VerifyReport VerifyBfs(const CsrGraph& g, NodeId source, const ParentArray& tree) {  // verify.hpp:62-98
  const int64_t n = g.num_nodes();
  if (static_cast<int64_t>(tree.size()) != n) return {false, "parent array has wrong length"};
  if (tree[source] != static_cast<ParentEntry>(source))
    return {false, "parent[source] != source at vertex " + std::to_string(source)};
  const std::vector<int32_t> depth = BfsDepths(g, source);
  for (int64_t v = 0; v < n; v++) {
    if (depth[v] == -1) {
      if (tree[v] != -1)
        return {false, "unreachable vertex " + std::to_string(v) + " has parent " + std::to_string(tree[v])};
      continue;
    }
    if (v == static_cast<int64_t>(source)) continue;
    const ParentEntry p = tree[v];
    if (p < 0) return {false, "reachable vertex " + std::to_string(v) + " marked unreached"};
    if (p >= n) return {false, "parent id out of range at vertex " + std::to_string(v)};
    if (!g.HasOutEdge(static_cast<NodeId>(p), static_cast<NodeId>(v)))
      return {false, "no edge (" + std::to_string(p) + "," + std::to_string(v) + ") for claimed parent"};
    if (depth[p] != depth[v] - 1)
      return {false, "parent of vertex " + std::to_string(v) + " has depth " + std::to_string(depth[p]) +
                         ", expected " + std::to_string(depth[v] - 1)};
  }
  return {};
}

struct BenchPlan {  // benchmark.hpp:51-82 (BFS row of Table 1: 64 trials x 1 source)
  int trials = 64;
  int64_t alpha = 15;
  int64_t beta = 18;
  uint64_t source_seed = kDefaultSeed;
  std::optional<NodeId> fixed_source;
  // Measurement columns beyond the reference's report:
  // the B_sec byte model of each trial (an untimed second traversal that
  // records depths) and its HBM-roofline fraction against peak_gbs.
  bool model = true;
  double peak_gbs = 6550.7;  // MEASURED_PEAKS.json hbm_gbs of this pool's B200s
  int gpus = 1;              // devices the traversal ran on
};

struct TrialResult {  // benchmark.hpp:84-90
  int trial = 0;
  NodeId source = 0;
  double seconds = 0;      // host wall clock around Bfs, parent array returned
  double device_ms = 0;    // CUDA-event time of the trial (gk_bfs_stats.device_ms)
  int64_t component_edges = 0;  // m_cc: undirected edges in the source's component
  double bytes_model = 0;       // B_sec algorithmic bytes, 0 without plan.model
  std::string schedule;
  std::optional<bool> verified;
  uint64_t digest = 0;
};

struct BenchReport {
  std::string graph_name;
  std::vector<TrialResult> trials;
  bool AllVerified() const {
    for (const auto& t : trials)
      if (t.verified.has_value() && !*t.verified) return false;
    return true;
  }
  double HmeanDeviceGteps() const {
    double inv = 0;
    int k = 0;
    for (const auto& t : trials)
      if (t.device_ms > 0 && t.component_edges > 0) {
        inv += (t.device_ms * 1e-3) / (static_cast<double>(t.component_edges) / 1e9);
        k++;
      }
    return inv > 0 ? k / inv : 0.0;
  }
};

inline uint64_t HashBytes(const void* data, size_t len) {  // benchmark.hpp:127-135
  const auto* p = static_cast<const unsigned char*>(data);
  uint64_t h = 14695981039346656037ULL;
  for (size_t i = 0; i < len; i++) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

// benchmark.hpp:153-193 for the BFS kernel: one picker sequence across the
// trials; each trial times exactly one Bfs call; verification is untimed.
inline BenchReport RunBenchmark(CsrGraph& g, const BenchPlan& plan, bool verify,
                                const std::string& graph_name = "graph") {
  if (plan.trials < 0) throw ConfigError("negative trial count");
  std::vector<NodeId> sources;
  if (plan.fixed_source) sources.assign(plan.trials, *plan.fixed_source);
  else sources = PickSources(g, plan.trials, plan.source_seed);
  if (verify) g.EnsureHostArrays();
  BenchReport report;
  report.graph_name = graph_name;
  for (int t = 0; t < plan.trials; t++) {
    TrialResult tr;
    tr.trial = t;
    tr.source = sources[t];
    BfsTelemetry tel;
    const auto t0 = std::chrono::steady_clock::now();
    ParentArray parent = Bfs(g, tr.source, {.alpha = plan.alpha, .beta = plan.beta}, &tel);
    const auto t1 = std::chrono::steady_clock::now();
    tr.seconds = std::chrono::duration<double>(t1 - t0).count();
    tr.device_ms = tel.device_ms;
    tr.component_edges = tel.component_edges;
    tr.schedule = tel.schedule;
    tr.digest = HashBytes(parent.data(), parent.size() * sizeof(ParentEntry));
    if (plan.model) {  // untimed: the same traversal again, recording depths, then the byte model
      gk_graph* dev = g.device();
      detail::CheckStatus(gk_bfs_keep_depth(dev, 1), "gk_bfs_keep_depth");
      detail::CheckStatus(gk_bfs(dev, tr.source, plan.alpha, plan.beta, 0, nullptr, nullptr, nullptr), "gk_bfs");
      double bs = 0, bu = 0;
      detail::CheckStatus(gk_bfs_byte_model(dev, tel.steps.data(), static_cast<int32_t>(tel.steps.size()), &bs, &bu),
                          "gk_bfs_byte_model");
      detail::CheckStatus(gk_bfs_keep_depth(dev, 0), "gk_bfs_keep_depth");
      tr.bytes_model = bs;
    }
    if (verify) {
      VerifyReport r = VerifyBfs(g, tr.source, parent);
      tr.verified = r.ok;
      if (!r.ok) std::fprintf(stderr, "bfs trial %d from %u failed verification: %s\n", t, tr.source,
                              r.failure_detail.c_str());
    }
    report.trials.push_back(tr);
  }
  return report;
}

// benchmark.hpp:302-320 plus the device columns: device_ms, m_cc, GTEPS,
// the B_sec byte model (bytes_model), roofline_frac = bytes_model /
// device time / peak, gpus, and the executed direction schedule.
inline void WriteCsv(std::ostream& out, const BenchReport& r, const BenchPlan& plan = {}) {
  out << "kernel,graph,trial,source,elapsed_seconds,verified,device_ms,m_cc,gteps,bytes_model,roofline_frac,gpus,"
         "schedule\n";
  for (const auto& t : r.trials) {
    const double sec = t.device_ms * 1e-3;
    const double gteps = sec > 0 ? t.component_edges / sec / 1e9 : 0.0;
    const double frac = sec > 0 && t.bytes_model > 0 ? t.bytes_model / sec / 1e9 / plan.peak_gbs : 0.0;
    out << "bfs," << r.graph_name << "," << t.trial << "," << t.source << "," << t.seconds << ","
        << (t.verified.has_value() ? (*t.verified ? "1" : "0") : "") << "," << t.device_ms << ","
        << t.component_edges << "," << gteps << "," << t.bytes_model << "," << frac << "," << plan.gpus << ","
        << (t.schedule.size() <= 64 ? t.schedule : t.schedule.substr(0, 61) + "...") << "\n";
  }
}

}  // namespace gapkit

#endif  // GAPKIT_B200_HARNESS_HPP_
