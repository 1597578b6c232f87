// gapkit_b200 host surface: Brandes(g, sources) -> ScoreArray.
//
// Drop-in for the reference's
//     inline ScoreArray Brandes(const CsrGraph& g,
//                               std::span<const NodeId> sources);
//                                   (kernels/betweenness.hpp:84-145)
// with the same validation order and messages (:86-93) and the same max
// normalisation (:136-143).  Both passes run in libgk_bfs.so (gk_brandes).
#ifndef GAPKIT_B200_BETWEENNESS_HPP_
#define GAPKIT_B200_BETWEENNESS_HPP_

#include <algorithm>
#include <chrono>
#include <cmath>
#include <optional>
#include <ostream>
#include <span>
#include <string>
#include <vector>

#include "gk_bfs.h"
#include "gapkit_b200/fresh_vector.hpp"
#include "gapkit_b200/graph.hpp"
#include "gapkit_b200/harness.hpp"
#include "gapkit_b200/types.hpp"

namespace gapkit {

inline ScoreArray Brandes(const CsrGraph& g, std::span<const NodeId> sources, double* device_ms = nullptr) {
  if (sources.empty()) throw ConfigError("betweenness requires at least one source");
  ScoreArray scores = gk_host::FreshVector<Score>(static_cast<size_t>(g.num_nodes()));
  detail::CheckStatus(gk_brandes(g.device(), sources.data(), static_cast<int64_t>(sources.size()),
                                 scores.data(), device_ms),
                      "gk_brandes");
  return scores;
}

// VerifyBetweenness (verify.hpp:216-270 checks the same thing): an
// independent host recount, level-synchronous rather than queue-driven.
// Pass 1 grows the BFS one level at a time, recording each level's vertex
// range in `layer` and adding path counts forward.  Pass 2 walks the levels
// deepest-first and lets every vertex PULL its dependency from its
// successors (out-neighbours exactly one level deeper), so no predecessor
// lists are kept.  Same sources and max normalisation as Brandes; ok iff
// |diff| < tolerance everywhere.  Host-side checker for the CLI's -v (the
// reference CLI verifies the same way), never on the compute path.
inline VerifyReport VerifyBetweenness(const CsrGraph& g, std::span<const NodeId> sources, const ScoreArray& scores,
                                      double tolerance = 1e-4) {
  const int64_t n = g.num_nodes();
  if (static_cast<int64_t>(scores.size()) != n) return {false, "score array has wrong length"};
  std::vector<double> acc(n, 0.0), paths(n), dep(n);
  std::vector<int32_t> level(n);
  std::vector<NodeId> visit;
  std::vector<size_t> layer;  // visit[layer[d] .. layer[d+1]) = level d
  visit.reserve(n);
  for (NodeId s : sources) {
    std::fill(level.begin(), level.end(), -1);
    std::fill(paths.begin(), paths.end(), 0.0);
    std::fill(dep.begin(), dep.end(), 0.0);
    visit.assign(1, s);
    layer.assign({0, 1});
    level[s] = 0;
    paths[s] = 1;
    for (int32_t d = 0; layer[d] < layer[d + 1]; d++) {
      for (size_t i = layer[d]; i < layer[d + 1]; i++) {
        const NodeId u = visit[i];
        for (NodeId v : g.out_neigh(u)) {
          if (level[v] < 0) {
            level[v] = d + 1;
            visit.push_back(v);
          }
          if (level[v] == d + 1) paths[v] += paths[u];
        }
      }
      layer.push_back(visit.size());
    }
    for (size_t d = layer.size() - 2; d-- > 0;) {
      for (size_t i = layer[d]; i < layer[d + 1]; i++) {
        const NodeId u = visit[i];
        double pull = 0;
        for (NodeId v : g.out_neigh(u))
          if (level[v] == level[u] + 1) pull += (1.0 + dep[v]) / paths[v];
        dep[u] = paths[u] * pull;
        if (u != s) acc[u] += dep[u];
      }
    }
  }
  const double top = acc.empty() ? 0.0 : *std::max_element(acc.begin(), acc.end());
  for (int64_t v = 0; v < n; v++) {
    const double want = top > 0 ? acc[v] / top : acc[v];
    if (!(std::fabs(want - static_cast<double>(scores[v])) < tolerance))
      return {false, "score mismatch at vertex " + std::to_string(v) + ": got " + std::to_string(scores[v]) +
                         ", expected " + std::to_string(want)};
  }
  return {};
}

// The reference harness's bc row (benchmark.hpp:51-82, 238-251): `trials`
// trials of `per_trial` sources drawn in order from one picker sequence,
// one timed Brandes per trial (host wall clock incl. the score copy), -v
// verification untimed.
struct BcTrial {
  int trial = 0;
  std::vector<NodeId> sources;
  double seconds = 0;
  double device_ms = 0;
  std::optional<bool> verified;
  uint64_t digest = 0;
};

inline std::vector<BcTrial> RunBetweenness(CsrGraph& g, int trials, int per_trial, uint64_t seed, bool verify,
                                           std::string* failure = nullptr) {
  std::vector<NodeId> all = PickSources(g, static_cast<int64_t>(trials) * per_trial, seed);
  if (verify) g.EnsureHostArrays();
  std::vector<BcTrial> out;
  for (int t = 0; t < trials; t++) {
    BcTrial tr;
    tr.trial = t;
    tr.sources.assign(all.begin() + static_cast<int64_t>(t) * per_trial,
                      all.begin() + static_cast<int64_t>(t + 1) * per_trial);
    const auto t0 = std::chrono::steady_clock::now();
    ScoreArray sc = Brandes(g, tr.sources, &tr.device_ms);
    tr.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    tr.digest = HashBytes(sc.data(), sc.size() * sizeof(Score));
    if (verify) {
      VerifyReport r = VerifyBetweenness(g, tr.sources, sc);
      tr.verified = r.ok;
      if (!r.ok && failure) *failure = r.failure_detail;
    }
    out.push_back(std::move(tr));
  }
  return out;
}

// benchmark.hpp:302-320 layout: one line per trial (sources joined by ';'),
// then a summary line with the mean.
inline void WriteBcCsv(std::ostream& os, const std::string& graph, const std::vector<BcTrial>& trials) {
  char buf[32];
  double sum = 0;
  bool any = false, all_ok = true;
  os << "kernel,graph,trial,source,elapsed_seconds,verified\n";
  for (const BcTrial& t : trials) {
    os << "bc," << graph << ',' << t.trial << ',';
    for (size_t i = 0; i < t.sources.size(); i++) os << (i ? ";" : "") << t.sources[i];
    std::snprintf(buf, sizeof(buf), "%.9f", t.seconds);
    os << ',' << buf << ',';
    if (t.verified.has_value()) {
      os << (*t.verified ? '1' : '0');
      any = true;
      all_ok &= *t.verified;
    }
    os << '\n';
    sum += t.seconds;
  }
  std::snprintf(buf, sizeof(buf), "%.9f", trials.empty() ? 0.0 : sum / trials.size());
  os << "bc," << graph << ",summary,," << buf << ',';
  if (any) os << (all_ok ? '1' : '0');
  os << '\n';
}

}  // namespace gapkit

#endif  // GAPKIT_B200_BETWEENNESS_HPP_
