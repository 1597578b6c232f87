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
#include "gapkit_b200/graph.hpp"
#include "gapkit_b200/harness.hpp"
#include "gapkit_b200/types.hpp"

namespace gapkit {

inline ScoreArray Brandes(const CsrGraph& g, std::span<const NodeId> sources, double* device_ms = nullptr) {
  if (sources.empty()) throw ConfigError("betweenness requires at least one source");
  ScoreArray scores(g.num_nodes());
  detail::CheckStatus(gk_brandes(g.device(), sources.data(), static_cast<int64_t>(sources.size()),
                                 scores.data(), device_ms),
                      "gk_brandes");
  return scores;
}

// VerifyBetweenness (verify.hpp:216-270): serial Brandes with explicit
// predecessor lists, same sources and max normalisation, |diff| < tolerance
// everywhere.  Host-side checker for the CLI's -v (the reference CLI does the
// same), never on the compute path.
inline VerifyReport VerifyBetweenness(const CsrGraph& g, std::span<const NodeId> sources, const ScoreArray& scores,
                                      double tolerance = 1e-4) {
  const int64_t n = g.num_nodes();
  if (static_cast<int64_t>(scores.size()) != n) return {false, "score array has wrong length"};
  std::vector<double> total(n, 0.0);
  for (NodeId source : sources) {
    std::vector<double> sigma(n, 0.0), delta(n, 0.0);
    std::vector<int32_t> depth(n, -1);
    std::vector<std::vector<NodeId>> preds(n);
    std::vector<NodeId> order;
    order.reserve(n);
    sigma[source] = 1;
    depth[source] = 0;
    order.push_back(source);
    for (size_t qi = 0; qi < order.size(); qi++) {
      const NodeId u = order[qi];
      for (NodeId v : g.out_neigh(u)) {
        if (depth[v] == -1) {
          depth[v] = depth[u] + 1;
          order.push_back(v);
        }
        if (depth[v] == depth[u] + 1) {
          sigma[v] += sigma[u];
          preds[v].push_back(u);
        }
      }
    }
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      const NodeId w = *it;
      for (NodeId v : preds[w]) delta[v] += (sigma[v] / sigma[w]) * (1 + delta[w]);
      if (w != source) total[w] += delta[w];
    }
  }
  double mx = 0;
  for (double t : total) mx = std::max(mx, t);
  if (mx > 0)
    for (double& t : total) t /= mx;
  for (int64_t v = 0; v < n; v++)
    if (std::fabs(total[v] - static_cast<double>(scores[v])) >= tolerance)
      return {false, "score mismatch at vertex " + std::to_string(v) + ": got " + std::to_string(scores[v]) +
                         ", expected " + std::to_string(total[v])};
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
