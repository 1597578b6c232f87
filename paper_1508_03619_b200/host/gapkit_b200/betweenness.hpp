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

#include <span>

#include "gk_bfs.h"
#include "gapkit_b200/graph.hpp"
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

}  // namespace gapkit

#endif  // GAPKIT_B200_BETWEENNESS_HPP_
