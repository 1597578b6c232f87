// ref_graph.hpp -- the handle behind every gkr_* entry point of
// oracle/_ref/libgapref.so (ref_shim.cc, ref_bench.cc).  TEST / BASELINE
// INFRASTRUCTURE ONLY (see gk_oracle.h).
#pragma once

#include <cstdint>
#include <vector>

#include "gapkit/gapkit.hpp"

namespace gkref {

struct RefGraph {
  bool directed = false;
  int64_t n = 0;
  std::vector<int64_t> off;  // filled by the caller before gkr_graph_seal
  std::vector<gapkit::NodeId> nb;
  std::vector<int64_t> in_off;
  std::vector<gapkit::NodeId> in_nb;
  gapkit::CsrGraph g;
  bool sealed = false;
};

}  // namespace gkref
