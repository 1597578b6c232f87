// gapkit_b200 host surface: serialized-graph cache.
//
// ReadSerialized / WriteSerialized (proj/include/gapkit/io.hpp:364-456) for
// the binary ".sg"/".wsg" layout, streamed file <-> HBM by libgk_bfs.so
// (gk_graph_load_sg / gk_graph_save_sg) without a host copy of the graph.
#ifndef GAPKIT_B200_IO_HPP_
#define GAPKIT_B200_IO_HPP_

#include <string>

#include "gk_bfs.h"
#include "gapkit_b200/graph.hpp"
#include "gapkit_b200/types.hpp"

namespace gapkit {

struct LoadError : Error {  // errors.hpp:35-46
  using Error::Error;
};

inline CsrGraph ReadSerializedOnDevice(const std::string& path, int device = 0) {
  gk_graph* h = nullptr;
  const gk_status st = gk_graph_load_sg(path.c_str(), device, &h);
  if (st == GK_ERR_LOAD) throw LoadError(gk_last_error());
  if (st == GK_ERR_INVALID) throw ConfigError(gk_last_error());
  detail::CheckStatus(st, "gk_graph_load_sg");
  return CsrGraph::FromDevice(h);
}

inline void WriteSerialized(const CsrGraph& g, const std::string& path) {
  const gk_status st = gk_graph_save_sg(g.device(), path.c_str());
  if (st == GK_ERR_INVALID) throw ConfigError(gk_last_error());
  detail::CheckStatus(st, "gk_graph_save_sg");
}

}  // namespace gapkit

#endif  // GAPKIT_B200_IO_HPP_
