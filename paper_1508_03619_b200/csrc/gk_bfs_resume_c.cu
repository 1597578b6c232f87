// gk_bfs_resume_c.cu -- the grid kernel reading the compact offsets,
// continuing a traversal the cluster kernel handed back.
#define GK_OFFMODE 1
#include "gk_bfs_grid.cuh"

namespace gk {

const void* bfs_resume_c_fn() { return reinterpret_cast<const void*>(bfs_persistent<true>); }

}  // namespace gk
