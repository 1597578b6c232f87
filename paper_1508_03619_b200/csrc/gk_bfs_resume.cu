// gk_bfs_resume.cu -- the grid kernel instantiated for a traversal that
// continues after the cluster kernel handed it back (see gk_bfs_grid.cuh).
#define GK_OFFMODE 0
#include "gk_bfs_grid.cuh"

namespace gk {

const void* bfs_resume_fn() { return reinterpret_cast<const void*>(bfs_persistent<true>); }

}  // namespace gk
