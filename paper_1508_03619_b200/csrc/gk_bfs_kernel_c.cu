// gk_bfs_kernel_c.cu -- the grid kernel (gk_bfs_grid.cuh) reading the
// graph's compact offsets (BfsParams::off32), a fresh traversal.
#define GK_OFFMODE 1
#include "gk_bfs_grid.cuh"

namespace gk {

const void* bfs_fresh_c_fn() { return reinterpret_cast<const void*>(bfs_persistent<false>); }

}  // namespace gk
