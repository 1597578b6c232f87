// gk_bfs_kernel.cu -- direction-optimizing BFS as ONE persistent kernel.
//
// Restates gapkit::Bfs (proj/include/gapkit/kernels/bfs.hpp:117-177) for
// sm_100a.  The whole level loop runs on the device: one cooperative launch
// of 148 x k CTAs, grid barriers between phases, and the reference's
// alpha/beta direction decision (bfs.hpp:143-144, 153-154, 156, 158)
// evaluated redundantly by every thread from counters reduced in L2.  No
// host round trip per level, so high-diameter graphs pay ~a grid barrier
// per level instead of a launch + sync.
//
// Phases (each ends at a grid barrier):
//   init      parent[:] = -1 (a memset just ahead of the kernel, see bfs_launch),
//             visited := dead set, parent[src] = src, queue = [src]
//             (replaces the degree-encoding init bfs.hpp:126-132: the
//             claim test uses a 1-bit visited map in L2 instead of the
//             parent sign, and the claimed vertex's degree -- what the
//             encoding carries -- is read from the offsets at claim time;
//             scout = sum(max(deg,1)) is identical to sum(-old) of
//             bfs.hpp:83)
//   TD light  frontier tiles of 512 vertices, CTA-wide scan of degrees,
//             load-balanced edge gather (bfs.hpp:68-91); vertices of degree
//             > chunk are cut into chunk-edge chunks (128..1024 by step size)
//   TD heavy  chunks spread over all warps (hub expansion)
//   q2b       QueueToBitmap (bfs.hpp:93-97)
//   BU        one warp per 32-vertex bitmap word: visited-word skip, per-lane
//             scan of the first 4 in-neighbours, then warp-ballot scans of
//             the remaining lists; the first hit in ascending order is the
//             parent exactly as bfs.hpp:55-60 picks it
//   b2q       BitmapToQueue (bfs.hpp:99-113), CTA-aggregated appends
//   rescan    kTopDownRescan's extra degree pass (bfs.hpp:161-167)
#define GK_OFFMODE 0  // int64 offsets; gk_bfs_kernel_c.cu: the compact ones
#include "gk_bfs_grid.cuh"

namespace gk {
namespace {

// parent := -1 ahead of the traversal kernel (see bfs_launch)
__global__ void __launch_bounds__(512) k_fill_parent(int4* p4, long long n4, int32_t* p, long long n) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  const int4 m1 = make_int4(-1, -1, -1, -1);
#pragma unroll 4
  for (long long i = t; i < n4; i += nt) p4[i] = m1;
  for (long long i = (n4 << 2) + t; i < n; i += nt) p[i] = -1;
}

}  // namespace

cudaError_t bfs_configure(int device, BfsLaunch* cfg) {
  cudaError_t e;
  int sms = 0, optin = 0, coop = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device))) return e;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device))) return e;
  if ((e = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device))) return e;
  if (!coop) return cudaErrorNotSupported;
  cfg->smem_static = sizeof(SmemT);
  // Stage the front bitmap in shared memory when it fits next to the
  // static part at 1 CTA/SM; otherwise it is read through L1/L2.
  const size_t budget = (size_t)optin > cfg->smem_static + 1024 ? optin - cfg->smem_static - 1024 : 0;
  cfg->smem_front_max = budget & ~size_t(15);
  const void* fns[4] = {(const void*)bfs_persistent<false>, bfs_resume_fn(), bfs_fresh_c_fn(), bfs_resume_c_fn()};
  int occ = 1 << 30;
  for (const void* f : fns) {
    if ((e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg->smem_front_max)))
      return e;
    int o = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, f, kBlock, 0))) return e;
    occ = std::min(occ, o);
  }
  if (occ < 1) return cudaErrorInvalidConfiguration;
  cfg->grid = sms * occ;
  cfg->block = kBlock;
  size_t keep = 0;
  if ((e = cudaOccupancyAvailableDynamicSMemPerBlock(&keep, bfs_persistent<false>, occ, kBlock))) return e;
  cfg->smem_keep_occ = keep & ~size_t(15);
  return cudaSuccess;
}

cudaError_t bfs_launch(const BfsParams& p, const BfsLaunch& cfg, cudaStream_t st) {
  const void* fn = p.off32 ? (p.resume ? bfs_resume_c_fn() : bfs_fresh_c_fn())
                           : (p.resume ? bfs_resume_fn() : (const void*)bfs_persistent<false>);
  size_t dyn = 0;
  int grid = cfg.grid;
  if (p.front_in_smem) {
    dyn = ((size_t)p.w32 * 4 + 15) & ~size_t(15);
    int occ = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, dyn);
    if (e) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    grid = sms * occ;
  } else {
    // bottom-up pending lists; the owned-range slice when hub expansion is on
    dyn = kBuListBytes;
    if (p.own_list) {
      if (p.own_r != grid) return cudaErrorInvalidConfiguration;
      dyn = std::max(dyn, (size_t)p.own_span_w * 4);
    }
    if (dyn > cfg.smem_keep_occ) return cudaErrorInvalidConfiguration;
  }
  BfsParams local = p;
  // barrier counter, counter ring, step count, trace tags := 0
  if (cudaError_t e = cudaMemsetAsync(p.ctrl, 0, kCtrlClear, st)) return e;
  // parent := -1 ahead of the kernel on the launch stream, inside the
  // caller's timed region.  GK_INIT_MODE: 1 (default) cudaMemsetAsync,
  // measured 1% faster per BFS at scale 27 than 0 (the same stores in the
  // kernel's init phase) or 2 (a fill kernel); gk_bfs_batch's overlapped
  // parent copies run at the same rate with all three.  Below 2^22 vertices
  // the init phase clears parent (kron16: the memset launch cost 7 %).
  static const int init_mode = getenv("GK_INIT_MODE") ? atoi(getenv("GK_INIT_MODE")) : GK_INIT_MODE_DEF;
  if (p.resume) {
    // the traversal's arrays are live: nothing to initialise
  } else if (init_mode == 1 && p.n >= (int64_t(1) << 22)) {  // small graphs: the extra launch costs more than it saves
    cudaError_t e = cudaMemsetAsync(p.parent, 0xFF, sizeof(int32_t) * (size_t)p.n, st);
    if (e) return e;
    local.parent_preset = 1;
  } else if (init_mode == 2 && !p.resume) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_fill_parent<<<sms * 4, 512, 0, st>>>(reinterpret_cast<int4*>(p.parent), p.n >> 2, p.parent, p.n);
    cudaError_t e = cudaGetLastError();
    if (e) return e;
    local.parent_preset = 1;
  }
  void* args[] = {&local};
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(cfg.block), args, dyn, st);
}

}  // namespace gk
