// gk_pack.cu -- compact device->host transfer of a ParentArray (gk_bfs_batch).
//
// gk_bfs_batch returns every source's full ParentArray (bfs.hpp:117-177's
// result, n int32) in host memory.  At scale 27 that is 537 MB per source over
// PCIe (~50 GB/s: 10.7 ms against a 2.3 ms traversal), so the batch is bound by
// the copy.  On Kronecker graphs about half of the vertices are unreached
// (kron27: 63.0 M of 134.2 M) and their parent is -1; the transfer therefore
// ships, per 1024-vertex block b,
//   off[b]            exclusive prefix of reached vertices before block b
//   bits[32 b + k]    reached bitmap of vertices [1024 b + 32 k, +32)
//   packed[off[b]..]  the reached vertices' parents in vertex order
// laid out contiguously as [off (nblk + 1)] [bits (32 nblk)] [packed (count)]
// so one cudaMemcpyAsync of (nblk + 1 + 32 nblk + count) words moves it.  The
// host expands it into the caller's array (gk_expand.cpp), overlapped with the
// next source's traversal and copy.  Three kernels: count (bitmap + block
// counts), a one-CTA scan, scatter -- 2 reads of the parent array and one
// write of the packed words, ~0.2 ms at scale 27, off the copy's critical
// path.
#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "gk_internal.cuh"

namespace gk {
namespace {

constexpr int kPkThreads = 256;
constexpr int kScanThreads = 1024;

__device__ __forceinline__ int warp_id_global() { return (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); }

// One warp per 1024-vertex block: 32 coalesced 128-byte loads in flight, one
// ballot each; lane k keeps word k of the block's bitmap.
__global__ void __launch_bounds__(kPkThreads) k_pack_count(const int32_t* __restrict__ parent, int64_t n,
                                                           int64_t nblk, uint32_t* __restrict__ bits,
                                                           uint32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp_id_global(); b < nblk; b += nw) {
    const int64_t v0 = b * 1024 + lane;
    int32_t p[32];
#pragma unroll
    for (int k = 0; k < 32; k++) p[k] = v0 + 32 * k < n ? parent[v0 + 32 * k] : -1;
    uint32_t mine = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < 32; k++) {
      const uint32_t m = __ballot_sync(0xffffffffu, p[k] >= 0);
      if (lane == k) mine = m;
      tot += __popc(m);
    }
    bits[b * 32 + lane] = mine;
    if (lane == 0) cnt[b] = tot;
  }
}

// Exclusive prefix of the block counts (nblk <= 2^21): each thread sums a
// contiguous run, one block-wide scan, then writes its run's offsets.
__global__ void __launch_bounds__(kScanThreads) k_pack_scan(const uint32_t* __restrict__ cnt, int64_t nblk,
                                                            uint32_t* __restrict__ off, int64_t probe,
                                                            volatile uint32_t* host_out) {
  typedef cub::BlockScan<uint32_t, kScanThreads> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const int64_t per = (nblk + kScanThreads - 1) / kScanThreads;
  const int64_t lo = min(nblk, (int64_t)threadIdx.x * per), hi = min(nblk, lo + per);
  uint32_t s = 0;
  for (int64_t i = lo; i < hi; i++) s += cnt[i];
  uint32_t ex = 0, total = 0;
  Scan(tmp).ExclusiveSum(s, ex, total);
  for (int64_t i = lo; i < hi; i++) {
    off[i] = ex;
    ex += cnt[i];
  }
  if (threadIdx.x == 0) off[nblk] = total;
  if (host_out) {  // mapped pinned memory: the total and off[probe] reach the host without a copy-engine slot
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      host_out[0] = total;
      host_out[1] = off[probe];
      __threadfence_system();
    }
  }
}

// Same walk as k_pack_count: lane l of word k stores its parent at
// off[b] + (reached before it in the block).
__global__ void __launch_bounds__(kPkThreads) k_pack_scatter(const int32_t* __restrict__ parent, int64_t n,
                                                             int64_t nblk, const uint32_t* __restrict__ off,
                                                             int32_t* __restrict__ packed) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp_id_global(); b < nblk; b += nw) {
    const int64_t v0 = b * 1024 + lane;
    uint32_t base = off[b];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      int32_t p[16];
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const int64_t v = v0 + 32 * (16 * h + k);
        p[k] = v < n ? parent[v] : -1;
      }
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const uint32_t m = __ballot_sync(0xffffffffu, p[k] >= 0);
        if (p[k] >= 0) packed[base + __popc(m & lt)] = p[k];
        base += __popc(m);
      }
    }
  }
}

int pack_grid(int64_t nblk) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (nblk + kPkThreads / 32 - 1) / (kPkThreads / 32);
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
}

}  // namespace

size_t pack_words(int64_t n) {
  const int64_t nblk = (n + 1023) / 1024;
  return (size_t)(nblk + 1 + 32 * nblk + n);
}

cudaError_t pack_count(const int32_t* parent, int64_t n, uint32_t* buf, uint32_t* cnt, int64_t probe,
                       uint32_t* host_out, cudaStream_t s) {
  const int64_t nblk = (n + 1023) / 1024;
  if (nblk > (int64_t(1) << 21) || probe < 0 || probe > nblk) return cudaErrorInvalidValue;
  k_pack_count<<<pack_grid(nblk), kPkThreads, 0, s>>>(parent, n, nblk, buf + nblk + 1, cnt);
  k_pack_scan<<<1, kScanThreads, 0, s>>>(cnt, nblk, buf, probe, host_out);
  return cudaGetLastError();
}

cudaError_t pack_scatter(const int32_t* parent, int64_t n, uint32_t* buf, cudaStream_t s) {
  const int64_t nblk = (n + 1023) / 1024;
  k_pack_scatter<<<pack_grid(nblk), kPkThreads, 0, s>>>(parent, n, nblk, buf,
                                                       reinterpret_cast<int32_t*>(buf + nblk + 1 + 32 * nblk));
  return cudaGetLastError();
}

}  // namespace gk
