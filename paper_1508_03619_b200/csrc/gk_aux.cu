// gk_aux.cu -- untimed auxiliary kernels: reached/component-edge counts, the
// algorithmic byte model of SURVEY.md §8(d) (the roofline numerator) and the
// device BFS certificate (§8(f)-2).  None runs inside the timed traversal.
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "gk_internal.cuh"

namespace gk {
namespace {

constexpr int kAuxBlock = 256;
constexpr int kLocalLevels = 64;

__device__ __forceinline__ unsigned long long sec_bytes(long long k) {
  return 32ull * (unsigned long long)((4 * k + 31) / 32);
}

template <typename T>
__device__ __forceinline__ T block_sum(T x, T* sm) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = x;
  __syncthreads();
  T t = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kAuxBlock / 32; i++) t += sm[i];
  __syncthreads();
  return t;
}

// Bit v set when v has no in-edges (it can never be reached from another
// vertex) or v >= n (padding of the last word).  The traversal seeds its
// visited map with it so bottom-up sweeps never revisit such vertices.
__global__ void k_dead(const int64_t* __restrict__ in_off, int64_t n, int64_t w32, uint32_t* __restrict__ dead) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // a multiple of 32
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < w32 * 32; v += stride) {
    const bool d = v >= n || in_off[v + 1] == in_off[v];
    const unsigned bits = __ballot_sync(0xffffffffu, d);
    if ((threadIdx.x & 31) == 0) dead[v >> 5] = bits;
  }
}

// CSR invariants every kernel relies on (graph.hpp:26-45): off[0] = 0,
// non-decreasing, off[n] = m, every neighbour id < n.
__global__ void k_validate_csr(const int64_t* __restrict__ off, const uint32_t* __restrict__ nb, int64_t n,
                               int64_t m, int64_t id_bound, unsigned long long* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    if (off[v] > off[v + 1] || off[v + 1] > m) atomicAdd(&bad[0], 1ull);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != m)) atomicAdd(&bad[0], 1ull);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
    if ((int64_t)nb[i] >= id_bound) atomicAdd(&bad[1], 1ull);
}

// Vertices with in-edges per CTA (popcount of ~dead), summed into *live.
__global__ void k_count_live(const uint32_t* __restrict__ dead, int64_t w32, unsigned long long* live) {
  __shared__ unsigned long long sm[kAuxBlock / 32];
  unsigned long long c = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < w32; w += (int64_t)gridDim.x * blockDim.x)
    c += __popc(~dead[w]);
  c = block_sum(c, sm);
  if (threadIdx.x == 0 && c) atomicAdd(live, c);
}

// Neighbour lists strictly ascending (graph.hpp:25: sorted, no duplicates):
// a warp per vertex compares each arc with its predecessor.
__global__ void k_check_sorted(const int64_t* __restrict__ off, const uint32_t* __restrict__ nb, int64_t n,
                               unsigned long long* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long c = 0;
  for (int64_t v = gw; v < n; v += nw) {
    const int64_t b = off[v], e = off[v + 1];
    for (int64_t j = b + 1 + lane; j < e; j += 32)
      if (nb[j] <= nb[j - 1]) c++;
  }
  if (c) atomicAdd(bad, c);
}


__global__ void k_canary(const unsigned char* __restrict__ p, size_t len, unsigned char fill,
                         unsigned long long* out) {
  unsigned long long c = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
    c += p[i] != fill;
  if (c) atomicAdd(out, c);
}

__global__ void k_count_reached(const int32_t* __restrict__ parent, const int64_t* __restrict__ off,
                                int64_t n, unsigned long long* out) {
  __shared__ unsigned long long sm[kAuxBlock / 32];
  unsigned long long r = 0, d = 0;
  for (long long v = (long long)blockIdx.x * kAuxBlock + threadIdx.x; v < n;
       v += (long long)gridDim.x * kAuxBlock) {
    if (parent[v] >= 0) {
      r++;
      d += (unsigned long long)(off[v + 1] - off[v]);
    }
  }
  r = block_sum(r, sm);
  d = block_sum(d, sm);
  if (threadIdx.x == 0) {
    atomicAdd(out, r);
    atomicAdd(out + 1, d);
  }
}

// Per-depth TD terms: acc[3*d+0] = |{depth==d}|, acc[3*d+1] = sum(36 + sec(deg)),
// acc[3*d+2] = sum(12 + 4 deg).  Levels < kLocalLevels are privatised in smem.
__global__ void k_model_levels(const int32_t* __restrict__ depth, const int64_t* __restrict__ off,
                               int64_t n, int32_t nlev, unsigned long long* acc) {
  __shared__ unsigned long long loc[kLocalLevels * 3];
  for (int i = threadIdx.x; i < kLocalLevels * 3; i += kAuxBlock) loc[i] = 0;
  __syncthreads();
  for (long long v = (long long)blockIdx.x * kAuxBlock + threadIdx.x; v < n;
       v += (long long)gridDim.x * kAuxBlock) {
    const int d = depth[v];
    if (d < 0 || d >= nlev) continue;
    const long long deg = off[v + 1] - off[v];
    const unsigned long long a = 36ull + sec_bytes(deg), b = 12ull + 4ull * deg;
    if (d < kLocalLevels) {
      atomicAdd(&loc[3 * d], 1ull);
      atomicAdd(&loc[3 * d + 1], a);
      atomicAdd(&loc[3 * d + 2], b);
    } else {
      atomicAdd(&acc[3 * d], 1ull);
      atomicAdd(&acc[3 * d + 1], a);
      atomicAdd(&acc[3 * d + 2], b);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kLocalLevels * 3 && i < nlev * 3; i += kAuxBlock)
    if (loc[i]) atomicAdd(&acc[i], loc[i]);
}

// BU step i terms: sum over unvisited (depth -1 or > i) vertices with in-arcs
// of (8 + sec(s_v)) and (8 + 4 s_v), s_v = arcs scanned to the first
// in-neighbour at depth i (all when none).
__global__ void k_model_bu(const int32_t* __restrict__ depth, const int64_t* __restrict__ in_off,
                           const uint32_t* __restrict__ in_nb, int64_t n, int32_t lvl,
                           unsigned long long* out) {
  __shared__ unsigned long long sm[kAuxBlock / 32];
  unsigned long long bs = 0, bu = 0;
  for (long long v = (long long)blockIdx.x * kAuxBlock + threadIdx.x; v < n;
       v += (long long)gridDim.x * kAuxBlock) {
    const int d = depth[v];
    if (d >= 0 && d <= lvl) continue;
    const long long b = in_off[v], e = in_off[v + 1];
    if (b == e) continue;
    long long sv = e - b;
    for (long long j = b; j < e; j++)
      if (depth[in_nb[j]] == lvl) {
        sv = j - b + 1;
        break;
      }
    bs += 8ull + sec_bytes(sv);
    bu += 8ull + 4ull * (unsigned long long)sv;
  }
  bs = block_sum(bs, sm);
  bu = block_sum(bu, sm);
  if (threadIdx.x == 0) {
    atomicAdd(out, bs);
    atomicAdd(out + 1, bu);
  }
}

// ---- device BFS certificate ---------------------------
// depth/parent of a finished BFS are a valid BFS iff
//   (1) depth[src] = 0, parent[src] = src;
//   (2) every reached v != src has parent p with an edge p->v and
//       depth[p] = depth[v]-1; every unreached v has parent -1;
//   (3) every arc v->w with v reached has w reached and depth[w] <= depth[v]+1.
// (2) gives depth >= true distance along the parent chain, (3) gives <= by
// induction along a shortest path, so the depths are exactly the BFS
// distances (the verify.hpp:62-98 conditions, without a serial BFS).
// errs: [0] source, [1] unreached-with-parent, [2] parent range, [3] parent
// depth, [4] missing parent edge, [5] arc reachability, [6] arc level,
// [7] first offending vertex (min).
__global__ void k_verify_vertices(const int64_t* __restrict__ off, const uint32_t* __restrict__ nb,
                                  const int32_t* __restrict__ parent, const int32_t* __restrict__ depth,
                                  int64_t n, uint32_t src, unsigned long long* errs) {
  for (long long v = (long long)blockIdx.x * kAuxBlock + threadIdx.x; v < n;
       v += (long long)gridDim.x * kAuxBlock) {
    const int d = depth[v], p = parent[v];
    int bad = -1;
    if (v == (long long)src) {
      if (p != (int)src || d != 0) bad = 0;
    } else if (d < 0) {
      if (p != -1) bad = 1;
    } else if (p < 0 || (int64_t)p >= n) {
      bad = 2;
    } else if (d < 1 || depth[p] != d - 1) {
      // d >= 1: only the source sits at depth 0, so every parent chain
      // descends to it (a depth-0 vertex whose parent is unreached, depth -1,
      // would otherwise pass d-1 == depth[p] and take a fake subtree with it
      // on a directed graph, where no reverse arc exposes it)
      bad = 3;
    } else {
      int64_t lo = off[p], hi = off[p + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (nb[mid] < (uint32_t)v) lo = mid + 1;
        else hi = mid;
      }
      if (lo >= off[p + 1] || nb[lo] != (uint32_t)v) bad = 4;
    }
    if (bad >= 0) {
      atomicAdd(&errs[bad], 1ull);
      atomicMin(&errs[7], (unsigned long long)v);
    }
  }
}

// Arc rule (3): a warp per 32 vertices, each list scanned 32 arcs at a time.
__global__ void k_verify_arcs(const int64_t* __restrict__ off, const uint32_t* __restrict__ nb,
                              const int32_t* __restrict__ depth, int64_t n, unsigned long long* errs) {
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * kAuxBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kAuxBlock) >> 5;
  for (long long base = gw * 32; base < n; base += nw * 32) {
    const long long mine = base + lane;
    const int dmine = mine < n ? depth[mine] : -1;
    unsigned todo = __ballot_sync(0xffffffffu, dmine >= 0);
    while (todo) {
      const int l = __ffs(todo) - 1;
      todo &= todo - 1;
      const long long v = base + l;
      const int dv = __shfl_sync(0xffffffffu, dmine, l);
      const int64_t b = off[v], e = off[v + 1];
      unsigned long long reach = 0, level = 0;
      for (int64_t j = b + lane; j < e; j += 32) {
        const int dw = depth[nb[j]];
        if (dw < 0) reach++;
        else if (dw > dv + 1) level++;
      }
      if (reach | level) {
        atomicAdd(&errs[5], reach);
        atomicAdd(&errs[6], level);
        atomicMin(&errs[7], (unsigned long long)v);
      }
    }
  }
}

int aux_grid(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long want = (n + kAuxBlock - 1) / kAuxBlock;
  long long cap = (long long)sms * 8;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

// Compact offsets: low 32 bits of every offset; the first vertex of each
// 2^32 block of arcs goes to hi[block - 1] (one vertex's list is shorter
// than 2^32 arcs, so consecutive offsets cross at most one block edge).
__global__ void k_off32(const int64_t* off, int64_t n, uint32_t* off32, uint32_t* hi, int nhi) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = t; v <= n; v += nt) {
    const int64_t o = off[v];
    off32[v] = (uint32_t)o;
    if (v > 0) {
      const int64_t b = o >> 32, a = off[v - 1] >> 32;
      for (int64_t k = a; k < b && k < nhi; k++) hi[k] = (uint32_t)v;
    }
  }
}

}  // namespace

cudaError_t compact_offsets(const int64_t* off, int64_t n, uint32_t* off32, uint32_t* hi, int nhi, cudaStream_t s) {
  k_off32<<<aux_grid(n + 1), kAuxBlock, 0, s>>>(off, n, off32, hi, nhi);
  return cudaGetLastError();
}

cudaError_t dead_bitmap(const int64_t* in_off, int64_t n, uint32_t* dead, int64_t* live, cudaStream_t s) {
  const int64_t w32 = (n + 31) / 32;
  *live = 0;
  if (w32 == 0) return cudaSuccess;
  k_dead<<<aux_grid(w32 * 32), kAuxBlock, 0, s>>>(in_off, n, w32, dead);
  unsigned long long* d = nullptr;
  unsigned long long h = 0;
  cudaError_t e = cudaMallocAsync(&d, sizeof(h), s);
  if (e) return e;
  if (!(e = cudaMemsetAsync(d, 0, sizeof(h), s))) {
    k_count_live<<<aux_grid(w32), kAuxBlock, 0, s>>>(dead, w32, d);
    if (!(e = cudaGetLastError()) && !(e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s)))
      e = cudaStreamSynchronize(s);
  }
  cudaFreeAsync(d, s);
  *live = (int64_t)h;
  return e;
}

cudaError_t validate_csr(const int64_t* off, const uint32_t* nb, int64_t n, int64_t m, int64_t id_bound,
                         bool* offsets_ok, bool* ids_ok, bool* sorted, cudaStream_t s) {
  unsigned long long* bad = nullptr;
  unsigned long long hb[3] = {0, 0, 0};
  cudaError_t e;
  if ((e = cudaMalloc(&bad, sizeof(hb)))) return e;
  if (!(e = cudaMemsetAsync(bad, 0, sizeof(hb), s))) {
    k_validate_csr<<<aux_grid(std::max<int64_t>(n, m)), kAuxBlock, 0, s>>>(off, nb, n, m, id_bound, bad);
    e = cudaGetLastError();
    if (!e && sorted) {
      e = cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s);
      if (!e) e = cudaStreamSynchronize(s);
      if (!e && hb[0] == 0) {  // list bounds are trustworthy
        k_check_sorted<<<aux_grid(32 * n), kAuxBlock, 0, s>>>(off, nb, n, bad + 2);
        e = cudaGetLastError();
      }
    }
    if (!e && !(e = cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s))) e = cudaStreamSynchronize(s);
  }
  cudaFree(bad);
  *offsets_ok = hb[0] == 0;
  *ids_ok = hb[1] == 0;
  if (sorted) *sorted = hb[0] == 0 && hb[2] == 0;
  return e;
}

cudaError_t canary_count(const void* p, size_t len, unsigned char fill, unsigned long long* d_out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), s);
  if (e) return e;
  k_canary<<<16, kAuxBlock, 0, s>>>(static_cast<const unsigned char*>(p), len, fill, d_out);
  return cudaGetLastError();
}

cudaError_t count_reached(const int32_t* parent, const int64_t* off, int64_t n,
                          unsigned long long* d_out2, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(d_out2, 0, 2 * sizeof(unsigned long long), s);
  if (e) return e;
  k_count_reached<<<aux_grid(n), kAuxBlock, 0, s>>>(parent, off, n, d_out2);
  return cudaGetLastError();
}

cudaError_t verify_bfs(const int64_t* off, const uint32_t* nb, const int32_t* parent, const int32_t* depth,
                       int64_t n, uint32_t src, long long* errs8, cudaStream_t s) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 8 * sizeof(unsigned long long), s);
  if (e) return e;
  unsigned long long init[8] = {0, 0, 0, 0, 0, 0, 0, ~0ull};
  cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, s);
  k_verify_vertices<<<aux_grid(n), kAuxBlock, 0, s>>>(off, nb, parent, depth, n, src, d);
  k_verify_arcs<<<aux_grid(n), kAuxBlock, 0, s>>>(off, nb, depth, n, d);
  unsigned long long h[8];
  e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  cudaFreeAsync(d, s);
  for (int i = 0; i < 8; i++) errs8[i] = (long long)h[i];
  if (h[7] == ~0ull) errs8[7] = -1;
  return e;
}

cudaError_t byte_model(const BfsParams& p, const int32_t* depth, const char* dirs, int32_t nsteps,
                       unsigned long long* /*unused*/, double* b_sec, double* b_use,
                       cudaStream_t s) {
  const int32_t nlev = nsteps + 2;
  unsigned long long* acc = nullptr;
  size_t bytes = sizeof(unsigned long long) * (3 * (size_t)nlev + 2);
  cudaError_t e = cudaMallocAsync(&acc, bytes, s);
  if (e) return e;
  cudaMemsetAsync(acc, 0, bytes, s);
  k_model_levels<<<aux_grid(p.n), kAuxBlock, 0, s>>>(depth, p.out_off, p.n, nlev, acc);
  std::vector<unsigned long long> lev(3 * (size_t)nlev + 2);
  const double W = (double)((p.n + 7) / 8);
  double bs = 4.0 * (double)p.n, bu = 4.0 * (double)p.n;
  std::vector<double> bu_sec(nsteps, 0.0), bu_use(nsteps, 0.0);
  unsigned long long* tail = acc + 3 * (size_t)nlev;
  for (int i = 0; i < nsteps; i++) {
    if (dirs[i] != 'B') continue;
    cudaMemsetAsync(tail, 0, 2 * sizeof(unsigned long long), s);
    k_model_bu<<<aux_grid(p.n), kAuxBlock, 0, s>>>(depth, p.in_off, p.in_nb, p.n, i, tail);
    unsigned long long two[2];
    e = cudaMemcpyAsync(two, tail, sizeof(two), cudaMemcpyDeviceToHost, s);
    if (e) break;
    cudaStreamSynchronize(s);
    bu_sec[i] = (double)two[0];
    bu_use[i] = (double)two[1];
  }
  if (!e) e = cudaMemcpyAsync(lev.data(), acc, lev.size() * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  cudaFreeAsync(acc, s);
  if (e) return e;
  auto cnt = [&](int d) { return (double)lev[3 * (size_t)d]; };
  for (int i = 0; i < nsteps; i++) {
    if (dirs[i] == 'T') {
      bs += (double)lev[3 * (size_t)i + 1] + 36.0 * cnt(i + 1);
      bu += (double)lev[3 * (size_t)i + 2] + 4.0 * cnt(i + 1);
    } else {
      if (i == 0 || dirs[i - 1] != 'B') {
        bs += W + 4.0 * cnt(i);
        bu += W + 4.0 * cnt(i);
      }
      bs += 3.0 * W + bu_sec[i];
      bu += 3.0 * W + bu_use[i];
      if (i + 1 == nsteps || dirs[i + 1] != 'B') {
        bs += W + 4.0 * cnt(i + 1);
        bu += W + 4.0 * cnt(i + 1);
      }
    }
  }
  *b_sec = bs;
  *b_use = bu;
  return cudaSuccess;
}

}  // namespace gk
