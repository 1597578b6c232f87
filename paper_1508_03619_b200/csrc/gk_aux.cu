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

__global__ void k_live_count(const uint32_t* __restrict__ dead, int64_t w32, uint32_t* __restrict__ cnt) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < w32; w += (int64_t)gridDim.x * blockDim.x)
    cnt[w] = __popc(~dead[w]);
}

// Heads are stored only for live (not dead) vertices, in vertex order:
// v's record is hbase[v/32] + (live vertices before v in its word).
__global__ void k_head(const int64_t* __restrict__ in_off, const uint32_t* __restrict__ in_nb, int64_t n,
                       const uint32_t* __restrict__ dead, const uint32_t* __restrict__ hbase,
                       HeadRec* __restrict__ head, HeadRec* __restrict__ head2) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t live = ~dead[v >> 5];
    const uint32_t bit = (uint32_t)(v & 31);
    if (!((live >> bit) & 1u)) continue;
    const int64_t idx = (int64_t)hbase[v >> 5] + __popc(live & ((1u << bit) - 1u));
    const int64_t b = in_off[v], d = in_off[v + 1] - b;
    uint32_t h[kHead];
#pragma unroll
    for (int j = 0; j < kHead; j++) h[j] = j < d ? in_nb[b + j] : kNoVertex;
    head[idx] = head_pack(h, (HeadRec*)nullptr);
    if (head2) {
#pragma unroll
      for (int j = 0; j < kHead; j++) h[j] = kHead + j < d ? in_nb[b + kHead + j] : kNoVertex;
      head2[idx] = head_pack(h, (HeadRec*)nullptr);
    }
  }
}

// Owned-range split rows (gk_internal.cuh OwnEnt).
__global__ void k_hv_bits(const int64_t* __restrict__ off, int64_t n, int64_t w32, int64_t dmin,
                          uint32_t* __restrict__ bits) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < w32 * 32;
       v += (int64_t)gridDim.x * blockDim.x) {
    const bool h = v < n && off[v + 1] - off[v] >= dmin;
    const unsigned b = __ballot_sync(0xffffffffu, h);
    if ((threadIdx.x & 31) == 0) bits[v >> 5] = b;
  }
}

__global__ void k_popc(const uint32_t* __restrict__ bits, int64_t w32, uint32_t* __restrict__ cnt) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < w32; w += (int64_t)gridDim.x * blockDim.x)
    cnt[w] = __popc(bits[w]);
}

__global__ void k_hv_list(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ base, int64_t w32,
                          uint32_t* __restrict__ ids) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < w32; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = bits[w], r = base[w];
    while (b) {
      ids[r++] = (uint32_t)(w * 32 + __ffs(b) - 1);
      b &= b - 1;
    }
  }
}

// One CTA per row: check the list is ascending, then row[r] = lower_bound of
// r*span in it for r = 0..nr.
__global__ void k_split(const int64_t* __restrict__ off, const uint32_t* __restrict__ nb,
                        const uint32_t* __restrict__ ids, int nr, int64_t span, uint32_t* __restrict__ split,
                        unsigned long long* bad) {
  const uint32_t u = ids[blockIdx.x];
  const int64_t b = off[u], d = off[u + 1] - b;
  for (int64_t i = threadIdx.x + 1; i < d; i += blockDim.x)
    if (nb[b + i] < nb[b + i - 1]) atomicAdd(bad, 1ull);
  for (int r = threadIdx.x; r <= nr; r += blockDim.x) {
    const int64_t t = (int64_t)r * span;
    int64_t lo = 0, hi = d;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)nb[b + mid] < t) lo = mid + 1;
      else hi = mid;
    }
    split[(int64_t)blockIdx.x * (nr + 1) + r] = (uint32_t)lo;
  }
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
    } else if (depth[p] != d - 1) {
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

// Out-degree per vertex clamped to 65535 (= "read the offsets"), zero past
// n up to a whole bitmap word: the large top-down step's claim sweep sums
// the claimed vertices' degrees from these 2n bytes instead of from the
// 8n-byte offsets.
__global__ void k_deg16(const int64_t* off, int64_t n, int64_t nw, uint16_t* deg16) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nw; v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = 0;
    if (v < n) d = off[v + 1] - off[v];
    deg16[v] = (uint16_t)(d < 65535 ? d : 65535);
  }
}

}  // namespace

cudaError_t build_deg16(const int64_t* off, int64_t n, uint16_t* deg16, cudaStream_t s) {
  const int64_t nw = (n + 31) / 32 * 32;
  if (nw == 0) return cudaSuccess;
  k_deg16<<<aux_grid(nw), kAuxBlock, 0, s>>>(off, n, nw, deg16);
  return cudaGetLastError();
}

cudaError_t dead_bitmap(const int64_t* in_off, int64_t n, uint32_t* dead, cudaStream_t s) {
  const int64_t w32 = (n + 31) / 32;
  k_dead<<<aux_grid(w32 * 32), kAuxBlock, 0, s>>>(in_off, n, w32, dead);
  return cudaGetLastError();
}

cudaError_t validate_csr(const int64_t* off, const uint32_t* nb, int64_t n, int64_t m, int64_t id_bound,
                         bool* offsets_ok, bool* ids_ok, cudaStream_t s) {
  unsigned long long* bad = nullptr;
  unsigned long long hb[2] = {0, 0};
  cudaError_t e;
  if ((e = cudaMalloc(&bad, sizeof(hb)))) return e;
  if (!(e = cudaMemsetAsync(bad, 0, sizeof(hb), s))) {
    k_validate_csr<<<aux_grid(std::max<int64_t>(n, m)), kAuxBlock, 0, s>>>(off, nb, n, m, id_bound, bad);
    if (!(e = cudaGetLastError()) && !(e = cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s)))
      e = cudaStreamSynchronize(s);
  }
  cudaFree(bad);
  *offsets_ok = hb[0] == 0;
  *ids_ok = hb[1] == 0;
  return e;
}

cudaError_t build_head(const int64_t* in_off, const uint32_t* in_nb, int64_t n, const uint32_t* dead,
                       uint32_t* hbase, HeadRec** head, HeadRec** head2, int64_t* nlive, cudaStream_t s) {
  const int64_t w32 = (n + 31) / 32;
  *head = nullptr;
  *nlive = 0;
  if (head2) *head2 = nullptr;
  if (w32 == 0) return cudaSuccess;
  uint32_t* cnt = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  uint32_t last[2] = {0, 0};
  cudaError_t e;
  if ((e = cudaMalloc(&cnt, sizeof(uint32_t) * (w32 + 1)))) return e;
  k_live_count<<<aux_grid(w32), kAuxBlock, 0, s>>>(dead, w32, cnt);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, hbase, (int)w32, s))) goto out;
  if ((e = cudaMalloc(&tmp, tb))) goto out;
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, hbase, (int)w32, s))) goto out;
  if ((e = cudaMemcpyAsync(&last[0], hbase + w32 - 1, 4, cudaMemcpyDeviceToHost, s))) goto out;
  if ((e = cudaMemcpyAsync(&last[1], cnt + w32 - 1, 4, cudaMemcpyDeviceToHost, s))) goto out;
  if ((e = cudaStreamSynchronize(s))) goto out;
  {
    const int64_t live = (int64_t)last[0] + last[1];
    *nlive = live;
    if ((e = cudaMalloc(head, sizeof(HeadRec) * (live > 0 ? live : 1)))) goto out;
    if (head2 && cudaMalloc(head2, sizeof(HeadRec) * (live > 0 ? live : 1)) != cudaSuccess) {
      cudaGetLastError();  // optional: without it the second round reads in_off/in_nb
      *head2 = nullptr;
    }
    k_head<<<aux_grid(n), kAuxBlock, 0, s>>>(in_off, in_nb, n, dead, hbase, *head, head2 ? *head2 : nullptr);
    e = cudaGetLastError();
  }
out:
  cudaFree(tmp);
  cudaFree(cnt);
  return e;
}

cudaError_t build_own(const int64_t* out_off, const uint32_t* out_nb, int64_t n, int64_t dmin, int r,
                      int64_t span_w, size_t max_bytes, uint32_t** hv_bits, uint32_t** hv_base,
                      uint32_t** split, int64_t* nh, cudaStream_t s) {
  const int64_t w32 = (n + 31) / 32;
  *hv_bits = *hv_base = *split = nullptr;
  *nh = 0;
  if (w32 == 0 || r < 1) return cudaSuccess;
  uint32_t* cnt = nullptr;
  uint32_t* ids = nullptr;
  unsigned long long* bad = nullptr;
  unsigned long long hbad = 0;
  void* tmp = nullptr;
  size_t tb = 0;
  uint32_t last[2] = {0, 0};
  int64_t rows = 0;
  cudaError_t e;
  if ((e = cudaMalloc(hv_bits, sizeof(uint32_t) * w32))) goto out;
  if ((e = cudaMalloc(hv_base, sizeof(uint32_t) * w32))) goto out;
  if ((e = cudaMalloc(&cnt, sizeof(uint32_t) * w32))) goto out;
  k_hv_bits<<<aux_grid(w32 * 32), kAuxBlock, 0, s>>>(out_off, n, w32, dmin, *hv_bits);
  k_popc<<<aux_grid(w32), kAuxBlock, 0, s>>>(*hv_bits, w32, cnt);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, *hv_base, (int)w32, s))) goto out;
  if ((e = cudaMalloc(&tmp, tb))) goto out;
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, *hv_base, (int)w32, s))) goto out;
  if ((e = cudaMemcpyAsync(&last[0], *hv_base + w32 - 1, 4, cudaMemcpyDeviceToHost, s))) goto out;
  if ((e = cudaMemcpyAsync(&last[1], cnt + w32 - 1, 4, cudaMemcpyDeviceToHost, s))) goto out;
  if ((e = cudaStreamSynchronize(s))) goto out;
  rows = (int64_t)last[0] + last[1];
  if (rows == 0 || (size_t)rows * (r + 1) * 4 > max_bytes) goto out;
  if ((e = cudaMalloc(&ids, sizeof(uint32_t) * rows))) goto out;
  if ((e = cudaMalloc(split, sizeof(uint32_t) * rows * (r + 1)))) goto out;
  if ((e = cudaMalloc(&bad, sizeof(unsigned long long)))) goto out;
  if ((e = cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s))) goto out;
  k_hv_list<<<aux_grid(w32), kAuxBlock, 0, s>>>(*hv_bits, *hv_base, w32, ids);
  k_split<<<(unsigned)rows, 512, 0, s>>>(out_off, out_nb, ids, r, span_w * 32, *split, bad);
  if ((e = cudaGetLastError())) goto out;
  if ((e = cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, s))) goto out;
  if ((e = cudaStreamSynchronize(s))) goto out;
  if (hbad == 0) *nh = rows;
out:
  cudaFree(tmp);
  cudaFree(cnt);
  cudaFree(ids);
  cudaFree(bad);
  if (*nh == 0) {  // off: nothing qualifies, a list is unsorted, too large, or an error
    cudaFree(*hv_bits);
    cudaFree(*hv_base);
    cudaFree(*split);
    *hv_bits = *hv_base = *split = nullptr;
  }
  return e;
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
